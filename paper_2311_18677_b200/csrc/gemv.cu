// Decode linear layers: weight-streaming skinny GEMM for M = 1..16 rows.
//
//   out[m, n] = epilogue( sum_k x[m,k] * W[n,k] )
//
// At decode batch sizes the step is > 95 % weight bytes, so
// this kernel is an HBM-bandwidth kernel: every weight byte is read exactly
// once with 128-bit non-allocating loads, each warp streams 4 weight rows with
// 4 independent 16-byte loads per row in flight per lane, and the tiny
// activation block x (<= 16 rows) is served from L1.  fp32 accumulation,
// warp-shuffle reduction, fused epilogues identical to swb_gemm_bf16.
//
// Replaces PerfModel.token_iter_time (reference perf.py:125-132) for the
// linear layers of a token-phase iteration.
#include "common.cuh"

namespace swb {

constexpr int GV_ROWS = 4;     // weight rows per warp
constexpr int GV_UNROLL = 4;   // 16-byte chunks per row in flight per lane
constexpr int GV_WARPS = 4;    // warps per CTA

template <int MB>
__global__ void __launch_bounds__(GV_WARPS * 32)
    gemv_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                     const __nv_bfloat16* __restrict__ W, void* out,
                     const float* resid, int M, int N, int K,
                     int epi) {
  const int lane = threadIdx.x & 31;
  const int gwarp = blockIdx.x * GV_WARPS + (threadIdx.x >> 5);
  const bool swiglu = epi == SWB_EPI_SWIGLU;
  // weight rows handled by this warp
  int wrow[GV_ROWS];
  int out0;
  if (swiglu) {
    // 2 outputs per warp; output o uses gate row g(o) and up row g(o)+128
    out0 = gwarp * 2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int o = out0 + j;
      const int g = (o >> 7) * 256 + (o & 127);
      wrow[2 * j] = g;
      wrow[2 * j + 1] = g + 128;
    }
    if (out0 >= (N >> 1)) return;
  } else {
    out0 = gwarp * GV_ROWS;
#pragma unroll
    for (int j = 0; j < GV_ROWS; ++j) wrow[j] = out0 + j;
    if (out0 >= N) return;
  }
  bool rvalid[GV_ROWS];
#pragma unroll
  for (int j = 0; j < GV_ROWS; ++j) {
    rvalid[j] = wrow[j] < N;
    if (!rvalid[j]) wrow[j] = 0;
  }

  float acc[GV_ROWS][MB];
#pragma unroll
  for (int j = 0; j < GV_ROWS; ++j)
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[j][m] = 0.f;

  const int nchunk = K >> 3;  // 8 bf16 per 16-byte chunk
  const uint4* Wv = reinterpret_cast<const uint4*>(W);
  const uint4* xv = reinterpret_cast<const uint4*>(x);

  int c = lane;
  for (; c + 32 * (GV_UNROLL - 1) < nchunk; c += 32 * GV_UNROLL) {
    uint4 wv[GV_ROWS][GV_UNROLL];
#pragma unroll
    for (int j = 0; j < GV_ROWS; ++j)
#pragma unroll
      for (int u = 0; u < GV_UNROLL; ++u)
        wv[j][u] = ld_nc_v4(Wv + (size_t)wrow[j] * nchunk + c + 32 * u);
#pragma unroll
    for (int u = 0; u < GV_UNROLL; ++u) {
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        if (m >= M) break;
        const uint4 xq = xv[(size_t)m * nchunk + c + 32 * u];
        const float2 x0 = bf2_to_f2(xq.x), x1 = bf2_to_f2(xq.y),
                     x2 = bf2_to_f2(xq.z), x3 = bf2_to_f2(xq.w);
#pragma unroll
        for (int j = 0; j < GV_ROWS; ++j) {
          const float2 w0 = bf2_to_f2(wv[j][u].x), w1 = bf2_to_f2(wv[j][u].y),
                       w2 = bf2_to_f2(wv[j][u].z), w3 = bf2_to_f2(wv[j][u].w);
          float a = acc[j][m];
          a = fmaf(x0.x, w0.x, a); a = fmaf(x0.y, w0.y, a);
          a = fmaf(x1.x, w1.x, a); a = fmaf(x1.y, w1.y, a);
          a = fmaf(x2.x, w2.x, a); a = fmaf(x2.y, w2.y, a);
          a = fmaf(x3.x, w3.x, a); a = fmaf(x3.y, w3.y, a);
          acc[j][m] = a;
        }
      }
    }
  }
  for (; c < nchunk; c += 32) {
    uint4 wv[GV_ROWS];
#pragma unroll
    for (int j = 0; j < GV_ROWS; ++j) wv[j] = ld_nc_v4(Wv + (size_t)wrow[j] * nchunk + c);
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      if (m >= M) break;
      const uint4 xq = xv[(size_t)m * nchunk + c];
      const float2 x0 = bf2_to_f2(xq.x), x1 = bf2_to_f2(xq.y), x2 = bf2_to_f2(xq.z),
                   x3 = bf2_to_f2(xq.w);
#pragma unroll
      for (int j = 0; j < GV_ROWS; ++j) {
        const float2 w0 = bf2_to_f2(wv[j].x), w1 = bf2_to_f2(wv[j].y),
                     w2 = bf2_to_f2(wv[j].z), w3 = bf2_to_f2(wv[j].w);
        float a = acc[j][m];
        a = fmaf(x0.x, w0.x, a); a = fmaf(x0.y, w0.y, a);
        a = fmaf(x1.x, w1.x, a); a = fmaf(x1.y, w1.y, a);
        a = fmaf(x2.x, w2.x, a); a = fmaf(x2.y, w2.y, a);
        a = fmaf(x3.x, w3.x, a); a = fmaf(x3.y, w3.y, a);
        acc[j][m] = a;
      }
    }
  }

#pragma unroll
  for (int j = 0; j < GV_ROWS; ++j)
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[j][m] = warp_sum(acc[j][m]);

  // lane m writes row m's outputs (lanes >= M idle)
#pragma unroll
  for (int m = 0; m < MB; ++m) {
    if (m >= M) break;
    if (lane != (m & 31)) continue;
    if (swiglu) {
      const int nout = N >> 1;
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + (size_t)m * nout;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int oi = out0 + j;
        if (oi < nout && rvalid[2 * j]) {
          const float g = acc[2 * j][m], u = acc[2 * j + 1][m];
          o[oi] = __float2bfloat16(g / (1.f + __expf(-g)) * u);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < GV_ROWS; ++j) {
        if (!rvalid[j]) continue;
        const size_t idx = (size_t)m * N + wrow[j];
        if (epi == SWB_EPI_BF16)
          reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(acc[j][m]);
        else if (epi == SWB_EPI_F32)
          reinterpret_cast<float*>(out)[idx] = acc[j][m];
        else
          reinterpret_cast<float*>(out)[idx] = resid[idx] + acc[j][m];
      }
    }
  }
}

}  // namespace swb

using namespace swb;

extern "C" int swb_gemv_bf16(const void* x, const void* w, void* out,
                             const void* resid, int M, int N, int K, int epilogue,
                             uintptr_t stream) {
  SWB_REQUIRE(x && w && out, "swb_gemv_bf16: null pointer");
  SWB_REQUIRE(M >= 1 && M <= 16, "swb_gemv_bf16: M=%d outside 1..16", M);
  SWB_REQUIRE(N > 0 && K > 0 && K % 8 == 0, "swb_gemv_bf16: bad shape N=%d K=%d", N, K);
  SWB_REQUIRE(epilogue >= SWB_EPI_BF16 && epilogue <= SWB_EPI_SWIGLU,
              "swb_gemv_bf16: bad epilogue %d", epilogue);
  SWB_REQUIRE(epilogue != SWB_EPI_SWIGLU || N % 256 == 0,
              "swb_gemv_bf16: SwiGLU needs N %% 256 == 0");
  SWB_REQUIRE(epilogue != SWB_EPI_RESID_F32 || resid, "swb_gemv_bf16: resid needed");
  SWB_REQUIRE((((uintptr_t)x | (uintptr_t)w) & 15) == 0,
              "swb_gemv_bf16: pointers must be 16-byte aligned");
  const int warps = epilogue == SWB_EPI_SWIGLU ? (N / 2 + 1) / 2 : (N + GV_ROWS - 1) / GV_ROWS;
  const int grid = (warps + GV_WARPS - 1) / GV_WARPS;
  auto xs = reinterpret_cast<const __nv_bfloat16*>(x);
  auto ws = reinterpret_cast<const __nv_bfloat16*>(w);
  auto rs = reinterpret_cast<const float*>(resid);
  cudaStream_t s = (cudaStream_t)stream;
  if (M == 1)
    gemv_bf16_kernel<1><<<grid, GV_WARPS * 32, 0, s>>>(xs, ws, out, rs, M, N, K, epilogue);
  else if (M <= 2)
    gemv_bf16_kernel<2><<<grid, GV_WARPS * 32, 0, s>>>(xs, ws, out, rs, M, N, K, epilogue);
  else if (M <= 4)
    gemv_bf16_kernel<4><<<grid, GV_WARPS * 32, 0, s>>>(xs, ws, out, rs, M, N, K, epilogue);
  else if (M <= 8)
    gemv_bf16_kernel<8><<<grid, GV_WARPS * 32, 0, s>>>(xs, ws, out, rs, M, N, K, epilogue);
  else
    gemv_bf16_kernel<16><<<grid, GV_WARPS * 32, 0, s>>>(xs, ws, out, rs, M, N, K, epilogue);
  return swb_check_launch("gemv_bf16_kernel");
}
