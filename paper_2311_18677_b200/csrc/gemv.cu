// Decode linear layers: weight-streaming skinny GEMM for M = 1..16 rows.
//
//   out[m, n] = epilogue( sum_k x[m,k] * W[n,k] )
//
// At decode batch sizes the step is > 95 % weight bytes, so
// this is an HBM-bandwidth kernel.  Design (Blackwell): a persistent grid of
// 2 CTAs per SM; in each CTA one producer lane streams the weight rows of
// its work items into a 6-stage shared-memory ring with 1-D bulk async copies
// (cp.async.bulk -> mbarrier complete_tx, L2 evict-first), so ~192 KB per SM
// are in flight independent of register pressure; eight consumer warps each
// own one of the item's 8 weight rows, read their 2 KB slice of every stage
// with 128-bit shared loads, multiply by x (L1-resident, <= 16 rows) in fp32
// and reduce with warp shuffles once per item.  Epilogues: bf16 / fp32 store,
// fp32 residual add (in place), SwiGLU over gate/up rows interleaved in
// 128-row groups (warps 0-3 gate, 4-7 up of the same 4 outputs).
//
// Replaces PerfModel.token_iter_time (reference perf.py:125-132) for the
// linear layers of a token-phase iteration.
#include "common.cuh"

namespace swb {

constexpr int TV_ROWS = 8;                    // weight rows per item = consumer warps
constexpr int TV_KC = 1024;                   // K elements per stage per row (2 KB)
constexpr int TV_STAGES = 6;
constexpr int TV_ROW_BYTES = TV_KC * 2;
constexpr int TV_STAGE_BYTES = TV_ROWS * TV_ROW_BYTES;  // 16 KB
constexpr int TV_THREADS = (TV_ROWS + 1) * 32;
constexpr int TV_SMEM = TV_STAGES * TV_STAGE_BYTES + 2 * TV_STAGES * 8 + 4 * 16 * 4 + 128;

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// weight row of slot j (0..7) of work item `item`
__device__ __forceinline__ int item_row(int item, int j, bool swiglu) {
  if (!swiglu) return item * TV_ROWS + j;
  const int o = item * 4 + (j & 3);               // output feature
  return (o >> 7) * 256 + (o & 127) + (j >= 4 ? 128 : 0);
}

template <int MB>
__global__ void __launch_bounds__(TV_THREADS, 2)
    gemv_bulk_kernel(const __nv_bfloat16* __restrict__ x,
                     const __nv_bfloat16* __restrict__ W, void* out, const float* resid,
                     int M, int N, int K, int epi, int n_items) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TV_STAGES * TV_STAGE_BYTES);
  uint64_t* empty = full + TV_STAGES;
  float* xchg = reinterpret_cast<float*>(empty + TV_STAGES);  // [4][16] gate/up exchange
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool swiglu = epi == SWB_EPI_SWIGLU;
  const int nk = (K + TV_KC - 1) / TV_KC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TV_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TV_ROWS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == TV_ROWS) {
    // ------------------------------------------------ producer (1 lane)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % TV_STAGES;
          if (it >= TV_STAGES) mbar_wait(&empty[s], ((it / TV_STAGES) - 1) & 1);
          const int k0 = kc * TV_KC;
          const uint32_t bytes = (uint32_t)min(TV_KC, K - k0) * 2;
          uint32_t total = 0;
          for (int j = 0; j < TV_ROWS; ++j)
            if (item_row(item, j, swiglu) < N) total += bytes;
          mbar_arrive_expect_tx(&full[s], total);
          uint8_t* st = smem + s * TV_STAGE_BYTES;
          for (int j = 0; j < TV_ROWS; ++j) {
            const int row = item_row(item, j, swiglu);
            if (row < N)
              bulk_load(st + j * TV_ROW_BYTES, W + (size_t)row * K + k0, bytes, &full[s], pol);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumers (8 warps)
  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int row = item_row(item, warp, swiglu);
    const bool valid = row < N;
    float acc[MB];
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[m] = 0.f;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % TV_STAGES;
      mbar_wait(&full[s], (it / TV_STAGES) & 1);
      if (valid) {
        const __nv_bfloat16* wr =
            reinterpret_cast<const __nv_bfloat16*>(smem + s * TV_STAGE_BYTES + warp * TV_ROW_BYTES);
        uint4 wv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) wv[j] = *reinterpret_cast<const uint4*>(wr + j * 256 + lane * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = kc * TV_KC + j * 256 + lane * 8;
          if (k < K) {
            const float2 w0 = bf2_to_f2(wv[j].x), w1 = bf2_to_f2(wv[j].y),
                         w2 = bf2_to_f2(wv[j].z), w3 = bf2_to_f2(wv[j].w);
#pragma unroll
            for (int m = 0; m < MB; ++m) {
              if (m >= M) break;
              const uint4 xq = *reinterpret_cast<const uint4*>(x + (size_t)m * K + k);
              const float2 x0 = bf2_to_f2(xq.x), x1 = bf2_to_f2(xq.y),
                           x2 = bf2_to_f2(xq.z), x3 = bf2_to_f2(xq.w);
              float a = acc[m];
              a = fmaf(x0.x, w0.x, a); a = fmaf(x0.y, w0.y, a);
              a = fmaf(x1.x, w1.x, a); a = fmaf(x1.y, w1.y, a);
              a = fmaf(x2.x, w2.x, a); a = fmaf(x2.y, w2.y, a);
              a = fmaf(x3.x, w3.x, a); a = fmaf(x3.y, w3.y, a);
              acc[m] = a;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[m] = warp_sum(acc[m]);

    if (swiglu) {
      // warps 4..7 hand their (up) sums to warps 0..3 (gate) of the same output
      asm volatile("bar.sync 1, %0;" ::"n"(TV_ROWS * 32));
      if (warp >= 4 && lane == 0) {
#pragma unroll
        for (int m = 0; m < MB; ++m) xchg[(warp - 4) * 16 + m] = acc[m];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TV_ROWS * 32));
      if (warp < 4) {
        const int o = item * 4 + warp;
        const int nout = N >> 1;
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          if (m >= M) break;
          if (lane == m && o < nout) {
            const float g = acc[m], u = xchg[warp * 16 + m];
            reinterpret_cast<__nv_bfloat16*>(out)[(size_t)m * nout + o] =
                __float2bfloat16(g / (1.f + __expf(-g)) * u);
          }
        }
      }
    } else if (valid) {
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        if (m >= M) break;
        if (lane != m) continue;
        const size_t idx = (size_t)m * N + row;
        if (epi == SWB_EPI_BF16)
          reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(acc[m]);
        else if (epi == SWB_EPI_F32)
          reinterpret_cast<float*>(out)[idx] = acc[m];
        else
          reinterpret_cast<float*>(out)[idx] = resid[idx] + acc[m];
      }
    }
  }
}

template <int MB>
static int launch_gemv(const __nv_bfloat16* x, const __nv_bfloat16* w, void* out,
                       const float* r, int M, int N, int K, int epi, int items,
                       cudaStream_t s) {
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemv_bulk_kernel<MB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, TV_SMEM));
    attr[dev] = true;
  }
  const int grid = min(items, 2 * kNumSMs);
  gemv_bulk_kernel<MB><<<grid, TV_THREADS, TV_SMEM, s>>>(x, w, out, r, M, N, K, epi, items);
  return swb_check_launch("gemv_bulk_kernel");
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
  const int items = (N + TV_ROWS - 1) / TV_ROWS;  // 8 rows (or 4 SwiGLU outputs) per item
  auto xs = reinterpret_cast<const __nv_bfloat16*>(x);
  auto ws = reinterpret_cast<const __nv_bfloat16*>(w);
  auto rs = reinterpret_cast<const float*>(resid);
  cudaStream_t s = (cudaStream_t)stream;
  if (M == 1) return launch_gemv<1>(xs, ws, out, rs, M, N, K, epilogue, items, s);
  if (M <= 2) return launch_gemv<2>(xs, ws, out, rs, M, N, K, epilogue, items, s);
  if (M <= 4) return launch_gemv<4>(xs, ws, out, rs, M, N, K, epilogue, items, s);
  if (M <= 8) return launch_gemv<8>(xs, ws, out, rs, M, N, K, epilogue, items, s);
  return launch_gemv<16>(xs, ws, out, rs, M, N, K, epilogue, items, s);
}
