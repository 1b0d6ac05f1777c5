// Decode linear layers: weight-streaming skinny GEMM for M = 1..16 rows.
//
//   out[m, n] = epilogue( sum_k x[m,k] * W[n,k] )
//
// At decode batch sizes the step is > 95 % weight bytes, so
// this is an HBM-bandwidth kernel.  Design (Blackwell): a persistent grid of
// 2 CTAs per SM; in each CTA one producer lane streams the weight rows of
// its work items into a 6-stage shared-memory ring with 1-D bulk async copies
// (cp.async.bulk -> mbarrier complete_tx, L2 evict-first), so ~192 KB per SM
// are in flight independent of register pressure.  A work item is 4 weight
// rows (small items keep the 148-SM grid balanced at ~7 items per SM for a
// 4096-row matrix); eight consumer warps each take one row's K half, read
// their 2 KB slice of every 16 KB stage with 128-bit shared loads, multiply
// by x (L1-resident, <= 16 rows) in fp32, shuffle-reduce once per item and
// combine halves through smem.  Epilogues: bf16 / fp32 store, fp32 residual
// add (in place), SwiGLU over gate/up rows interleaved in 128-row groups
// (slots 0,1 gate and 2,3 up of the same 2 outputs).
//
// Replaces PerfModel.token_iter_time (reference perf.py:125-132) for the
// linear layers of a token-phase iteration.
#include "common.cuh"

namespace swb {

constexpr int TV_ROWS = 4;                    // weight rows per work item
constexpr int TV_WARPS = 8;                   // consumer warps: 2 per row (K halves)
constexpr int TV_KC = 2048;                   // K elements per stage per row (4 KB)
constexpr int TV_STAGES = 6;
constexpr int TV_ROW_BYTES = TV_KC * 2;
constexpr int TV_STAGE_BYTES = TV_ROWS * TV_ROW_BYTES;  // 16 KB
constexpr int TV_THREADS = (TV_WARPS + 1) * 32;
constexpr int TV_SMEM = TV_STAGES * TV_STAGE_BYTES + 2 * TV_STAGES * 8 + 2 * TV_WARPS * 16 * 4 + 128;

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

// weight row of slot j (0..3) of work item `item`.  Plain: rows 4i..4i+3.
// SwiGLU: outputs 2i, 2i+1 -> gate rows g, g+1 (slots 0,1), up rows g+128,
// g+129 (slots 2,3), with gate/up interleaved in 128-row groups.
__device__ __forceinline__ int item_row(int item, int j, bool swiglu) {
  if (!swiglu) return item * TV_ROWS + j;
  const int o = item * 2 + (j & 1);
  return (o >> 7) * 256 + (o & 127) + (j >= 2 ? 128 : 0);
}

template <int MB>
__global__ void __launch_bounds__(TV_THREADS, 1)
    gemv_bulk_kernel(const __nv_bfloat16* __restrict__ x,
                     const __nv_bfloat16* __restrict__ W, void* out, const float* resid,
                     int M, int N, int K, int epi, int n_items) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TV_STAGES * TV_STAGE_BYTES);
  uint64_t* empty = full + TV_STAGES;
  float* part = reinterpret_cast<float*>(empty + TV_STAGES);  // [2][WARPS][16]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool swiglu = epi == SWB_EPI_SWIGLU;
  const int nk = (K + TV_KC - 1) / TV_KC;

  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < TV_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TV_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == TV_WARPS) {
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

  // ------------------------------ consumers: warp w -> row w&3, K half w>>2
  // The producer above streams static weights before the previous kernel has
  // finished (PDL); consumers read x / write out only after it has.
  pdl_wait();
  const int slot = warp & 3, khalf = warp >> 2;
  int it = 0, parity = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, parity ^= 1) {
    const int row = item_row(item, slot, swiglu);
    const bool valid = row < N;
    float acc[MB];
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[m] = 0.f;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % TV_STAGES;
      mbar_wait(&full[s], (it / TV_STAGES) & 1);
      if (valid) {
        const __nv_bfloat16* wr = reinterpret_cast<const __nv_bfloat16*>(
            smem + s * TV_STAGE_BYTES + slot * TV_ROW_BYTES) + khalf * (TV_KC / 2);
        uint4 wv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) wv[j] = *reinterpret_cast<const uint4*>(wr + j * 256 + lane * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = kc * TV_KC + khalf * (TV_KC / 2) + j * 256 + lane * 8;
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
    // per-warp partial sums -> smem (double-buffered by item parity), then
    // warp 0 combines the two K halves of each row and applies the epilogue
    float* pb = part + parity * TV_WARPS * 16;
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const float v = warp_sum(acc[m]);
      if (lane == 0) pb[warp * 16 + m] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
    if (warp == 0) {
      if (swiglu) {
        // lane = m*2 + o : outputs 2*item + o
        const int m = lane >> 1, o = lane & 1;
        const int nout = N >> 1, oi = item * 2 + o;
        if (m < M && oi < nout) {
          const float g = pb[o * 16 + m] + pb[(o + 4) * 16 + m];
          const float u = pb[(o + 2) * 16 + m] + pb[(o + 6) * 16 + m];
          reinterpret_cast<__nv_bfloat16*>(out)[(size_t)m * nout + oi] =
              __float2bfloat16(g / (1.f + __expf(-g)) * u);
        }
      } else {
        for (int e = lane; e < M * TV_ROWS; e += 32) {
          const int m = e / TV_ROWS, j = e % TV_ROWS;
          const int r = item_row(item, j, false);
          if (r >= N) continue;
          const float v = pb[j * 16 + m] + pb[(j + 4) * 16 + m];
          const size_t idx = (size_t)m * N + r;
          if (epi == SWB_EPI_BF16)
            reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(v);
          else if (epi == SWB_EPI_F32)
            reinterpret_cast<float*>(out)[idx] = v;
          else
            reinterpret_cast<float*>(out)[idx] = resid[idx] + v;
        }
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
  const int grid = min(items, kNumSMs);  // 1 CTA/SM: leaves room for the next kernel
  {
    const cudaError_t le_ = launch(gemv_bulk_kernel<MB>, dim3(grid), dim3(TV_THREADS), TV_SMEM, s,
        x, w, out, r, M, N, K, epi, items);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch gemv_bulk_kernel: %s", cudaGetErrorString(le_));
  }
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
  const int items = (N + TV_ROWS - 1) / TV_ROWS;  // 4 rows (or 2 SwiGLU outputs) per item
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
