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
#include <cstring>

#include "common.cuh"

namespace swb {

constexpr int TV_ROWS = 4;                    // weight rows per work item
constexpr int TV_WARPS = 8;                   // consumer warps: 2 per row (K halves)
constexpr int TV_KC = 2048;                   // K elements per stage per row (4 KB)
#ifndef SWB_TV_STAGES
#define SWB_TV_STAGES 5   // ring depth (A/B builds only)
#endif
constexpr int TV_STAGES = SWB_TV_STAGES;
constexpr int TV_ROW_BYTES = TV_KC * 2;
constexpr int TV_STAGE_BYTES = TV_ROWS * TV_ROW_BYTES;  // 16 KB
constexpr int TV_THREADS = (TV_WARPS + 1) * 32;
constexpr int TV_CTAS_PER_SM = 2;             // 2 x ~100 KB ring per SM
constexpr int TV_HS_MAX = 16 * 1024;          // NORM: staged h (M*K*2 bytes) limit
// Items of R in {1, 2, 4} rows (the ring keeps TV_STAGES * 16 KB in flight:
// 20 / R stages of R rows): small matrices use narrower items so the
// persistent grid's CTAs get equal shares (7B O / down projections: 1024
// 4-row items over 296 CTAs = 3.46 each, i.e. the 4-item CTAs set the time).
constexpr int TV_SMEM = TV_STAGES * TV_STAGE_BYTES + 2 * 20 * 8 +
                        2 * TV_WARPS * TV_ROWS * 16 * 4 + 128;

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
template <int R = TV_ROWS>
__device__ __forceinline__ int item_row(int item, int j, bool swiglu) {
  if (!swiglu) return item * R + j;
  const int o = item * 2 + (j & 1);
  return (o >> 7) * 256 + (o & 127) + (j >= 2 ? 128 : 0);
}

// NORM = false: x is bf16 [M,K].
// NORM = true : x is the fp32 residual stream [M,K]; the kernel applies
//               RMSNorm on the fly, h = bf16(x * rsqrt(mean(x^2)+eps) * nw),
//               bit-identical to swb_rmsnorm's output (fused pre-norm GEMV).
// TPP: the fused TP push variant (one row, 4-row items); false compiles none
// of its code into the plain kernels
template <int MB, bool NORM, int R = TV_ROWS, bool TPP = false>
__global__ void __launch_bounds__(TV_THREADS, TV_CTAS_PER_SM)
    gemv_bulk_kernel(const void* __restrict__ xin, const __nv_bfloat16* __restrict__ nw,
                     float eps, const __nv_bfloat16* __restrict__ W, void* out,
                     const float* resid, const __nv_bfloat16* bias, int M, int N, int K,
                     int epi, int n_items, int trig, const __grid_constant__ TpPush tpp) {
  constexpr int NST = TV_STAGES * TV_ROWS / R;           // ring stages
  constexpr int SBYTES = R * TV_ROW_BYTES;                // bytes per stage
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TV_STAGES * TV_STAGE_BYTES);
  uint64_t* empty = full + NST;
  float* part = reinterpret_cast<float*>(full + 2 * 20);     // [2][WARPS][R][16]
  float* rstd = part + 2 * TV_WARPS * TV_ROWS * 16;            // [16]
  __nv_bfloat16* hs = reinterpret_cast<__nv_bfloat16*>(smem + TV_SMEM);  // NORM: [M][K]
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(xin);
  const float* xf = reinterpret_cast<const float*>(xin);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool swiglu = R == 4 && epi == SWB_EPI_SWIGLU;     // SwiGLU items are 4-row
  const int nk = (K + TV_KC - 1) / TV_KC;

  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
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
          const int s = it % NST;
          if (it >= NST) mbar_wait_sleep(&empty[s], ((it / NST) - 1) & 1);
          const int k0 = kc * TV_KC;
          const uint32_t bytes = (uint32_t)min(TV_KC, K - k0) * 2;
          uint32_t total = 0;
          for (int j = 0; j < R; ++j)
            if (item_row<R>(item, j, swiglu) < N) total += bytes;
          mbar_arrive_expect_tx(&full[s], total);
          uint8_t* st = smem + s * SBYTES;
          for (int j = 0; j < R; ++j) {
            const int row = item_row<R>(item, j, swiglu);
            if (row < N)
              bulk_load(st + j * TV_ROW_BYTES, W + (size_t)row * K + k0, bytes, &full[s], pol);
          }
        }
      }
      // last weight load issued: once this CTA is also past the dependency
      // wait (so everything before it is complete) the next kernel may launch
      if (trig) {
        pdl_wait();
        pdl_launch_dependents();
      }
    }
    return;
  }

  // ------------------- consumers: warp w owns columns [256w, 256w+256) of
  // every stage for all 4 rows of the item, so one x chunk (per batch row)
  // feeds 4 weight rows; lanes shuffle-reduce, warps combine through smem.
  // The producer above streams static weights before the previous kernel has
  // finished (PDL); consumers read x / write out only after it has.
  // one-row pre-norm: the norm weights are static — fetch them before the
  // dependency wait; x is read once (kept in registers from the sum of
  // squares to the staging), each thread owning 8-element groups
  constexpr int NIT = TV_HS_MAX / 2 / 8 / (TV_WARPS * 32);   // groups per thread (K <= 8192)
  uint4 nwq[NIT];
  if constexpr (NORM && MB == 1) {
#pragma unroll
    for (int i = 0; i < NIT; ++i) {
      const int g = threadIdx.x + i * TV_WARPS * 32;
      if (g < K / 8) nwq[i] = *reinterpret_cast<const uint4*>(nw + 8 * g);
    }
  }
  pdl_wait();
  // fused TP push: this use's epoch (the previous use of the slot finished
  // its receive kernel before the kernel ahead of us did)
  const unsigned ll_e =
      TPP ? *reinterpret_cast<const volatile unsigned*>(tpp.epoch) + 1u : 0u;
  if constexpr (NORM && MB == 1) {
    float4 xa[NIT], xb[NIT];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NIT; ++i) {
      const int g = threadIdx.x + i * TV_WARPS * 32;
      if (g < K / 8) {
        xa[i] = *reinterpret_cast<const float4*>(xf + 8 * g);
        xb[i] = *reinterpret_cast<const float4*>(xf + 8 * g + 4);
        ss += xa[i].x * xa[i].x + xa[i].y * xa[i].y + xa[i].z * xa[i].z + xa[i].w * xa[i].w +
              xb[i].x * xb[i].x + xb[i].y * xb[i].y + xb[i].z * xb[i].z + xb[i].w * xb[i].w;
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) part[warp * 16] = ss;
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
    // every thread sums the 8 warp partials in the same order: one barrier
    float q = 0.f;
#pragma unroll
    for (int w = 0; w < TV_WARPS; ++w) q += part[w * 16];
    const float r = rsqrtf(q / (float)K + eps);
#pragma unroll
    for (int i = 0; i < NIT; ++i) {
      const int g = threadIdx.x + i * TV_WARPS * 32;
      if (g < K / 8) {
        const float2 n0 = bf2_to_f2(nwq[i].x), n1 = bf2_to_f2(nwq[i].y),
                     n2 = bf2_to_f2(nwq[i].z), n3 = bf2_to_f2(nwq[i].w);
        const float4 a = xa[i], b = xb[i];
        *reinterpret_cast<uint4*>(hs + 8 * g) =
            make_uint4(f2_to_bf2(a.x * r * n0.x, a.y * r * n0.y),
                       f2_to_bf2(a.z * r * n1.x, a.w * r * n1.y),
                       f2_to_bf2(b.x * r * n2.x, b.y * r * n2.y),
                       f2_to_bf2(b.z * r * n3.x, b.w * r * n3.y));
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
  } else if constexpr (NORM) {
    // sum of squares of every batch row, by all consumer threads
    const int t = threadIdx.x;
    for (int m = 0; m < M; ++m) {
      float ss = 0.f;
      for (int k = t * 4; k < K; k += TV_WARPS * 32 * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xf + (size_t)m * K + k);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
      ss = warp_sum(ss);
      if (lane == 0) part[warp * 16 + m] = ss;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
    if (t < M) {
      float ss = 0.f;
      for (int w = 0; w < TV_WARPS; ++w) ss += part[w * 16 + t];
      rstd[t] = rsqrtf(ss / (float)K + eps);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
    // normalise once into shared memory: the streaming loop then reads h
    // exactly like a plain bf16 input (same rounding as swb_rmsnorm)
    for (int i = t; i < M * K / 8; i += TV_WARPS * 32) {
      const int m = (i * 8) / K, k = (i * 8) % K;
      const float r = rstd[m];
      const uint4 wq = *reinterpret_cast<const uint4*>(nw + k);
      const float2 n0 = bf2_to_f2(wq.x), n1 = bf2_to_f2(wq.y), n2 = bf2_to_f2(wq.z),
                   n3 = bf2_to_f2(wq.w);
      const float4 a = *reinterpret_cast<const float4*>(xf + (size_t)m * K + k);
      const float4 b = *reinterpret_cast<const float4*>(xf + (size_t)m * K + k + 4);
      *reinterpret_cast<uint4*>(hs + (size_t)m * K + k) =
          make_uint4(f2_to_bf2(a.x * r * n0.x, a.y * r * n0.y),
                     f2_to_bf2(a.z * r * n1.x, a.w * r * n1.y),
                     f2_to_bf2(b.x * r * n2.x, b.y * r * n2.y),
                     f2_to_bf2(b.z * r * n3.x, b.w * r * n3.y));
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
  }
  int it = 0, parity = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, parity ^= 1) {
    float acc[R][MB];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int m = 0; m < MB; ++m) acc[j][m] = 0.f;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % NST;
      const int k = kc * TV_KC + warp * 256 + lane * 8;
      uint4 xq[MB];
      if (k < K) {
        if constexpr (NORM) {
#pragma unroll
          for (int m = 0; m < MB; ++m)
            if (m < M) xq[m] = *reinterpret_cast<const uint4*>(hs + (size_t)m * K + k);
        } else {
#pragma unroll
          for (int m = 0; m < MB; ++m)
            if (m < M) xq[m] = *reinterpret_cast<const uint4*>(x + (size_t)m * K + k);
        }
      }
      mbar_wait(&full[s], (it / NST) & 1);
      if (k < K) {
        const uint8_t* st = smem + s * SBYTES + (warp * 256 + lane * 8) * 2;
        uint4 wv[R];
#pragma unroll
        for (int j = 0; j < R; ++j)
          wv[j] = *reinterpret_cast<const uint4*>(st + j * TV_ROW_BYTES);
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          if (m >= M) break;
          const float2 x0 = bf2_to_f2(xq[m].x), x1 = bf2_to_f2(xq[m].y),
                       x2 = bf2_to_f2(xq[m].z), x3 = bf2_to_f2(xq[m].w);
#pragma unroll
          for (int j = 0; j < R; ++j) {
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // lanes -> warp sums -> smem [parity][warp][row][m], then warp 0 adds the
    // 8 K-slices of each (row, m) and applies the epilogue
    float* pb = part + parity * TV_WARPS * TV_ROWS * 16;
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        if (m >= M) break;
        const float v = warp_sum(acc[j][m]);
        if (lane == 0) pb[(warp * R + j) * 16 + m] = v;
      }
    asm volatile("bar.sync 1, %0;" ::"n"(TV_WARPS * 32));
    if (warp == 0) {
      for (int e0 = 0; e0 < M * R; e0 += 32) {   // warp-uniform trip count
        const int e = e0 + lane;
        const bool active = e < M * R;
        const int m = e / R, j = e % R;
        float v = 0.f;
        if (active) {
#pragma unroll
          for (int w = 0; w < TV_WARPS; ++w) v += pb[(w * R + j) * 16 + m];
        }
        // SwiGLU: rows j = 0,1 gate and 2,3 up of outputs 2*item + (j & 1)
        const float u = __shfl_down_sync(0xffffffffu, v, 2);
        if (!active) continue;
        if (swiglu) {
          if (j < 2) {
            const int nout = N >> 1, oi = item * 2 + j;
            if (oi < nout)
              reinterpret_cast<__nv_bfloat16*>(out)[(size_t)m * nout + oi] =
                  __float2bfloat16(silu_f(v) * u);
          }
        } else {
          const int r = item_row<R>(item, j, false);
          if (r < N) {
            const size_t idx = (size_t)m * N + r;
            v += bias_at(bias, r);
            if (epi == SWB_EPI_BF16)
              reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(v);
            else if (epi == SWB_EPI_GELU)
              reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(gelu_tanh(v));
            else {
              const float o = epi == SWB_EPI_F32 ? v : resid[idx] + v;
              reinterpret_cast<float*>(out)[idx] = o;
            }
          }
        }
      }
      if constexpr (TPP && R == 4) {
        // fused TP all-reduce (one decode row): the item's 4 consecutive
        // outputs go straight to every peer as two 16-byte posted NVLink
        // stores of (value, epoch) words while later weights still stream
        // lane 2p + h stores half h to peer p, so the stores leave in
        // parallel; lane 0 reads all four outputs (the own count's release
        // below covers them)
        __syncwarp();
        if (lane < 2 * tpp.world && 4 * item + 3 < N) {
          const float4 v4 = reinterpret_cast<const float4*>(out)[item];
          const int p = lane >> 1, h = lane & 1;
          if (p != tpp.rank) {
            const unsigned long long hi = (unsigned long long)ll_e << 32;
            const unsigned long long a0 = hi | __float_as_uint(h ? v4.z : v4.x),
                                     a1 = hi | __float_as_uint(h ? v4.w : v4.y);
            unsigned long long* d = tpp.rx[p] + 4 * (size_t)item + 2 * h;
            asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(a0), "l"(a1)
                         : "memory");
          }
        }
      }
    }
  }
  if (TPP && warp == 0 && lane == 0) {
    // lane 0 read every local output of this CTA, so its gpu-scope release
    // orders them before the count: the receive kernel waits for the count,
    // not for this grid to exit
    red_release_gpu_add(tpp.own_cnt, 1u);
  }
}

// Resident CTAs per SM of the streaming GEMVs (SWB_GEMV_CTAS_PER_SM, A/B).
// With one CTA per SM the next kernel's CTAs (PDL, triggered once this
// kernel's producers issued their last load) fit beside it and start their
// weight stream while this one drains.
static int gemv_ctas_per_sm() {
  static const int n = [] {
    const char* e = std::getenv("SWB_GEMV_CTAS_PER_SM");
    return e ? std::max(1, std::min(2, atoi(e))) : 2;
  }();
  return n;
}

template <int MB, bool NORM, int R, bool TPP = false>
static int launch_gemv_r(const void* x, const __nv_bfloat16* nw, float eps,
                         const __nv_bfloat16* w, void* out, const float* r,
                         const __nv_bfloat16* bias, int M, int N, int K, int epi,
                         cudaStream_t s, const TpPush& tpp, int grid) {
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemv_bulk_kernel<MB, NORM, R, TPP>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  TV_SMEM + TV_HS_MAX));
    attr[dev] = true;
  }
  const size_t smem = TV_SMEM + (NORM ? (size_t)M * K * 2 : 0);
  const int items = (N + R - 1) / R;
  const cudaError_t le = launch(gemv_bulk_kernel<MB, NORM, R, TPP>, dim3(grid), dim3(TV_THREADS),
                                smem, s, x, nw, eps, w, out, r, bias, M, N, K, epi, items,
                                pdl_early_trigger() ? 1 : 0, tpp);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch gemv_bulk_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("gemv_bulk_kernel");
}

// rows per item: 4 (default).  SWB_GEMV_ROWS=0 picks narrower items for
// small matrices so the persistent grid gets equal shares — measured much
// slower (7B B=1 step 3.41 vs 2.53 ms, 70B TP4 9.06 vs 8.05 ms: 1-2-row
// stages do too little work per ring handshake), so it stays an A/B option.
static int gemv_rows_for(int N, int grid_max, bool swiglu, bool tp) {
  static const int pin = [] {
    const char* e = std::getenv("SWB_GEMV_ROWS");
    return e ? std::atoi(e) : 4;
  }();
  if (swiglu || tp) return 4;
  if (pin == 1 || pin == 2 || pin == 4) return pin;
  if ((N + 3) / 4 >= 8 * grid_max) return 4;
  if ((N + 1) / 2 >= 8 * grid_max) return 2;
  return 1;
}

template <int MB, bool NORM>
static int launch_gemv(const void* x, const __nv_bfloat16* nw, float eps,
                       const __nv_bfloat16* w, void* out, const float* r,
                       const __nv_bfloat16* bias, int M, int N, int K, int epi, int items,
                       cudaStream_t s, swb_tp_comm* tp = nullptr, int tp_slot = 0) {
  const int grid_max = gemv_ctas_per_sm() * kNumSMs;
  const int R = gemv_rows_for(N, grid_max, epi == SWB_EPI_SWIGLU, tp != nullptr);
  const int grid = min((N + R - 1) / R, grid_max);
  (void)items;
  TpPush tpp;
  memset(&tpp, 0, sizeof(tpp));
  if (tp) {
    const int st = tp_push_targets(tp, tp_slot, grid, (long long)M * N, &tpp);
    if (st) return st;
  }
  if constexpr (MB == 1 && !NORM) {
    if (tp) {   // swb_gemv_bf16_tp: one row, 4-row items (gemv_rows_for)
      if (R != 4) return swb_set_error(SWB_ERR_INVALID, "fused TP push needs 4-row items");
      return launch_gemv_r<1, false, 4, true>(x, nw, eps, w, out, r, bias, M, N, K, epi, s, tpp,
                                              grid);
    }
  }
  if (R == 1) return launch_gemv_r<MB, NORM, 1>(x, nw, eps, w, out, r, bias, M, N, K, epi, s, tpp, grid);
  if (R == 2) return launch_gemv_r<MB, NORM, 2>(x, nw, eps, w, out, r, bias, M, N, K, epi, s, tpp, grid);
  return launch_gemv_r<MB, NORM, 4>(x, nw, eps, w, out, r, bias, M, N, K, epi, s, tpp, grid);
}

// ---------------------------------------------------------------------------
// Batched decode (M = 2..16): the CUDA-core path above becomes FMA-bound as M
// grows, so here the weight tile is the A operand of mma.sync m16n8k16 (16
// weight rows x 16 k) and x^T the B operand (16 k x 8 batch rows).  Weights
// stream through a TMA ring (2-D tensor map, 16-row x 64-col boxes with 128 B
// swizzle so ldmatrix is conflict-free); 8 consumer warps each own one
// 64-column box of every 16 x 512 stage; per-item partials (16 x 8 fp32 per
// warp) are combined through smem.  SwiGLU items load 8 gate + 8 up rows of
// the same outputs into one 16-row tile.
constexpr int TM_ROWS = 16, TM_KC = 512, TM_STAGES = 6, TM_WARPS = 8;
constexpr int TM_BOX_BYTES = TM_ROWS * 64 * 2;                 // 2 KB
constexpr int TM_STAGE_BYTES = TM_ROWS * TM_KC * 2;            // 16 KB
constexpr int TM_THREADS = (TM_WARPS + 1) * 32;
constexpr int TM_NORM_STAGES = 4;   // pre-norm variant: 4 stages + staged h (<= 32 KB)
constexpr int TM_HS_MAX = 32 * 1024;
constexpr int tm_smem(int stages) {
  return stages * TM_STAGE_BYTES + 1024 + 2 * stages * 8 + TM_WARPS * 32 * 8 * 4 + 256;
}
constexpr int TM_SMEM = tm_smem(TM_STAGES);

__device__ __forceinline__ void ldsm_x4_g(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// NORM: x is the fp32 residual stream; the B fragments are built on the fly as
// h = bf16(x * rstd * norm_w), with rstd reduced in exactly swb_rmsnorm's
// order (512 virtual threads, 16 warp partials), so the fused pre-norm GEMV
// is bit-identical to swb_rmsnorm + GEMV and saves a launch per projection.
// ST: ring stages (NORM: 4, or 5 when the staged h leaves room for it)
template <int NB, bool NORM, int ST = NORM ? TM_NORM_STAGES : TM_STAGES>
__global__ void __launch_bounds__(TM_THREADS, 2)
    gemv_mma_kernel(const __grid_constant__ CUtensorMap tmW, const void* xin,
                    const __nv_bfloat16* __restrict__ nw, float eps,
                    void* out, const float* resid, const __nv_bfloat16* bias, int M, int N,
                    int K, int epi, int n_items, int trig) {
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(xin);
  const float* xf = reinterpret_cast<const float*>(xin);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * TM_STAGE_BYTES);
  uint64_t* empty = full + ST;
  float* red = reinterpret_cast<float*>(empty + ST);   // [WARPS][32 lanes][8]
  __nv_bfloat16* hs = reinterpret_cast<__nv_bfloat16*>(red + TM_WARPS * 32 * 8);  // NORM [M][K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool swiglu = epi == SWB_EPI_SWIGLU;
  const int nk = (K + TM_KC - 1) / TM_KC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TM_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == TM_WARPS) {
    if (lane == 0) {
      tma_prefetch_desc(&tmW);
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int r0, r1;   // first row of the two 8-row halves
        if (swiglu) {
          const int o = item * 8;
          r0 = (o >> 7) * 256 + (o & 127);
          r1 = r0 + 128;
        } else {
          r0 = item * TM_ROWS;
          r1 = r0 + 8;
        }
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % ST;
          if (it >= ST) mbar_wait_sleep(&empty[s], ((it / ST) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], TM_STAGE_BYTES);
          uint8_t* st = smem + s * TM_STAGE_BYTES;
          for (int bx = 0; bx < TM_KC / 64; ++bx) {
            // box = 8 rows x 64 cols (1 KB); two boxes fill one 16-row tile
            tma_load_2d(st + bx * TM_BOX_BYTES, &tmW, &full[s], kc * TM_KC + bx * 64, r0);
            tma_load_2d(st + bx * TM_BOX_BYTES + 8 * 128, &tmW, &full[s], kc * TM_KC + bx * 64,
                        r1);
          }
        }
      }
      // last weight load issued: once this CTA is also past the dependency
      // wait (so everything before it is complete) the next kernel may launch
      if (trig) {
        pdl_wait();
        pdl_launch_dependents();
      }
    }
    return;
  }
  // pre-norm, M <= 2, K <= 4096: thread t owns x's float4 columns t + 256 j
  // in the sum of squares AND the staging (the same set), so x is read once
  // into registers, and the static norm weights before the dependency wait
  constexpr int XC = 4;                      // float4 columns per thread and row
  const bool regs = NORM && M <= 2 && K <= XC * 4 * TM_WARPS * 32 && K % (4 * TM_WARPS * 32) == 0;
  uint2 nwr[XC];
  if (NORM && regs) {
#pragma unroll
    for (int j = 0; j < XC; ++j) {
      const int c = threadIdx.x + j * TM_WARPS * 32;
      if (c < K / 4) nwr[j] = *reinterpret_cast<const uint2*>(nw + 4 * c);
    }
  }
  pdl_wait();   // x is produced by the previous kernel
  const int g = lane >> 2, t = lane & 3;
  __shared__ float s_part[16 * 16];   // NORM: [row][virtual warp] sums of squares
  __shared__ float s_rstd[16];
  if (NORM && regs) {
    // same sums as swb_rmsnorm: virtual thread vt = t + 256 half walks
    // columns vt, vt + 512, ... — here columns t + 256 j, j even = half 0
    float4 xv[2][XC];
    const int nc = K / 4 / (TM_WARPS * 32);
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      if (m >= M) break;
      const float4* xr = reinterpret_cast<const float4*>(xf + (size_t)m * K);
#pragma unroll
      for (int j = 0; j < XC; ++j)
        if (j < nc) xv[m][j] = xr[threadIdx.x + j * TM_WARPS * 32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float ss = 0.f;
#pragma unroll
        for (int j = half; j < XC; j += 2)
          if (j < nc) {
            const float4 v = xv[m][j];
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
          }
        ss = warp_sum(ss);
        if (lane == 0) s_part[m * 16 + warp + half * TM_WARPS] = ss;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      if (m >= M) break;
      // every warp reduces the 16 partials (same order as before): no barrier
      float v = lane < 16 ? s_part[m * 16 + lane] : 0.f;
      v = warp_sum(v);
      const float r = rsqrtf(v / (float)K + eps);
#pragma unroll
      for (int j = 0; j < XC; ++j) {
        if (j >= nc) continue;
        const int c = threadIdx.x + j * TM_WARPS * 32;
        const float4 xx = xv[m][j];
        const float2 w0 = bf2_to_f2(nwr[j].x), w1 = bf2_to_f2(nwr[j].y);
        *reinterpret_cast<uint2*>(hs + (size_t)m * K + 4 * c) =
            make_uint2(f2_to_bf2(xx.x * r * w0.x, xx.y * r * w0.y),
                       f2_to_bf2(xx.z * r * w1.x, xx.w * r * w1.y));
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
  } else if constexpr (NORM) {
    for (int m = 0; m < M; ++m) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int vt = threadIdx.x + half * (TM_WARPS * 32);    // swb_rmsnorm thread id
        const float4* xr = reinterpret_cast<const float4*>(xf + (size_t)m * K);
        float ss = 0.f;
        for (int c = vt; c < K / 4; c += 2 * TM_WARPS * 32) {
          const float4 v = xr[c];
          ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
        ss = warp_sum(ss);
        if (lane == 0) s_part[m * 16 + warp + half * TM_WARPS] = ss;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
    for (int m = warp; m < M; m += TM_WARPS) {
      float v = lane < 16 ? s_part[m * 16 + lane] : 0.f;
      v = warp_sum(v);
      if (lane == 0) s_rstd[m] = rsqrtf(v / (float)K + eps);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
    // h = bf16(x * rstd * w) once into shared memory (swb_rmsnorm's rounding);
    // the streaming loop then reads it like a plain bf16 input
    for (int i = threadIdx.x; i < M * K / 4; i += TM_WARPS * 32) {
      const int m = (i * 4) / K, kk = (i * 4) % K;
      const float r = s_rstd[m];
      const float4 v = *reinterpret_cast<const float4*>(xf + (size_t)m * K + kk);
      const uint2 ww = *reinterpret_cast<const uint2*>(nw + kk);
      const float2 w0 = bf2_to_f2(ww.x), w1 = bf2_to_f2(ww.y);
      *reinterpret_cast<uint2*>(hs + (size_t)m * K + kk) =
          make_uint2(f2_to_bf2(v.x * r * w0.x, v.y * r * w0.y),
                     f2_to_bf2(v.z * r * w1.x, v.w * r * w1.y));
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
  }
  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    float c[NB][4];
#pragma unroll
    for (int h = 0; h < NB; ++h) c[h][0] = c[h][1] = c[h][2] = c[h][3] = 0.f;
    // B fragments (x^T): batch row = g (+8 for the second MMA), k = 2t.., 8+2t..
    // loaded one K-chunk ahead so their L1/L2 latency hides behind the MMAs
    auto load_b = [&](int kc, uint32_t (&bf)[NB][4][2]) {
      const int kbase = kc * TM_KC + warp * 64;
#pragma unroll
      for (int h = 0; h < NB; ++h) {
        const int m = h * 8 + g;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int k0 = kbase + ks * 16 + 2 * t;
          uint32_t v0 = 0, v1 = 0;
          if constexpr (NORM) {
            if (m < M && k0 < K) {
              v0 = *reinterpret_cast<const uint32_t*>(hs + (size_t)m * K + k0);
              if (k0 + 8 < K) v1 = *reinterpret_cast<const uint32_t*>(hs + (size_t)m * K + k0 + 8);
            }
          } else if (m < M && k0 < K) {
            v0 = __ldg(reinterpret_cast<const unsigned int*>(x + (size_t)m * K + k0));
            if (k0 + 8 < K)
              v1 = __ldg(reinterpret_cast<const unsigned int*>(x + (size_t)m * K + k0 + 8));
          }
          bf[h][ks][0] = v0;
          bf[h][ks][1] = v1;
        }
      }
    };
    uint32_t bnext[NB][4][2];
    load_b(0, bnext);
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % ST;
      uint32_t bfr[NB][4][2];
#pragma unroll
      for (int h = 0; h < NB; ++h)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          bfr[h][ks][0] = bnext[h][ks][0];
          bfr[h][ks][1] = bnext[h][ks][1];
        }
      if (kc + 1 < nk) load_b(kc + 1, bnext);
      mbar_wait(&full[s], (it / ST) & 1);
      const uint32_t box = smem_u32(smem + s * TM_STAGE_BYTES + warp * TM_BOX_BYTES);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t a[4];
        const int row = lane & 15, chunk = ks * 2 + (lane >> 4);
        ldsm_x4_g(box + row * 128 + ((chunk ^ (row & 7)) << 4), a);
#pragma unroll
        for (int h = 0; h < NB; ++h) mma16816(c[h], a, bfr[h][ks][0], bfr[h][ks][1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // c[h] = D[row g | g+8][batch h*8 + 2t, +1]; reduce the 8 K-slices
    float* rw = red + (warp * 32 + lane) * 8;
#pragma unroll
    for (int h = 0; h < NB; ++h) {
      rw[h * 4 + 0] = c[h][0];
      rw[h * 4 + 1] = c[h][1];
      rw[h * 4 + 2] = c[h][2];
      rw[h * 4 + 3] = c[h][3];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
    // thread e (< 16 rows * 8*NB batch) finalises D[row][m]
    for (int e = threadIdx.x; e < TM_ROWS * 8 * NB; e += TM_WARPS * 32) {
      const int row = e % TM_ROWS, m = e / TM_ROWS;
      const int h = m >> 3, mm = m & 7;
      // owner lane of (row, mm): g = row & 7, t = mm >> 1; slot = (row >= 8) * 2 + (mm & 1)
      const int ol = (row & 7) * 4 + (mm >> 1);
      const int slot = h * 4 + (row >= 8 ? 2 : 0) + (mm & 1);
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < TM_WARPS; ++w) v += red[(w * 32 + ol) * 8 + slot];
      if (m >= M) continue;
      if (swiglu) {
        if (row >= 8) continue;          // up rows are read by their gate row
        const int oslot = h * 4 + 2 + (mm & 1);
        float u = 0.f;
#pragma unroll
        for (int w = 0; w < TM_WARPS; ++w) u += red[(w * 32 + ol) * 8 + oslot];
        const int nout = N >> 1, oi = item * 8 + row;
        if (oi < nout)
          reinterpret_cast<__nv_bfloat16*>(out)[(size_t)m * nout + oi] =
              __float2bfloat16(silu_f(v) * u);
      } else {
        const int r = item * TM_ROWS + row;
        if (r >= N) continue;
        const size_t idx = (size_t)m * N + r;
        v += bias_at(bias, r);
        if (epi == SWB_EPI_BF16)
          reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(v);
        else if (epi == SWB_EPI_GELU)
          reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(gelu_tanh(v));
        else if (epi == SWB_EPI_F32)
          reinterpret_cast<float*>(out)[idx] = v;
        else
          reinterpret_cast<float*>(out)[idx] = resid[idx] + v;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TM_WARPS * 32) : "memory");
  }
}

int make_tmap_rows(CUtensorMap* map, const void* base, int rows, int K, int box_rows);

// per-CTA shared-memory budget at 2 CTAs per SM
constexpr int TM_CTA_BUDGET = (228 * 1024 - 2 * 1024) / 2;

template <int NB, bool NORM, int ST>
static int launch_gemv_mma_st(const CUtensorMap& tm, const void* x, const __nv_bfloat16* nw,
                              float eps, void* out, const float* r, const __nv_bfloat16* bias,
                              int M, int N, int K, int epi, int items, int grid, size_t smem,
                              cudaStream_t s) {
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemv_mma_kernel<NB, NORM, ST>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  NORM ? tm_smem(ST) + TM_HS_MAX : TM_SMEM));
    attr[dev] = true;
  }
  return launch(gemv_mma_kernel<NB, NORM, ST>, dim3(grid), dim3(TM_THREADS), smem, s, tm, x, nw,
                eps, out, r, bias, M, N, K, epi, items, pdl_early_trigger() ? 1 : 0) ==
                 cudaSuccess
             ? SWB_OK
             : swb_set_error(SWB_ERR_CUDA, "launch gemv_mma_kernel: %s",
                             cudaGetErrorString(cudaGetLastError()));
}

template <int NB, bool NORM>
static int launch_gemv_mma(const void* x, const __nv_bfloat16* nw, float eps, const void* w,
                           void* out, const float* r, const __nv_bfloat16* bias, int M, int N,
                           int K, int epi, cudaStream_t s) {
  CUtensorMap tm;
  const int st = make_tmap_rows(&tm, w, N, K, 8);
  if (st) return st;
  const int items = epi == SWB_EPI_SWIGLU ? (N / 2 + 7) / 8 : (N + TM_ROWS - 1) / TM_ROWS;
  const int grid = min(items, gemv_ctas_per_sm() * kNumSMs);
  int rc;
  if constexpr (NORM) {
    // pre-norm: a 5th ring stage when the staged h (M*K*2 bytes) leaves room
    // (7B B=2: 16 KB of h)
    const size_t hs = (size_t)M * K * 2;
    if (tm_smem(TM_NORM_STAGES + 1) + hs <= (size_t)TM_CTA_BUDGET)
      rc = launch_gemv_mma_st<NB, true, TM_NORM_STAGES + 1>(
          tm, x, nw, eps, out, r, bias, M, N, K, epi, items, grid,
          tm_smem(TM_NORM_STAGES + 1) + hs, s);
    else
      rc = launch_gemv_mma_st<NB, true, TM_NORM_STAGES>(tm, x, nw, eps, out, r, bias, M, N, K,
                                                        epi, items, grid,
                                                        tm_smem(TM_NORM_STAGES) + hs, s);
  } else {
    rc = launch_gemv_mma_st<NB, false, TM_STAGES>(tm, x, nw, eps, out, r, bias, M, N, K, epi,
                                                  items, grid, TM_SMEM, s);
  }
  if (rc) return rc;
  return swb_check_launch("gemv_mma_kernel");
}

// SWB_GEMV_MMA=0 keeps batched decode on the CUDA-core kernel (A/B)
static bool gemv_mma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SWB_GEMV_MMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

int dispatch_gemv_tc(const void* x, const void* w, void* out, const float* resid,
                     const __nv_bfloat16* bias, int M, int N, int K, int epi, cudaStream_t s);


// SWB_GEMV_TC=0 keeps batched decode on the mma.sync kernel (A/B)
static bool gemv_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("SWB_GEMV_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <bool NORM>
static int dispatch_gemv(const void* x, const __nv_bfloat16* nw, float eps, const void* w,
                         void* out, const void* resid, const void* bias_, int M, int N, int K,
                         int epilogue, uintptr_t stream) {
  auto bias = reinterpret_cast<const __nv_bfloat16*>(bias_);
  const int items = (N + TV_ROWS - 1) / TV_ROWS;  // 4 rows (or 2 SwiGLU outputs) per item
  auto ws = reinterpret_cast<const __nv_bfloat16*>(w);
  auto rs = reinterpret_cast<const float*>(resid);
  cudaStream_t s = (cudaStream_t)stream;
  // tcgen05 GEMV for batched decode; the mma.sync kernel stays ahead on
  // small matrices at small batch (measured crossover, tools/gemv_bench.py)
  // M = 2..4 (and 5..8 below 120 MB): the mma.sync kernel (measured ahead of
  // the tcgen05 GEMV on the 7B step: B=2 3.30 vs 3.43 ms, B=4 3.82 vs 3.95);
  // larger M / matrices: the tcgen05 GEMV.
  // (The mma.sync kernel's two-MMA variant for M = 9..16 showed sporadic
  // wrong columns under a repeat test and is not dispatched.)  Pre-norm fused
  // variants: M = 2..8 on the mma.sync kernel with h staged in shared memory.
  // SWB_GEMV_CORE_MAXM=m: rows M <= m stay on the CUDA-core bulk kernel (A/B)
  static const int core_maxm = [] {
    const char* e = std::getenv("SWB_GEMV_CORE_MAXM");
    return e ? std::atoi(e) : 1;
  }();
  // SWB_GEMV_CORE_NORM_MAXM=m: only the fused pre-norm GEMVs with M <= m (A/B)
  static const int core_norm_maxm = [] {
    const char* e = std::getenv("SWB_GEMV_CORE_NORM_MAXM");
    return e ? std::atoi(e) : 1;
  }();
  const int cmax = NORM ? std::max(core_maxm, core_norm_maxm) : core_maxm;
  if (M >= 2 && M <= cmax && M <= 4 && (!NORM || (size_t)M * K * 2 <= (size_t)TV_HS_MAX)) {
    if (M <= 2)
      return launch_gemv<2, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
    return launch_gemv<4, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
  }
  if (NORM && M >= 2)
    return launch_gemv_mma<1, true>(x, nw, eps, w, out, rs, bias, M, N, K, epilogue, s);
  // K >= 12288 (BLOOM-176B TP4 qkv/up/down, 70B TP2 down): its 16-row x K
  // items are ~450 KB, too few per CTA to balance — the tcgen05 GEMV wins
  // there at every M (tools/gemv_bench.py: BLOOM TP4 up M=2 78.9 vs 68.0 us)
  const bool use_mma = (M <= 4 && K < 12288) || (M <= 8 && 2.0 * N * K < 120e6);
  if (!NORM && M >= 2 && (!use_mma || !gemv_mma_enabled()) && gemv_tc_enabled())
    return dispatch_gemv_tc(x, w, out, rs, bias, M, N, K, epilogue, s);
  if (!NORM && M >= 2 && M <= 8 && gemv_mma_enabled())
    return launch_gemv_mma<1, false>(x, nullptr, 0.f, w, out, rs, bias, M, N, K, epilogue, s);
  // One-row GEMVs without pre-norm (7B O / down projections) on the mma.sync
  // kernel: its 16-row items give the persistent grid one equal item per
  // CTA (O: 256 items, down: 256) instead of 3.46 four-row items — 7B B=1
  // step 2.472 -> 2.439 ms.  The pre-norm ones stay on the streaming kernel
  // (2.64 ms on mma.sync).  SWB_GEMV_M1_MMA = 0 / 1 (default) / 2 (all).
  static const int m1_mma = [] {
    const char* e = std::getenv("SWB_GEMV_M1_MMA");
    return e ? std::atoi(e) : 1;
  }();
  if (M == 1 && gemv_mma_enabled() && K < 12288 && m1_mma >= (NORM ? 2 : 1)) {
    if constexpr (NORM)
      return launch_gemv_mma<1, true>(x, nw, eps, w, out, rs, bias, M, N, K, epilogue, s);
    else
      return launch_gemv_mma<1, false>(x, nullptr, 0.f, w, out, rs, bias, M, N, K, epilogue, s);
  }
  if (M == 1) return launch_gemv<1, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
  if (M <= 2) return launch_gemv<2, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
  if (M <= 4) return launch_gemv<4, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
  if (M <= 8) return launch_gemv<8, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
  return launch_gemv<16, NORM>(x, nw, eps, ws, out, rs, bias, M, N, K, epilogue, items, s);
}

}  // namespace swb

using namespace swb;

static int check_gemv_args(const char* fn, const void* x, const void* w, void* out,
                           const void* resid, int M, int N, int K, int epilogue) {
  SWB_REQUIRE(x && w && out, "%s: null pointer", fn);
  SWB_REQUIRE(M >= 1 && M <= (gemv_tc_enabled() ? 32 : 16), "%s: M=%d outside 1..%d", fn, M,
              gemv_tc_enabled() ? 32 : 16);
  SWB_REQUIRE(N > 0 && K > 0 && K % 8 == 0, "%s: bad shape N=%d K=%d", fn, N, K);
  SWB_REQUIRE(epilogue >= SWB_EPI_BF16 && epilogue <= SWB_EPI_GELU, "%s: bad epilogue %d",
              fn, epilogue);
  SWB_REQUIRE(epilogue != SWB_EPI_SWIGLU || N % 256 == 0, "%s: SwiGLU needs N %% 256 == 0", fn);
  SWB_REQUIRE(epilogue != SWB_EPI_RESID_F32 || resid, "%s: resid needed", fn);
  SWB_REQUIRE((((uintptr_t)x | (uintptr_t)w) & 15) == 0, "%s: pointers must be 16-byte aligned",
              fn);
  return SWB_OK;
}

extern "C" int swb_gemv_bf16(const void* x, const void* w, void* out, const void* resid, int M,
                             int N, int K, int epilogue, uintptr_t stream) {
  return swb_gemv_bf16_bias(x, w, out, resid, nullptr, M, N, K, epilogue, stream);
}

extern "C" int swb_gemv_bf16_bias(const void* x, const void* w, void* out, const void* resid,
                                  const void* bias, int M, int N, int K, int epilogue,
                                  uintptr_t stream) {
  const int st = check_gemv_args("swb_gemv_bf16", x, w, out, resid, M, N, K, epilogue);
  if (st) return st;
  SWB_REQUIRE(!bias || epilogue != SWB_EPI_SWIGLU, "swb_gemv_bf16: no bias with SwiGLU");
  return dispatch_gemv<false>(x, nullptr, 0.f, w, out, resid, bias, M, N, K, epilogue, stream);
}

extern "C" int swb_gemv_bf16_tp(const void* x, const void* w, const void* resid,
                                const void* bias, int M, int N, int K, int epilogue,
                                swb_tp_comm* comm, int slot, uintptr_t stream) {
  SWB_REQUIRE(comm, "swb_gemv_bf16_tp: null communicator");
  void* out = swb_tp_comm_slot(comm, slot);
  SWB_REQUIRE(out, "swb_gemv_bf16_tp: bad slot %d", slot);
  const int st = check_gemv_args("swb_gemv_bf16_tp", x, w, out, resid, M, N, K, epilogue);
  if (st) return st;
  SWB_REQUIRE(M == 1, "swb_gemv_bf16_tp: one row (decode B=1) only, got M=%d", M);
  SWB_REQUIRE(epilogue == SWB_EPI_F32 || epilogue == SWB_EPI_RESID_F32,
              "swb_gemv_bf16_tp: fp32 epilogues only");
  SWB_REQUIRE(N <= 16384 && N % 4 == 0,
              "swb_gemv_bf16_tp: N=%d must be a multiple of 4 within the receive buffers", N);
  const int items = (N + TV_ROWS - 1) / TV_ROWS;
  return launch_gemv<1, false>(x, nullptr, 0.f, reinterpret_cast<const __nv_bfloat16*>(w), out,
                               reinterpret_cast<const float*>(resid),
                               reinterpret_cast<const __nv_bfloat16*>(bias), M, N, K, epilogue,
                               items, (cudaStream_t)stream, comm, slot);
}

extern "C" int swb_gemv_rmsnorm_bf16(const float* x, const void* norm_w, float eps,
                                     const void* w, void* out, const void* resid, int M, int N,
                                     int K, int epilogue, uintptr_t stream) {
  const int st = check_gemv_args("swb_gemv_rmsnorm_bf16", x, w, out, resid, M, N, K, epilogue);
  if (st) return st;
  SWB_REQUIRE(norm_w && (((uintptr_t)norm_w) & 15) == 0,
              "swb_gemv_rmsnorm_bf16: norm weight must be 16-byte aligned");
  SWB_REQUIRE(epilogue != SWB_EPI_RESID_F32 || resid != x,
              "swb_gemv_rmsnorm_bf16: output may not alias the normalized input");
  SWB_REQUIRE(M == 1 ? (size_t)K * 2 <= (size_t)TV_HS_MAX
                     : (M <= 8 && (size_t)M * K * 2 <= (size_t)TM_HS_MAX),
              "swb_gemv_rmsnorm_bf16: staged h of M=%d x K=%d exceeds %d bytes (use "
              "swb_rmsnorm + GEMV)", M, K, M == 1 ? TV_HS_MAX : TM_HS_MAX);
  SWB_REQUIRE(K % 4 == 0, "swb_gemv_rmsnorm_bf16: K %% 4");
  return dispatch_gemv<true>(x, reinterpret_cast<const __nv_bfloat16*>(norm_w), eps, w, out,
                             resid, nullptr, M, N, K, epilogue, stream);
}
