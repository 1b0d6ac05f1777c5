// Batched decode linears (M = 2..32 rows) on the 5th-generation tensor cores.
//
// Swap-AB: D[128 weight rows x NPAD batch] = W_tile[128 x K] . X^T[K x NPAD]
// with tcgen05.mma (M=128, N=NPAD, K=16), so the weights are the 128-row A
// operand streamed once from HBM by TMA (128 x 64 boxes, 128 B swizzle,
// L2 evict-first) and the batch is the narrow B operand (NPAD x 64 boxes,
// rows >= M zero-filled by TMA).  The MMA cost is negligible; the kernel is a
// pure HBM stream, like the M=1 bulk-copy GEMV, but its cost no longer grows
// with the batch.
//
// Work: output tiles of 128 rows (256 = gate+up groups for SwiGLU, R = 2)
// are split along K over the S CTAs of a thread-block cluster (S chosen on
// the host so clusters x S fills the 148 SMs with the fewest tile rounds).
// Each CTA accumulates its K-slice in TMEM (double-buffered, so the epilogue
// of tile i overlaps the MMAs of tile i+1); partial tiles are exchanged
// through distributed shared memory and every CTA of the cluster reduces a
// disjoint share of the tile in fixed rank order (deterministic, no global
// workspace, no atomics) and applies the epilogue (bias, GELU, SwiGLU,
// residual).  Weight loads of the first ring stages are issued before
// griddepcontrol.wait: they overlap the previous kernel's tail.
//   warp 0: TMA producer   warp 1: MMA issuer   warps 2-5: epilogue
#include <cudaTypedefs.h>

#include "common.cuh"

namespace swb {

int make_tmap_rows(CUtensorMap* map, const void* base, int rows, int K, int box_rows);

constexpr int GT_ROWS = 128;
constexpr int GT_WBOX = GT_ROWS * 128;   // 16 KB: 128 rows x 64 bf16
constexpr int GT_THREADS = 192;

template <int NPAD, int R>
struct GtCfg {
  static constexpr int XBOX = NPAD * 128;
  static constexpr int STAGE = R * GT_WBOX + XBOX;
  static constexpr int STAGES = (R == 1 ? 144 : 150) * 1024 / STAGE;
  static constexpr int RED = R * NPAD * GT_ROWS * 4;          // one partial tile, fp32
  static constexpr int OFF_RED = STAGES * STAGE;
  static constexpr int OFF_BAR = OFF_RED + 2 * RED;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int ACC = R * NPAD;                         // TMEM columns per buffer
  static constexpr int TCOLS = 2 * ACC <= 32 ? 32 : (2 * ACC <= 64 ? 64 : (2 * ACC <= 128 ? 128 : 256));
};

struct GtArgs {
  void* out;
  const float* resid;
  const __nv_bfloat16* bias;
  int M, N, K, epi;
  int tiles, nkb;
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ uint64_t gt_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Final value of output (m, n) from the K-summed accumulator(s).
__device__ __forceinline__ void gt_store(const GtArgs& a, int m, int n, float v, float u) {
  if (a.epi == SWB_EPI_SWIGLU) {   // v = gate, u = up; out [M, N/2]
    const int nout = a.N >> 1;
    reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)m * nout + n] =
        __float2bfloat16(silu_f(v) * u);
    return;
  }
  v += bias_at(a.bias, n);
  const size_t idx = (size_t)m * a.N + n;
  if (a.epi == SWB_EPI_BF16)
    reinterpret_cast<__nv_bfloat16*>(a.out)[idx] = __float2bfloat16(v);
  else if (a.epi == SWB_EPI_GELU)
    reinterpret_cast<__nv_bfloat16*>(a.out)[idx] = __float2bfloat16(gelu_tanh(v));
  else if (a.epi == SWB_EPI_F32)
    reinterpret_cast<float*>(a.out)[idx] = v;
  else
    reinterpret_cast<float*>(a.out)[idx] = a.resid[idx] + v;
}

template <int NPAD, int R>
__global__ void __launch_bounds__(GT_THREADS, 1)
    gemv_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GtArgs a) {
  using C = GtCfg<NPAD, R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;      // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint64_t* red_full = tempty + 2;          // [2] peers' partials landed (S-1 arrivals)
  uint64_t* red_free = red_full + 2;        // [2] peers finished reading mine
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_free + 2);
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [2][R][NPAD][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = (int)cluster_size();
  const int q = (int)cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();
  // this CTA's K-slice (in 64-wide blocks)
  const int kb_lo = (int)((long long)a.nkb * q / S), kb_hi = (int)((long long)a.nkb * (q + 1) / S);
  const int nkb = kb_hi - kb_lo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], 4);
    mbar_init(&tempty[1], 4);
    mbar_init(&red_full[0], S > 1 ? S - 1 : 1);
    mbar_init(&red_full[1], S > 1 ? S - 1 : 1);
    mbar_init(&red_free[0], S > 1 ? S - 1 : 1);
    mbar_init(&red_free[1], S > 1 ? S - 1 : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();          // peers' barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      tma_prefetch_desc(&tmW);
      tma_prefetch_desc(&tmX);
      const uint64_t pol = gt_policy_evict_first();
      int it = 0, pre = 0;
      bool waited = false;
      // X of the stages issued before griddepcontrol.wait (weights only)
      auto late_x = [&]() {
        pdl_wait();
        waited = true;
        for (int i = 0; i < pre; ++i)
          tma_load_2d(smem + i * C::STAGE + R * GT_WBOX, &tmX, &full[i], (kb_lo + i % nkb) * 64,
                      0);
      };
      for (int t = cid; t < a.tiles; t += ncl) {
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % C::STAGES;
          if (it >= C::STAGES) {
            if (!waited) late_x();
            mbar_wait_sleep(&empty[s], ((it / C::STAGES) - 1) & 1);
          }
          uint8_t* st = smem + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], C::STAGE);
#pragma unroll
          for (int r = 0; r < R; ++r)
            tma_load_2d_hint(st + r * GT_WBOX, &tmW, &full[s], kb * 64,
                             t * R * GT_ROWS + r * GT_ROWS, pol);
          if (waited)
            tma_load_2d(st + R * GT_WBOX, &tmX, &full[s], kb * 64, 0);
          else
            ++pre;   // weights are static: safe to fetch before the wait
        }
      }
      if (!waited) late_x();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(GT_ROWS, NPAD);
      int it = 0, tl = 0;
      for (int t = cid; t < a.tiles; t += ncl, ++tl) {
        const int ab = tl & 1;
        if (tl >= 2) mbar_wait(&tempty[ab], ((tl >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + ab * C::ACC;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * C::STAGE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int r = 0; r < R; ++r)
              tc_mma_f16(acc + r * NPAD, umma_desc_k_sw128(st + r * GT_WBOX + kk * 32),
                         umma_desc_k_sw128(st + R * GT_WBOX + kk * 32), idesc,
                         (kb | kk) != 0);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[ab]);
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps
    pdl_wait();                                  // resid / out belong to the stream
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;         // tile row = TMEM lane
    const int et = threadIdx.x - 64;             // 0..127
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int tl = 0;
    for (int t = cid; t < a.tiles; t += ncl, ++tl) {
      const int ab = tl & 1;
      mbar_wait(&tfull[ab], (tl >> 1) & 1);
      tc_fence_after();
      float v[R][NPAD];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < NPAD / 16; ++c) {
          uint32_t u[16];
          tmem_ld16(tmem + ab * C::ACC + r * NPAD + c * 16 + lane_off, u);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) v[r][c * 16 + i] = __uint_as_float(u[i]);
        }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      const int nbase = t * GT_ROWS;   // output feature base (SwiGLU: 128 per 256 rows)
      if (S == 1) {
        const int n = nbase + row;
        const int nlim = R == 1 ? a.N : (a.N >> 1);
        if (n < nlim) {
#pragma unroll
          for (int m = 0; m < NPAD; ++m)
            if (m < a.M) gt_store(a, m, n, v[0][m], R == 2 ? v[R - 1][m] : 0.f);
        }
        continue;
      }
      // ---- split-K: publish the partial tile, reduce a share of it
      float* rb = red + ab * (R * NPAD * GT_ROWS);
      if (tl >= 2) mbar_wait_cluster(&red_free[ab], ((tl >> 1) - 1) & 1);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < NPAD; ++m) rb[(r * NPAD + m) * GT_ROWS + row] = v[r][m];
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) {
        const uint32_t bar_local = smem_u32(&red_full[ab]);
        for (int p = 0; p < S; ++p)
          if (p != q) mbar_arrive_remote(mapa(bar_local, p));
      }
      mbar_wait_cluster(&red_full[ab], (tl >> 1) & 1);
      const uint32_t rb_local = smem_u32(rb);
      const int nlim = R == 1 ? a.N : (a.N >> 1);
      // elements e = m*128 + row of the tile, CTA q takes every S-th 128-row slab
      uint32_t base[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) base[p] = p < S ? mapa(rb_local, p) : 0u;
      for (int e = q * GT_ROWS + et; e < a.M * GT_ROWS; e += S * GT_ROWS) {
        const int m = e / GT_ROWS, rw = e % GT_ROWS;
        float sv = 0.f, su = 0.f;
#pragma unroll
        for (int p = 0; p < 8; ++p) {     // fixed rank order: deterministic
          if (p < S) {
            sv += ld_dsmem(base[p] + (m * GT_ROWS + rw) * 4);
            if (R == 2) su += ld_dsmem(base[p] + ((NPAD + m) * GT_ROWS + rw) * 4);
          }
        }
        const int n = nbase + rw;
        if (n < nlim) gt_store(a, m, n, sv, su);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) {
        const uint32_t bar_local = smem_u32(&red_free[ab]);
        for (int p = 0; p < S; ++p)
          if (p != q) mbar_arrive_remote(mapa(bar_local, p));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();          // no CTA leaves while peers may read its smem
  if (warp == 1) tmem_dealloc<C::TCOLS>(tmem);
}

// Cluster size S (K split) minimising ceil(tiles / clusters) / S for the
// clusters that fit on the GPU at once.
template <int NPAD, int R>
static int gt_pick(int tiles, int nkb, int* clusters) {
  using C = GtCfg<NPAD, R>;
  int best_s = 1, best_nc = 1;
  double best = 1e30;
  for (int s = 1; s <= 8; ++s) {
    if (nkb < 4 * s && s > 1) break;             // keep >= 4 K-blocks per CTA
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((148 / s) * s);
    cfg.blockDim = dim3(GT_THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = s;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int maxc = 0;
    if (cudaOccupancyMaxActiveClusters(&maxc, gemv_tc_kernel<NPAD, R>, &cfg) != cudaSuccess ||
        maxc <= 0) {
      cudaGetLastError();
      continue;
    }
    const int nc = std::min(tiles, maxc);
    const double cost = (double)((tiles + nc - 1) / nc) / s + 1e-3 * s;
    if (cost < best) {
      best = cost;
      best_s = s;
      best_nc = nc;
    }
  }
  *clusters = best_nc;
  return best_s;
}

template <int NPAD, int R>
static int launch_gemv_tc(const void* x, const void* w, void* out, const float* resid,
                          const __nv_bfloat16* bias, int M, int N, int K, int epi,
                          cudaStream_t stream) {
  using C = GtCfg<NPAD, R>;
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemv_tc_kernel<NPAD, R>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev] = true;
  }
  CUtensorMap tw, tx;
  int st = make_tmap_rows(&tw, w, N, K, GT_ROWS);
  if (st) return st;
  st = make_tmap_rows(&tx, x, M, K, NPAD);
  if (st) return st;
  GtArgs a{out, resid, bias, M, N, K, epi, R == 1 ? (N + GT_ROWS - 1) / GT_ROWS : N / 256,
           (K + 63) / 64};
  // cache the split choice per shape (host-side, no device sync)
  struct Key { int tiles, nkb, s, nc; };
  static Key cache[64];
  static int ncache = 0;
  int S = 0, nc = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].tiles == a.tiles && cache[i].nkb == a.nkb) {
      S = cache[i].s;
      nc = cache[i].nc;
    }
  if (!S) {
    S = gt_pick<NPAD, R>(a.tiles, a.nkb, &nc);
    if (ncache < 64) cache[ncache++] = Key{a.tiles, a.nkb, S, nc};
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc * S);
  cfg.blockDim = dim3(GT_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t le = cudaLaunchKernelEx(&cfg, gemv_tc_kernel<NPAD, R>, tw, tx, a);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch gemv_tc_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("gemv_tc_kernel");
}

int dispatch_gemv_tc(const void* x, const void* w, void* out, const float* resid,
                     const __nv_bfloat16* bias, int M, int N, int K, int epi, cudaStream_t s) {
  const bool sw = epi == SWB_EPI_SWIGLU;
  if (M <= 16)
    return sw ? launch_gemv_tc<16, 2>(x, w, out, resid, bias, M, N, K, epi, s)
              : launch_gemv_tc<16, 1>(x, w, out, resid, bias, M, N, K, epi, s);
  return sw ? launch_gemv_tc<32, 2>(x, w, out, resid, bias, M, N, K, epi, s)
            : launch_gemv_tc<32, 1>(x, w, out, resid, bias, M, N, K, epi, s);
}

}  // namespace swb
