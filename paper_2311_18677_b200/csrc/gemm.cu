// Prefill GEMM on the 5th-generation tensor cores (sm_100a).
//
//   out[M,N] = epilogue( A[M,K] . W[N,K]^T )      bf16 x bf16 -> fp32 (TMEM)
//
// One CTA computes a 128 x 256 output tile.  Warp 0 (one elected lane) is the
// TMA producer feeding a 4-stage ring of 128B-swizzled smem tiles (A 16 KB +
// W 32 KB per stage); warp 1 (one elected lane) issues tcgen05.mma
// (M=128, N=256, K=16, cta_group::1) into a 256-column TMEM accumulator and
// releases ring slots with tcgen05.commit; warp 2 owns the TMEM allocation.
// After the last k-block all four warps drain TMEM with tcgen05.ld (warp w
// owns TMEM lanes 32w..32w+31 = tile rows) and apply the fused epilogue:
// bf16 store, fp32 store, fp32 residual add (O / down projections), or
// SwiGLU over gate/up rows interleaved in 128-row groups (gate/up projection).
//
// This replaces the prompt-phase cost lookup PerfModel.prompt_time
// (reference perf.py:119-123) for the linear layers of a prefill.
#include <cstdarg>
#include <cstdio>
#include <cudaTypedefs.h>
#include <algorithm>

#include "common.cuh"

namespace swb {

constexpr int GM = 128, GN = 256, GK = 64, GSTAGES = 4;
constexpr int G_A_BYTES = GM * GK * 2;  // 16 KB
constexpr int G_B_BYTES = GN * GK * 2;  // 32 KB
constexpr int G_STAGE_BYTES = G_A_BYTES + G_B_BYTES;
constexpr int G_SMEM_BYTES = GSTAGES * G_STAGE_BYTES + 1024 + 256;
constexpr uint32_t G_TMEM_COLS = 512;   // two 256-column fp32 accumulators
constexpr int G_THREADS = 192;          // TMA warp, MMA warp, 4 epilogue warps

struct GemmArgs {
  void* out;
  const float* resid;
  const __nv_bfloat16* bias;
  int M, N, K;
  int epi;
  int m_tiles, tiles;
  // EPI_QKV_ROPE (swb_gemm_qkv_rope): q/k heads rotated at pos[row], k/v
  // rows written to the paged pool at slots[row] (slots may be null)
  const int32_t* pos;
  float log2_theta;
  int H, Hkv, bs;
  __nv_bfloat16* kpool;
  __nv_bfloat16* vpool;
  const int32_t* slots;
  const float2* rope_tab;   // [tab_len][64] (sin, cos) or null
  int tab_len;
};
constexpr int EPI_QKV_ROPE = 100;   // internal epilogue id

// QKV projection epilogue: bias, round to bf16 (the stored qkv), RoPE on the
// q and k heads from the rounded values (bit-identical to swb_rope_kv_write
// after a plain GEMM), k/v rows appended to the paged pool.  A 256-column
// tile holds two whole 128-dim heads; thread = row; pairs (d, d+64) come from
// TMEM column chunks c and c+2 of the head.
__device__ __forceinline__ void qkv_rope_epilogue(const GemmArgs& a, uint32_t t_row, int row,
                                                  int n0) {
  const bool row_ok = row < a.M;
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out);
  const int qend = a.H * 128, kend = (a.H + a.Hkv) * 128;
  const int ipos = row_ok ? __ldg(a.pos + row) : 0;
  const float pos = (float)ipos;
  const bool use_tab = ipos < a.tab_len;
  size_t pbase = 0;
  const bool pool = row_ok && a.slots != nullptr;
  if (pool) {
    const int slot = __ldg(a.slots + row);
    pbase = (((size_t)(slot / a.bs) * a.Hkv) * a.bs + slot % a.bs) * 128;
  }
  const bool any_rot = n0 < kend && a.log2_theta > 0.f;      // block-uniform
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    // (sin, cos) of this row's 32 pairs of chunk c, shared by the tile's heads
    float sn[32], cs[32];
    if (any_rot && row_ok) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (use_tab) {
          const float2 v = __ldg(a.rope_tab + ipos * 64 + c * 32 + i);
          sn[i] = v.x;
          cs[i] = v.y;
        } else {
          rope_sincos(c * 32 + i, pos, a.log2_theta, 128, sn[i], cs[i]);
        }
      }
    }
#pragma unroll 1
    for (int hh = 0; hh < 2; ++hh) {
      const int hcol = n0 + hh * 128;
      if (hcol >= a.N) break;                      // block-uniform
      const bool rot = hcol < kend && a.log2_theta > 0.f;
      uint32_t lo[32], hi[32];
      tmem_ld32(t_row + hh * 128 + c * 32, lo);
      tmem_ld32(t_row + hh * 128 + 64 + c * 32, hi);
      tc_wait_ld();
      if (!row_ok) continue;
      uint32_t plo[16], phi[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float x[2], y[2];
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const int d = c * 32 + i + e2;
          float va = __uint_as_float(lo[i + e2]), vb = __uint_as_float(hi[i + e2]);
          if (a.bias) {
            va += __bfloat162float(a.bias[hcol + d]);
            vb += __bfloat162float(a.bias[hcol + 64 + d]);
          }
          va = __bfloat162float(__float2bfloat16(va));      // the stored qkv value
          vb = __bfloat162float(__float2bfloat16(vb));
          if (rot) {
            rope_apply(va, vb, sn[i + e2], cs[i + e2], x[e2], y[e2]);
          } else {
            x[e2] = va;
            y[e2] = vb;
          }
        }
        plo[i / 2] = f2_to_bf2(x[0], x[1]);
        phi[i / 2] = f2_to_bf2(y[0], y[1]);
      }
      uint4* o_lo = reinterpret_cast<uint4*>(out + (size_t)row * a.N + hcol + c * 32);
      uint4* o_hi = reinterpret_cast<uint4*>(out + (size_t)row * a.N + hcol + 64 + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o_lo[i] = make_uint4(plo[4 * i], plo[4 * i + 1], plo[4 * i + 2], plo[4 * i + 3]);
        o_hi[i] = make_uint4(phi[4 * i], phi[4 * i + 1], phi[4 * i + 2], phi[4 * i + 3]);
      }
      if (pool && hcol >= qend) {
        __nv_bfloat16* dst = (hcol < kend ? a.kpool + (size_t)((hcol - qend) / 128) * a.bs * 128
                                          : a.vpool + (size_t)((hcol - kend) / 128) * a.bs * 128) +
                             pbase;
        uint4* p_lo = reinterpret_cast<uint4*>(dst + c * 32);
        uint4* p_hi = reinterpret_cast<uint4*>(dst + 64 + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          p_lo[i] = make_uint4(plo[4 * i], plo[4 * i + 1], plo[4 * i + 2], plo[4 * i + 3]);
          p_hi[i] = make_uint4(phi[4 * i], phi[4 * i + 1], phi[4 * i + 2], phi[4 * i + 3]);
        }
      }
    }
  }
}

// Epilogue of one 128 x 256 tile held in TMEM columns [acc_col, acc_col+256):
// this warp owns TMEM lanes (= tile rows) 32*(warp%4) .. +31.
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& args, uint32_t t_row, int row,
                                              int n0) {
  if (args.epi == EPI_QKV_ROPE) {
    qkv_rope_epilogue(args, t_row, row, n0);
    return;
  }
  const bool row_ok = row < args.M;
  uint32_t r[32];
  if (args.epi == SWB_EPI_SWIGLU) {
    // tile cols [0,128) = gate, [128,256) = up for outputs n0/2 + [0,128)
    const int nout = args.N >> 1;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out);
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t u[32];
      tmem_ld32(t_row + c * 32, r);
      tmem_ld32(t_row + 128 + c * 32, u);
      tc_wait_ld();
      const int col = (n0 >> 1) + c * 32;
      if (row_ok && col < nout) {
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float g0 = __uint_as_float(r[2 * i]), g1 = __uint_as_float(r[2 * i + 1]);
          const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
          packed[i] = f2_to_bf2(silu_f(g0) * u0, silu_f(g1) * u1);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * nout + col);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                              packed[4 * i + 3]);
      }
    }
    return;
  }
#pragma unroll 1
  for (int c = 0; c < GN / 32; ++c) {
    tmem_ld32(t_row + c * 32, r);
    tc_wait_ld();
    const int col = n0 + c * 32;
    if (!row_ok || col >= args.N) continue;
    if (args.bias) {
      const uint4* bp = reinterpret_cast<const uint4*>(args.bias + col);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 bb = __ldg(bp + i);
        const uint32_t w4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = bf2_to_f2(w4[k]);
          r[8 * i + 2 * k] = __float_as_uint(__uint_as_float(r[8 * i + 2 * k]) + f.x);
          r[8 * i + 2 * k + 1] = __float_as_uint(__uint_as_float(r[8 * i + 2 * k + 1]) + f.y);
        }
      }
    }
    if (args.epi == SWB_EPI_GELU) {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(gelu_tanh(__uint_as_float(r[i])));
    }
    if (args.epi == SWB_EPI_BF16 || args.epi == SWB_EPI_GELU) {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out);
      uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * args.N + col);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(
            f2_to_bf2(__uint_as_float(r[8 * i + 0]), __uint_as_float(r[8 * i + 1])),
            f2_to_bf2(__uint_as_float(r[8 * i + 2]), __uint_as_float(r[8 * i + 3])),
            f2_to_bf2(__uint_as_float(r[8 * i + 4]), __uint_as_float(r[8 * i + 5])),
            f2_to_bf2(__uint_as_float(r[8 * i + 6]), __uint_as_float(r[8 * i + 7])));
    } else {
      float* out = reinterpret_cast<float*>(args.out) + (size_t)row * args.N + col;
      if (args.epi == SWB_EPI_RESID_F32) {
        const float4* res =
            reinterpret_cast<const float4*>(args.resid + (size_t)row * args.N + col);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 v = res[i];
          v.x += __uint_as_float(r[4 * i + 0]);
          v.y += __uint_as_float(r[4 * i + 1]);
          v.z += __uint_as_float(r[4 * i + 2]);
          v.w += __uint_as_float(r[4 * i + 3]);
          reinterpret_cast<float4*>(out)[i] = v;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          reinterpret_cast<float4*>(out)[i] =
              make_float4(__uint_as_float(r[4 * i + 0]), __uint_as_float(r[4 * i + 1]),
                          __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
      }
    }
  }
}

// Persistent: one CTA per SM walks the 128 x 256 tiles in M-fastest order
// (CTAs resident together share weight tiles through L2).  Warp 0 = TMA
// producer, warp 1 = single-thread tcgen05.mma issuer, warps 2..5 = epilogue.
// Two TMEM accumulators let the epilogue of tile i overlap the MMAs of tile
// i+1 (tmem_full / tmem_empty mbarriers).
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmW, GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + GSTAGES * G_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GSTAGES * G_STAGE_BYTES);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tfull = empty + GSTAGES;     // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_k = (args.K + GK - 1) / GK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<G_TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // A (activations) is produced by the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < args.tiles; t += gridDim.x) {
        const int m0 = (t % args.m_tiles) * GM, n0 = (t / args.m_tiles) * GN;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % GSTAGES;
          if (it >= GSTAGES) mbar_wait_sleep(&empty[s], ((it / GSTAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], G_STAGE_BYTES);
          tma_load_2d(sA + s * G_A_BYTES, &tmA, &full[s], kb * GK, m0);
          tma_load_2d(sB + s * G_B_BYTES, &tmW, &full[s], kb * GK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      constexpr uint32_t idesc = umma_idesc_bf16(GM, GN);
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < args.tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        if (i >= 2) mbar_wait(&tempty[acc], ((i >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * GN;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % GSTAGES;
          mbar_wait(&full[s], (it / GSTAGES) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * G_A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * G_B_BYTES);
#pragma unroll
          for (int k = 0; k < GK / 16; ++k) {
            // K-major SW128: advancing 16 bf16 along K = +32 B start address.
            tc_mma_f16(d_tmem, umma_desc_k_sw128(a_base + k * 32),
                       umma_desc_k_sw128(b_base + k * 32), idesc, (kb | k) != 0);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps: TMEM -> registers -> global
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int i = 0;
    for (int t = blockIdx.x; t < args.tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const int m0 = (t % args.m_tiles) * GM, n0 = (t / args.m_tiles) * GN;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      gemm_epilogue(args, tmem + acc * GN + ((uint32_t)(q * 32) << 16), m0 + q * 32 + lane, n0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<G_TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile with tcgen05.mma M=256 (issued by the leader CTA only).
// Each CTA stages ITS 128 rows of A and ITS 128 rows of W (one half of the
// N=256 operand) per k-block, so per-SM shared-memory traffic per FLOP drops
// by a third and each SM's TMEM holds its own 128 x 256 accumulator rows;
// TMA completions of both CTAs land on the leader's mbarrier, the leader's
// commits multicast to both CTAs' ring / accumulator barriers, and the
// peer's epilogue warps release accumulators on the leader's barrier.
constexpr int G2_STAGES = 6;
constexpr int G2_STAGE_BYTES = G_A_BYTES + G_A_BYTES;   // 16 KB A + 16 KB W half
constexpr int G2_SMEM_BYTES = G2_STAGES * G2_STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t g2_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t g2_mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void g2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D TMA load into this CTA's smem, completion counted on the leader's
// mbarrier (cluster address)
__device__ __forceinline__ void g2_tma_load(void* smem_dst, const void* desc,
                                            uint32_t leader_bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void g2_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in both CTAs of the pair once
// the leader's MMAs issued so far completed
__device__ __forceinline__ void g2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void g2_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void g2_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmW, GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + G2_STAGES * G_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G2_STAGES * G2_STAGE_BYTES);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;   // [2] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained (leader: 8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = g2_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_k = (args.K + GK - 1) / GK;
  const int m_pairs = (args.M + 2 * GM - 1) / (2 * GM);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(G_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  g2_cluster_sync();   // peer barriers initialised, TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // A (activations) is produced by the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs: own A rows, own W half)
      int it = 0;
      for (int t = pair; t < args.tiles; t += npairs) {
        const int m0 = (t % m_pairs) * 2 * GM + (int)rank * GM;
        const int n0 = (t / m_pairs) * GN + (int)rank * (GN / 2);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % G2_STAGES;
          if (it >= G2_STAGES) mbar_wait_sleep(&empty[s], ((it / G2_STAGES) - 1) & 1);
          const uint32_t lbar = g2_mapa(smem_u32(&full[s]), 0);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * G2_STAGE_BYTES);
          g2_tma_load(sA + s * G_A_BYTES, &tmA, lbar, kb * GK, m0);
          g2_tma_load(sB + s * G_A_BYTES, &tmW, lbar, kb * GK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA, single thread)
      constexpr uint32_t idesc = umma_idesc_bf16(2 * GM, GN);
      int it = 0, i = 0;
      for (int t = pair; t < args.tiles; t += npairs, ++i) {
        const int acc = i & 1;
        if (i >= 2) mbar_wait(&tempty[acc], ((i >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * GN;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % G2_STAGES;
          mbar_wait(&full[s], (it / G2_STAGES) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * G_A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * G_A_BYTES);
#pragma unroll
          for (int k = 0; k < GK / 16; ++k)
            g2_mma(d_tmem, umma_desc_k_sw128(a_base + k * 32), umma_desc_k_sw128(b_base + k * 32),
                   idesc, (kb | k) != 0);
          g2_commit_both(&empty[s]);
        }
        g2_commit_both(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps (both CTAs): own 128 rows x 256 cols
    const int q = warp & 3;
    const uint32_t lead_tempty[2] = {g2_mapa(smem_u32(&tempty[0]), 0),
                                     g2_mapa(smem_u32(&tempty[1]), 0)};
    int i = 0;
    for (int t = pair; t < args.tiles; t += npairs, ++i) {
      const int acc = i & 1;
      const int m0 = (t % m_pairs) * 2 * GM + (int)rank * GM, n0 = (t / m_pairs) * GN;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      gemm_epilogue(args, tmem + acc * GN + ((uint32_t)(q * 32) << 16), m0 + q * 32 + lane, n0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) g2_arrive_remote(lead_tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  g2_cluster_sync();   // the leader's last MMAs / the peer's reads are done in both CTAs
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(G_TMEM_COLS));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 K-major operand [rows, K] -> tiles of box_rows x 64 (128 B rows),
// 128-byte swizzle, out-of-bounds rows/cols zero filled.
int make_tmap_bf16_kmajor(CUtensorMap* map, const void* base, int rows, int K,
                          int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return swb_set_error(SWB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return swb_set_error(SWB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SWB_OK;
}

int make_tmap_rows(CUtensorMap* map, const void* base, int rows, int K, int box_rows) {
  return make_tmap_bf16_kmajor(map, base, rows, K, box_rows);
}

// SWB_GEMM_PAIR=0 keeps every prefill GEMM on the single-CTA kernel (A/B)
static bool gemm_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SWB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct RopeArgs {
  const int32_t* pos;
  float log2_theta;
  int H, Hkv, bs;
  __nv_bfloat16* kpool;
  __nv_bfloat16* vpool;
  const int32_t* slots;
  const float2* tab;
  int tab_len;
};

__global__ void rope_table_kernel(float log2_theta, int n, float2* tab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;   // pos * 64 + pair
  if (i >= n * 64) return;
  float s, c;
  rope_sincos(i & 63, (float)(i >> 6), log2_theta, 128, s, c);
  tab[i] = make_float2(s, c);
}

static int launch_gemm_pair(const CUtensorMap& ta, const void* w, void* out, const void* resid,
                            const void* bias, int M, int N, int K, int epilogue,
                            cudaStream_t stream, const RopeArgs* rope = nullptr) {
  CUtensorMap tw;
  int st = make_tmap_bf16_kmajor(&tw, w, N, K, GN / 2);   // each CTA loads half of W's tile
  if (st) return st;
  static bool attr_set[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_pair,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, G2_SMEM_BYTES));
    attr_set[dev] = true;
  }
  const int m_pairs = (M + 2 * GM - 1) / (2 * GM), n_tiles = (N + GN - 1) / GN;
  GemmArgs args{out, reinterpret_cast<const float*>(resid),
                reinterpret_cast<const __nv_bfloat16*>(bias), M, N, K, epilogue, m_pairs,
                m_pairs * n_tiles};
  if (rope) {
    args.pos = rope->pos; args.log2_theta = rope->log2_theta; args.H = rope->H;
    args.Hkv = rope->Hkv; args.bs = rope->bs; args.kpool = rope->kpool;
    args.vpool = rope->vpool; args.slots = rope->slots;
    args.rope_tab = rope->tab; args.tab_len = rope->tab_len;
  }
  const int pairs = std::min(args.tiles, kNumSMs / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(G_THREADS);
  cfg.dynamicSmemBytes = G2_SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t le = cudaLaunchKernelEx(&cfg, gemm_bf16_tcgen05_pair, ta, tw, args);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch gemm_bf16_tcgen05_pair: %s",
                         cudaGetErrorString(le));
  return swb_check_launch("gemm_bf16_tcgen05_pair");
}

}  // namespace swb

using namespace swb;

static int gemm_launch(const void* a, const void* w, void* out, const void* resid,
                       const void* bias, int M, int N, int K, int epilogue,
                       cudaStream_t stream, const RopeArgs* rope);

extern "C" int swb_gemm_bf16(const void* a, const void* w, void* out,
                             const void* resid, int M, int N, int K, int epilogue,
                             uintptr_t stream) {
  return swb_gemm_bf16_bias(a, w, out, resid, nullptr, M, N, K, epilogue, stream);
}

extern "C" int swb_gemm_bf16_bias(const void* a, const void* w, void* out,
                                  const void* resid, const void* bias, int M, int N, int K,
                                  int epilogue, uintptr_t stream) {
  SWB_REQUIRE(a && w && out, "swb_gemm_bf16: null pointer");
  SWB_REQUIRE(!bias || epilogue != SWB_EPI_SWIGLU, "swb_gemm_bf16: no bias with SwiGLU");
  SWB_REQUIRE((((uintptr_t)bias) & 15) == 0, "swb_gemm_bf16: bias must be 16-byte aligned");
  SWB_REQUIRE(M > 0 && N > 0 && K > 0, "swb_gemm_bf16: bad shape M=%d N=%d K=%d", M, N, K);
  SWB_REQUIRE(K % 8 == 0, "swb_gemm_bf16: K=%d must be a multiple of 8", K);
  SWB_REQUIRE(N % 32 == 0, "swb_gemm_bf16: N=%d must be a multiple of 32", N);
  SWB_REQUIRE(epilogue >= SWB_EPI_BF16 && epilogue <= SWB_EPI_GELU,
              "swb_gemm_bf16: bad epilogue %d", epilogue);
  SWB_REQUIRE(epilogue != SWB_EPI_SWIGLU || N % 256 == 0,
              "swb_gemm_bf16: SwiGLU epilogue needs N %% 256 == 0 (N=%d)", N);
  SWB_REQUIRE(epilogue != SWB_EPI_RESID_F32 || resid,
              "swb_gemm_bf16: residual epilogue needs resid");
  SWB_REQUIRE((((uintptr_t)a | (uintptr_t)w | (uintptr_t)out) & 15) == 0,
              "swb_gemm_bf16: pointers must be 16-byte aligned");
  return gemm_launch(a, w, out, resid, bias, M, N, K, epilogue, (cudaStream_t)stream, nullptr);
}

static int gemm_launch(const void* a, const void* w, void* out, const void* resid,
                       const void* bias, int M, int N, int K, int epilogue,
                       cudaStream_t stream_, const RopeArgs* rope) {
  const uintptr_t stream = (uintptr_t)stream_;
  CUtensorMap ta, tw;
  int st = make_tmap_bf16_kmajor(&ta, a, M, K, GM);
  if (st) return st;
  if (M > GM && gemm_pair_enabled())
    return launch_gemm_pair(ta, w, out, resid, bias, M, N, K, epilogue, (cudaStream_t)stream,
                            rope);
  st = make_tmap_bf16_kmajor(&tw, w, N, K, GN);
  if (st) return st;
  static bool attr_set[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  G_SMEM_BYTES));
    attr_set[dev] = true;
  }
  const int m_tiles = (M + GM - 1) / GM, n_tiles = (N + GN - 1) / GN;
  GemmArgs args{out, reinterpret_cast<const float*>(resid),
                reinterpret_cast<const __nv_bfloat16*>(bias), M, N, K, epilogue, m_tiles,
                m_tiles * n_tiles};
  if (rope) {
    args.pos = rope->pos; args.log2_theta = rope->log2_theta; args.H = rope->H;
    args.Hkv = rope->Hkv; args.bs = rope->bs; args.kpool = rope->kpool;
    args.vpool = rope->vpool; args.slots = rope->slots;
    args.rope_tab = rope->tab; args.tab_len = rope->tab_len;
  }
  dim3 grid(std::min(args.tiles, kNumSMs));
  {
    const cudaError_t le_ = launch(gemm_bf16_tcgen05, dim3(grid), dim3(G_THREADS), G_SMEM_BYTES, (cudaStream_t)stream,
        ta, tw, args);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch gemm_bf16_tcgen05: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("gemm_bf16_tcgen05");
}

extern "C" int swb_rope_table(float theta, int max_pos, void* table, uintptr_t stream) {
  SWB_REQUIRE(table && max_pos > 0 && theta > 1.f, "swb_rope_table: bad args");
  const cudaError_t le = launch(rope_table_kernel, dim3((max_pos * 64 + 255) / 256), dim3(256), 0,
                                (cudaStream_t)stream, log2f(theta), max_pos,
                                reinterpret_cast<float2*>(table));
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch rope_table_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("rope_table_kernel");
}

extern "C" int swb_gemm_qkv_rope(const void* a, const void* w, void* qkv, const void* bias,
                                 int M, int N, int K, const int32_t* positions, float theta,
                                 const void* rope_table, int table_len, int H, int Hkv,
                                 void* k_layer, void* v_layer, const int32_t* slots,
                                 int block_size, uintptr_t stream) {
  SWB_REQUIRE(a && w && qkv && positions, "swb_gemm_qkv_rope: null pointer");
  SWB_REQUIRE(M > 0 && K > 0 && K % 8 == 0, "swb_gemm_qkv_rope: bad shape M=%d K=%d", M, K);
  SWB_REQUIRE(H > 0 && Hkv > 0 && N == (H + 2 * Hkv) * 128,
              "swb_gemm_qkv_rope: N=%d must be (H + 2 Hkv) * 128 (head_dim 128)", N);
  SWB_REQUIRE(!slots || (k_layer && v_layer && block_size > 0),
              "swb_gemm_qkv_rope: pool write needs k/v layers and block_size");
  SWB_REQUIRE((((uintptr_t)a | (uintptr_t)w | (uintptr_t)qkv | (uintptr_t)bias) & 15) == 0,
              "swb_gemm_qkv_rope: pointers must be 16-byte aligned");
  RopeArgs r{positions, theta > 1.f ? log2f(theta) : 0.f, H, Hkv, block_size,
             reinterpret_cast<__nv_bfloat16*>(k_layer), reinterpret_cast<__nv_bfloat16*>(v_layer),
             slots, reinterpret_cast<const float2*>(rope_table), rope_table ? table_len : 0};
  return gemm_launch(a, w, qkv, nullptr, bias, M, N, K, EPI_QKV_ROPE, (cudaStream_t)stream, &r);
}
