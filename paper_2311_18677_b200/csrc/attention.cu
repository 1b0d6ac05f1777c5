// Attention kernels of the hot path.
//
// (1) attn_prefill: causal, varlen (several prompts packed back to back,
//     delimited by cu_seqlens), GQA.  FlashAttention-2 style online softmax:
//     one CTA = 64 query rows x one head, 4 warps x 16 rows, K/V tiles of 64
//     keys double-buffered in XOR-swizzled smem through cp.async, bf16
//     m16n8k16 tensor-core MMAs with P kept in registers.  (At the BASELINE
//     prompt lengths attention is 2-4 % of prefill FLOPs; the linear layers
//     run on tcgen05, see gemm.cu.)
// (2) attn_decode: paged decode attention over the KV block pool.  One CTA
//     per (sequence, kv head, context partition); the G = H/Hkv query heads
//     of a GQA group share one pass over the K/V blocks, which are streamed
//     with 16-byte coalesced loads (a (block, head) tile is 4 KB contiguous).
//     Scores live in smem, softmax uses warp-shuffle reductions, partitions
//     are merged in fp32 by a second kernel (split-K over the context).
//
// These replace the attention share of the reference's latency lookups
// (perf.py:119-132); the reference has no attention arithmetic at all.
#include <algorithm>

#include <cstring>

#include "common.cuh"

namespace swb {

// ============================================================ prefill
constexpr int PA_BQ = 128, PA_BK = 64, PA_D = 128;
constexpr int PA_WARPS = PA_BQ / 16;                 // 16 query rows per warp
constexpr int PA_THREADS = PA_WARPS * 32;
constexpr int PA_ROW_BYTES = PA_D * 2;               // 256 B
constexpr int PA_Q_BYTES = PA_BQ * PA_ROW_BYTES;     // 32 KB
constexpr int PA_KV_BYTES = PA_BK * PA_ROW_BYTES;    // 16 KB
constexpr int PA_SMEM = PA_Q_BYTES + 4 * PA_KV_BYTES;  // Q + 2xK + 2xV

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return row * PA_ROW_BYTES + ((chunk ^ (row & 7)) << 4);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                        uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4],
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// load a ROWS x 128-col bf16 tile (rows [r0, r0+ROWS) of a strided matrix,
// rows >= rmax zero-filled) into swizzled smem
template <int ROWS>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g,
                                          int stride, int r0, int rmax) {
#pragma unroll
  for (int i = 0; i < ROWS * 16 / PA_THREADS; ++i) {
    const int idx = threadIdx.x + i * PA_THREADS;
    const int row = idx >> 4, chunk = idx & 15;
    const bool valid = r0 + row < rmax;
    const __nv_bfloat16* src = g + (size_t)(valid ? r0 + row : 0) * stride + chunk * 8;
    cp_async16(sbase + swz(row, chunk), src, valid);
  }
}

__global__ void __launch_bounds__(PA_THREADS)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, int rs,
                        const int32_t* __restrict__ cu, int tiles_per_seq, int H,
                        int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(128) uint8_t sm[];
  const int seq = blockIdx.x / tiles_per_seq;
  // heavy (late) tiles first
  const int qt = tiles_per_seq - 1 - (blockIdx.x % tiles_per_seq);
  const int h = blockIdx.y;
  const int kh = h / (H / Hkv);
  const int s0 = cu[seq], len = cu[seq + 1] - s0;
  const int q0 = qt * PA_BQ;
  if (q0 >= len) return;

  const uint32_t sQ = smem_u32(sm);
  const uint32_t sK[2] = {sQ + PA_Q_BYTES, sQ + PA_Q_BYTES + PA_KV_BYTES};
  const uint32_t sV[2] = {sQ + PA_Q_BYTES + 2 * PA_KV_BYTES, sQ + PA_Q_BYTES + 3 * PA_KV_BYTES};
  const __nv_bfloat16* gq = qkv + (size_t)s0 * rs + h * PA_D;
  const __nv_bfloat16* gk = qkv + (size_t)s0 * rs + (H + kh) * PA_D;
  const __nv_bfloat16* gv = qkv + (size_t)s0 * rs + (H + Hkv + kh) * PA_D;

  load_tile<PA_BQ>(sQ, gq, rs, q0, len);
  load_tile<PA_BK>(sK[0], gk, rs, 0, len);
  load_tile<PA_BK>(sV[0], gv, rs, 0, len);
  cp_async_commit();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  uint32_t qf[8][4];
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  // causal: key tiles up to the one holding this query tile's last row
  const int nkv = (min(q0 + PA_BQ, len) - 1) / PA_BK + 1;

  for (int j = 0; j < nkv; ++j) {
    const int buf = j & 1;
    if (j + 1 < nkv) {
      load_tile<PA_BK>(sK[buf ^ 1], gk, rs, (j + 1) * PA_BK, len);
      load_tile<PA_BK>(sV[buf ^ 1], gv, rs, (j + 1) * PA_BK, len);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int row = warp * 16 + (lane & 15);
        const int chunk = kk * 2 + (lane >> 4);
        ldsm_x4(sQ + swz(row, chunk), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int chunk = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK[buf] + swz(key, chunk), b0, b1, b2, b3);
        mma_bf16(s[2 * np], qf[kk], b0, b1);
        mma_bf16(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // causal mask on tiles that reach past this warp's first row (also masks
    // keys beyond len)
    const int qrow0 = q0 + warp * 16 + g;
    if ((j + 1) * PA_BK > q0 + warp * 16) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int key = j * PA_BK + nt * 8 + 2 * t;
        if (key > qrow0) s[nt][0] = -INFINITY;
        if (key + 1 > qrow0) s[nt][1] = -INFINITY;
        if (key > qrow0 + 8) s[nt][2] = -INFINITY;
        if (key + 1 > qrow0 + 8) s[nt][3] = -INFINITY;
      }
    }
    // online softmax (rows g and g+8 of the warp's 16)
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mnew[0] = fmaxf(mnew[0], fmaxf(s[nt][0], s[nt][1]));
      mnew[1] = fmaxf(mnew[1], fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float corr[2], msc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      msc[r] = mnew[r] == -INFINITY ? 0.f : mnew[r] * scale_log2;
      corr[r] = exp2f(mrow[r] * scale_log2 - msc[r]);
      if (mrow[r] == -INFINITY) corr[r] = 0.f;
      mrow[r] = mnew[r];
    }
    float rsum[2] = {0.f, 0.f};
    uint32_t pf[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] * scale_log2 - msc[0]);
      const float p1 = exp2f(s[nt][1] * scale_log2 - msc[0]);
      const float p2 = exp2f(s[nt][2] * scale_log2 - msc[1]);
      const float p3 = exp2f(s[nt][3] * scale_log2 - msc[1]);
      rsum[0] += p0 + p1;
      rsum[1] += p2 + p3;
      const int kstep = nt >> 1;
      if ((nt & 1) == 0) {
        pf[kstep][0] = f2_to_bf2(p0, p1);
        pf[kstep][1] = f2_to_bf2(p2, p3);
      } else {
        pf[kstep][2] = f2_to_bf2(p0, p1);
        pf[kstep][3] = f2_to_bf2(p2, p3);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * corr[r] + rsum[r];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        const int key = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int chunk = dp * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sV[buf] + swz(key, chunk), b0, b1, b2, b3);
        mma_bf16(o[2 * dp], pf[ks], b0, b1);
        mma_bf16(o[2 * dp + 1], pf[ks], b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const int Hd = H * PA_D;
  const int r0 = q0 + warp * 16 + g;
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int col = h * PA_D + nt * 8 + 2 * t;
    if (r0 < len)
      *reinterpret_cast<uint32_t*>(out + (size_t)(s0 + r0) * Hd + col) =
          f2_to_bf2(o[nt][0] * inv0, o[nt][1] * inv0);
    if (r0 + 8 < len)
      *reinterpret_cast<uint32_t*>(out + (size_t)(s0 + r0 + 8) * Hd + col) =
          f2_to_bf2(o[nt][2] * inv1, o[nt][3] * inv1);
  }
}

// ============================================================ decode
constexpr int DA_D = 128;
constexpr int DA_MAXG = 8;
constexpr int DA_MAXPART = 128;

// Decode attention, one kernel per layer:
//   grid (NP, Hkv, B), 128 threads; CTA (p, kh, b) covers context tokens
//   [p*part, (p+1)*part) of sequence b for the G = H/Hkv query heads of kv
//   head kh (a GQA group shares one pass over its K/V pages).
// * STEP (the decode graph): ctx_lens[b] = tokens already cached; the current
//   token sits at position ctx_lens[b], its slot comes from the block table.
//   Tables, ctx and the cached pages are produced by earlier launches, so the
//   page gather is issued BEFORE griddepcontrol.wait and overlaps the QKV
//   projection's tail; only q and the current k/v wait for it.
//   !STEP: ctx_lens[b] = attention length including the current token, which
//   (when pos/slots are given) sits at pos[b] and is appended at slots[b].
// * Pages arrive as 4 KB (block, head) bulk copies; K and V have separate
//   mbarriers so the scores run while V is still in flight.
// * Scores: half-warp per token (4 tokens in flight), shuffle-reduced dots
//   against the G query heads; softmax max/exp-sum per head by one warp; P.V
//   with lane-owned dims; the current token's k/v (RoPE'd here) are patched
//   into the staged pages from shared memory, never re-read from global.
// * Split-K merge fused: every CTA publishes (o, m, l); the last CTA of a
//   (b, kh) group (atomic ticket) merges all partitions in fixed order.
// rope4 split in two: the angles (position known early) and the rotation
__device__ __forceinline__ void rope_sincos4(float* sn, float* cs, int i0, float pos, float l2t) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float inv_freq = exp2f(-l2t * (float)(2 * (i0 + j)) / (float)DA_D);
    sincosf(pos * inv_freq, &sn[j], &cs[j]);
  }
}
__device__ __forceinline__ void rope_apply4(float* a, float* b, const float* sn, const float* cs) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float x = a[j], y = b[j];
    a[j] = x * cs[j] - y * sn[j];
    b[j] = y * cs[j] + x * sn[j];
  }
}
__device__ __forceinline__ void rope4(float* a, float* b, int i0, float pos, float l2t) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float inv_freq = exp2f(-l2t * (float)(2 * (i0 + j)) / (float)DA_D);
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    const float x = a[j], y = b[j];
    a[j] = x * cs - y * sn;
    b[j] = y * cs + x * sn;
  }
}


// Split-K merge of the NP partition partials of one (b, kv head) group,
// executed by the last CTA: the (m, l) pairs are fetched in parallel and the
// per-partition factors exp2(m_p - M) computed once per head in shared
// memory, then every thread sums its float4 of O over the partitions with
// independent loads (a per-element dependent chain of L2 round trips made
// the merge the slowest phase for GQA groups).  Fixed partition order:
// deterministic.
__device__ __forceinline__ void decode_merge(const float* __restrict__ ws_bh, int NP, int G,
                                             int kh, int H, float* scratch,
                                             __nv_bfloat16* __restrict__ out_b, int nthreads) {
  // ws_bh = partials of (b, head 0): [H][NP][DA_D + 2]
  float* sf = scratch;              // [G][NP] factors
  float* sL = scratch + G * NP;     // [G]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
  for (int i = tid; i < G * NP; i += nthreads) {
    const int gi = i / NP, pp = i % NP;
    const float* w = ws_bh + ((size_t)(kh * G + gi) * NP + pp) * (DA_D + 2);
    sf[i] = __ldcg(w + DA_D);
    sf[G * NP + G + i] = __ldcg(w + DA_D + 1);   // l, after sL
  }
  __syncthreads();
  for (int gi = warp; gi < G; gi += nwarps) {
    float M = -INFINITY;
    for (int pp = lane; pp < NP; pp += 32) M = fmaxf(M, sf[gi * NP + pp]);
    M = warp_max(M);
    float L = 0.f;
    for (int pp = lane; pp < NP; pp += 32) {
      const float m = sf[gi * NP + pp];
      const float f = m == -INFINITY ? 0.f : exp2f(m - M);
      L += f * sf[G * NP + G + gi * NP + pp];
      sf[gi * NP + pp] = f;
    }
    L = warp_sum(L);
    if (lane == 0) sL[gi] = L;
  }
  __syncthreads();
  for (int i = tid; i < G * (DA_D / 4); i += nthreads) {
    const int gi = i / (DA_D / 4), d4 = i % (DA_D / 4);
    const float* base = ws_bh + (size_t)(kh * G + gi) * NP * (DA_D + 2) + d4 * 4;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int pp = 0; pp < NP; ++pp) {
      const float f = sf[gi * NP + pp];
      const float* w = base + (size_t)pp * (DA_D + 2);
      const float2 a = __ldcg(reinterpret_cast<const float2*>(w));
      const float2 c = __ldcg(reinterpret_cast<const float2*>(w + 2));
      o.x = fmaf(f, a.x, o.x); o.y = fmaf(f, a.y, o.y);
      o.z = fmaf(f, c.x, o.z); o.w = fmaf(f, c.y, o.w);
    }
    const float inv = 1.f / sL[gi];
    __nv_bfloat16* dst = out_b + (size_t)(kh * G + gi) * DA_D + d4 * 4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(f2_to_bf2(o.x * inv, o.y * inv),
                                                f2_to_bf2(o.z * inv, o.w * inv));
  }
}

template <bool STEP, int NW>
__global__ void __launch_bounds__(NW * 32)
    attn_decode_kernel(const __nv_bfloat16* __restrict__ qkv, int rs,
                       __nv_bfloat16* __restrict__ kpool, __nv_bfloat16* __restrict__ vpool,
                       const int32_t* __restrict__ tables, int max_blocks,
                       const int32_t* __restrict__ ctx_lens, const int32_t* __restrict__ pos,
                       const int32_t* __restrict__ slots, float log2_theta,
                       const float* __restrict__ alibi, int H, int Hkv, int bs,
                       float scale_log2, int part, float* __restrict__ ws,
                       int* __restrict__ tickets, __nv_bfloat16* __restrict__ out, int trig) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  const int p = blockIdx.x, kh = blockIdx.y, b = blockIdx.z;
  const int NP = gridDim.x;
  const int G = H / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto wsp = [&](int gh, int pp) {
    return ws + (((size_t)b * H + gh) * NP + pp) * (DA_D + 2);
  };
  __shared__ uint64_t bars[2];                       // K pages, V pages
  __shared__ int s_last;
  __shared__ __align__(16) __nv_bfloat16 scur[2][DA_D];  // current token's k (rotated), v
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(dsm_raw);      // [part][128]
  __nv_bfloat16* sv = sk + (size_t)part * DA_D;                        // [part][128]
  float* sq = reinterpret_cast<float*>(sv + (size_t)part * DA_D);      // [G][128]
  float* ss = sq + G * DA_D;                                           // [G][part]
  float* sacc = ss + G * part;                                         // [WARPS][G][128]
  float* sstat = sacc + NW * G * DA_D;                           // [G][2]
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int32_t* trow = tables + (size_t)b * max_blocks;
  const int lbs = __ffs(bs) - 1;
  int L, cur;  // attention length; current token position (-1: nothing appended)
  if constexpr (STEP) {
    const int c = __ldg(ctx_lens + b);
    L = c + 1;
    cur = c;
  } else {
    pdl_wait();
    L = ctx_lens[b];
    cur = pos ? pos[b] : -1;
  }
  const int t0 = p * part;
  const int t1 = min(L, t0 + part);
  const int ntok = t1 - t0;
  const bool own_cur = cur >= t0 && cur < t1;
  if (warp == 0 && ntok > 0) {
    // ---- gather the cached pages of the partition (4 KB per (block, head))
    const int cend = cur >= 0 ? min(t1, cur) : t1;
    const int nblk = (max(0, cend - t0) + bs - 1) >> lbs;
    const uint32_t tile = (uint32_t)bs * DA_D * 2;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[0], tile * nblk);
      mbar_arrive_expect_tx(&bars[1], tile * nblk);
    }
    __syncwarp();
    for (int j = lane; j < nblk; j += 32) {
      const int blk = __ldg(trow + (t0 >> lbs) + j);
      bulk_g2s(sk + (size_t)j * bs * DA_D, kpool + ((size_t)blk * Hkv + kh) * bs * DA_D, tile,
               &bars[0]);
    }
    for (int j = lane; j < nblk; j += 32) {
      const int blk = __ldg(trow + (t0 >> lbs) + j);
      bulk_g2s(sv + (size_t)j * bs * DA_D, vpool + ((size_t)blk * Hkv + kh) * bs * DA_D, tile,
               &bars[1]);
    }
  }
  if constexpr (STEP) pdl_wait();   // q / current k,v come from the QKV projection

  if (ntok > 0) {
    const int qpos = cur >= 0 ? cur : L - 1;    // query position (ALiBi)
    const __nv_bfloat16* qrow = qkv + (size_t)b * rs;
    const float fpos = (float)cur;
    // ---- q of the group (rotated), scaled by softmax scale * log2(e)
    for (int i = threadIdx.x; i < G * (DA_D / 8); i += (NW * 32)) {
      const int gi = i / (DA_D / 8), i0 = (i % (DA_D / 8)) * 4;
      const __nv_bfloat16* hp = qrow + (kh * G + gi) * DA_D;
      const uint2 ql = *reinterpret_cast<const uint2*>(hp + i0);
      const uint2 qh = *reinterpret_cast<const uint2*>(hp + 64 + i0);
      const float2 l0 = bf2_to_f2(ql.x), l1 = bf2_to_f2(ql.y);
      const float2 h0 = bf2_to_f2(qh.x), h1 = bf2_to_f2(qh.y);
      float lo[4] = {l0.x, l0.y, l1.x, l1.y}, hi[4] = {h0.x, h0.y, h1.x, h1.y};
      if (cur >= 0 && !alibi) {
        rope4(lo, hi, i0, fpos, log2_theta);
        // match the two-kernel path: rotated q is rounded to bf16
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          lo[j] = __bfloat162float(__float2bfloat16(lo[j]));
          hi[j] = __bfloat162float(__float2bfloat16(hi[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sq[gi * DA_D + i0 + j] = lo[j] * scale_log2;
        sq[gi * DA_D + 64 + i0 + j] = hi[j] * scale_log2;
      }
    }
    // ---- current token: rotate k, append k/v to the pool, stage in smem
    if (own_cur && threadIdx.x < 16) {
      const int i0 = threadIdx.x * 4;           // 16 threads x 4 pairs = 64 pairs
      const __nv_bfloat16* kp = qrow + (H + kh) * DA_D;
      const __nv_bfloat16* vp = qrow + (H + Hkv + kh) * DA_D;
      const uint2 kl = *reinterpret_cast<const uint2*>(kp + i0);
      const uint2 khi = *reinterpret_cast<const uint2*>(kp + 64 + i0);
      const float2 a0 = bf2_to_f2(kl.x), a1 = bf2_to_f2(kl.y);
      const float2 c0 = bf2_to_f2(khi.x), c1 = bf2_to_f2(khi.y);
      float lo[4] = {a0.x, a0.y, a1.x, a1.y}, hi[4] = {c0.x, c0.y, c1.x, c1.y};
      if (!alibi) rope4(lo, hi, i0, fpos, log2_theta);
      const int slot = STEP ? __ldg(trow + (cur >> lbs)) * bs + (cur & (bs - 1)) : slots[b];
      const size_t g = (((size_t)(slot >> lbs) * Hkv + kh) * bs + (slot & (bs - 1))) * DA_D;
      const uint2 klo = make_uint2(f2_to_bf2(lo[0], lo[1]), f2_to_bf2(lo[2], lo[3]));
      const uint2 khh = make_uint2(f2_to_bf2(hi[0], hi[1]), f2_to_bf2(hi[2], hi[3]));
      const uint2 vlo = *reinterpret_cast<const uint2*>(vp + i0);
      const uint2 vhi = *reinterpret_cast<const uint2*>(vp + 64 + i0);
      *reinterpret_cast<uint2*>(kpool + g + i0) = klo;
      *reinterpret_cast<uint2*>(kpool + g + 64 + i0) = khh;
      *reinterpret_cast<uint2*>(vpool + g + i0) = vlo;
      *reinterpret_cast<uint2*>(vpool + g + 64 + i0) = vhi;
      *reinterpret_cast<uint2*>(&scur[0][i0]) = klo;
      *reinterpret_cast<uint2*>(&scur[0][64 + i0]) = khh;
      *reinterpret_cast<uint2*>(&scur[1][i0]) = vlo;
      *reinterpret_cast<uint2*>(&scur[1][64 + i0]) = vhi;
    }
    __syncthreads();
    mbar_wait(&bars[0], 0);
    if (own_cur && threadIdx.x < 16)
      reinterpret_cast<uint4*>(sk + (size_t)(cur - t0) * DA_D)[threadIdx.x] =
          reinterpret_cast<const uint4*>(scur[0])[threadIdx.x];
    __syncthreads();

    // ---- scores: half-warp per token, 4 tokens in flight per half-warp
    {
      const int half = lane >> 4, hl = lane & 15;
      constexpr int STRIDE = NW * 2;
      const int hw = warp * 2 + half;
      for (int base = 0; base < ntok; base += 4 * STRIDE) {   // warp-uniform
        float kf[4][8];
        bool valid[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tt = base + hw + u * STRIDE;
          valid[u] = tt < ntok;
          const uint4 kv =
              *reinterpret_cast<const uint4*>(sk + (valid[u] ? tt : 0) * DA_D + hl * 8);
          const float2 a = bf2_to_f2(kv.x), c = bf2_to_f2(kv.y), e = bf2_to_f2(kv.z),
                       f = bf2_to_f2(kv.w);
          kf[u][0] = a.x; kf[u][1] = a.y; kf[u][2] = c.x; kf[u][3] = c.y;
          kf[u][4] = e.x; kf[u][5] = e.y; kf[u][6] = f.x; kf[u][7] = f.y;
        }
        for (int gi = 0; gi < G; ++gi) {
          // ALiBi (BLOOM): + slope * (key_pos - query_pos), log2 domain
          const float sl = alibi ? alibi[kh * G + gi] * 1.4426950408889634f : 0.f;
          const float4 q0 = *reinterpret_cast<const float4*>(sq + gi * DA_D + hl * 8);
          const float4 q1 = *reinterpret_cast<const float4*>(sq + gi * DA_D + hl * 8 + 4);
          float d[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float t = q0.x * kf[u][0];
            t = fmaf(q0.y, kf[u][1], t); t = fmaf(q0.z, kf[u][2], t);
            t = fmaf(q0.w, kf[u][3], t); t = fmaf(q1.x, kf[u][4], t);
            t = fmaf(q1.y, kf[u][5], t); t = fmaf(q1.z, kf[u][6], t);
            t = fmaf(q1.w, kf[u][7], t);
            d[u] = t;
          }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
          if (hl == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int tt = base + hw + u * STRIDE;
              if (valid[u]) ss[gi * part + tt] = fmaf(sl, (float)(t0 + tt - qpos), d[u]);
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- softmax statistics per head (one warp per head), p = exp2(s - m)
    for (int gi = warp; gi < G; gi += NW) {
      float m = -INFINITY;
      for (int i = lane; i < ntok; i += 32) m = fmaxf(m, ss[gi * part + i]);
      m = warp_max(m);
      float l = 0.f;
      for (int i = lane; i < ntok; i += 32) {
        const float e = exp2f(ss[gi * part + i] - m);
        ss[gi * part + i] = e;
        l += e;
      }
      l = warp_sum(l);
      if (lane == 0) {
        sstat[gi * 2] = m;
        sstat[gi * 2 + 1] = l;
      }
    }
    mbar_wait(&bars[1], 0);
    if (own_cur && threadIdx.x < 16)
      reinterpret_cast<uint4*>(sv + (size_t)(cur - t0) * DA_D)[threadIdx.x] =
          reinterpret_cast<const uint4*>(scur[1])[threadIdx.x];
    __syncthreads();
    // ---- P V: warp per token stripe, lane owns dims [4*lane, 4*lane+4)
    float acc[DA_MAXG][4];
#pragma unroll
    for (int gi = 0; gi < DA_MAXG; ++gi) acc[gi][0] = acc[gi][1] = acc[gi][2] = acc[gi][3] = 0.f;
    for (int tt = warp; tt < ntok; tt += NW) {
      const uint2 vv = *reinterpret_cast<const uint2*>(sv + tt * DA_D + lane * 4);
      const float2 v0 = bf2_to_f2(vv.x), v1 = bf2_to_f2(vv.y);
#pragma unroll
      for (int gi = 0; gi < DA_MAXG; ++gi) {
        if (gi >= G) break;
        const float pw = ss[gi * part + tt];
        acc[gi][0] = fmaf(pw, v0.x, acc[gi][0]);
        acc[gi][1] = fmaf(pw, v0.y, acc[gi][1]);
        acc[gi][2] = fmaf(pw, v1.x, acc[gi][2]);
        acc[gi][3] = fmaf(pw, v1.y, acc[gi][3]);
      }
    }
#pragma unroll
    for (int gi = 0; gi < DA_MAXG; ++gi) {
      if (gi >= G) break;
      *reinterpret_cast<float4*>(sacc + ((size_t)warp * G + gi) * DA_D + lane * 4) =
          make_float4(acc[gi][0], acc[gi][1], acc[gi][2], acc[gi][3]);
    }
    __syncthreads();
    if (trig) pdl_launch_dependents();
    for (int i = threadIdx.x; i < G * DA_D; i += (NW * 32)) {
      const int gi = i / DA_D, d = i % DA_D;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += sacc[((size_t)w * G + gi) * DA_D + d];
      if (NP == 1) {   // single partition: no merge
        out[((size_t)b * H + kh * G + gi) * DA_D + d] = __float2bfloat16(v / sstat[gi * 2 + 1]);
        continue;
      }
      float* wo = wsp(kh * G + gi, p);
      wo[d] = v;
      if (d == 0) {
        wo[DA_D] = sstat[gi * 2];
        wo[DA_D + 1] = sstat[gi * 2 + 1];
      }
    }
    if (NP == 1) return;
  } else {
    if (trig) pdl_launch_dependents();
    if (threadIdx.x < G) {
      float* w = wsp(kh * G + threadIdx.x, p);
      w[DA_D] = -INFINITY;
      w[DA_D + 1] = 0.f;
    }
  }
  // ---- fused split-K merge: the last CTA of (b, kh) combines the partitions
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* t = tickets + (size_t)b * Hkv + kh;
    const int prev = atomicAdd(t, 1);
    s_last = prev == NP - 1;
    if (s_last) *t = 0;  // reset for the next launch (graph replay)
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  decode_merge(ws + (size_t)b * H * NP * (DA_D + 2), NP, G, kh, H,
               reinterpret_cast<float*>(dsm_raw), out + (size_t)b * H * DA_D, NW * 32);
}


// ---------------------------------------------------------------- decode, cluster
// Streaming decode attention for MHA / small groups (G = 1 or 2 query heads
// per kv head, block_size 16, decode-graph form).  One thread-block CLUSTER of DCL_CL CTAs per (sequence,
// kv head); CTA r of the cluster streams pages [r*pp, (r+1)*pp) of the context
// through a DCL_S-stage shared-memory ring: a producer warp issues the 4 KB K
// and V bulk copies of each (block, head) page (the first DCL_S pages before
// griddepcontrol.wait, overlapping the QKV projection's tail), and DCL_CW
// consumer warps each own every DCL_CW-th page with an online softmax of
// their own — no block-wide barrier until the end, so a warp computes as
// soon as ITS page landed.  Warps combine through shared memory and the
// cluster's CTAs through distributed shared memory (every CTA stores its
// (m, l, o) into rank 0's inbox with st.shared::cluster and arrives on rank
// 0's merge barrier, then exits; rank 0 merges in fixed order): no global
// partials, no atomic ticket, no system fences.  The current token (position ctx) is
// RoPE'd and appended to the pool by the warp owning its page, which patches
// the staged page row from registers.
// Template: G query heads per kv head, DCL_CL CTAs per cluster (8 portable,
// 16 opt-in), DCL_CW consumer warps.
constexpr int DCL_PAGE = 16 * DA_D;   // elements of one (block, head) page
constexpr int DCL_ST = DA_D + 4;      // floats per (o[128], m, l) record (16-byte aligned)
#ifdef SWB_ATTN_PROBE
// timeline probe build (tools only): per-CTA globaltimer stamps
__device__ unsigned long long* g_attn_probe = nullptr;
#define ATTN_PROBE(k)                                                                    \
  do {                                                                                   \
    if (g_attn_probe && threadIdx.x == 0) {                                              \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
      g_attn_probe[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + \
                   (k)] = t_;                                                            \
    }                                                                                    \
  } while (0)
#else
#define ATTN_PROBE(k) do {} while (0)
#endif

__host__ __device__ constexpr size_t dcl_smem(int G, int CW, int S, int CL) {
  return (size_t)S * 2 * DCL_PAGE * 2 + sizeof(float) * (size_t)(CW + CL) * G * DCL_ST;
}

// DCL_S: ring stages (one page of K and V each); all of a CTA's pages are
// requested before the PDL wait when they fit the ring
template <int G, int DCL_CL, int DCL_CW, int DCL_S>
__global__ void __launch_bounds__((DCL_CW + 1) * 32)
    attn_decode_cl_kernel(const __nv_bfloat16* __restrict__ qkv, int rs,
                          __nv_bfloat16* __restrict__ kpool, __nv_bfloat16* __restrict__ vpool,
                          const int32_t* __restrict__ tables, int max_blocks,
                          const int32_t* __restrict__ ctx_lens, float log2_theta,
                          const float* __restrict__ alibi, int H, int Hkv, float scale_log2,
                          __nv_bfloat16* __restrict__ out, int trig) {
  constexpr int DCL_THREADS = (DCL_CW + 1) * 32;
  // GQA groups (G > 2): the consumer warps split the group's HEADS (GW each)
  // and every warp walks every page, instead of splitting the pages
  constexpr bool HS = G > 2;
  constexpr int GW = HS ? G / DCL_CW : G;
  static_assert(!HS || G % DCL_CW == 0, "head split needs G % warps == 0");
  extern __shared__ __align__(128) uint8_t dsm_raw[];
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(dsm_raw);         // [S][K|V][PAGE]
  float* wst = reinterpret_cast<float*>(ring + (size_t)DCL_S * 2 * DCL_PAGE);  // [CW][G][ST]
  float* inbox = wst + DCL_CW * G * DCL_ST;         // rank 0: [CL][G][ST] records of the CTAs
  __shared__ uint64_t full[DCL_S], empty[DCL_S];
  __shared__ uint64_t merge_bar;
  __shared__ __align__(16) float pw[DCL_CW * GW * 16];   // per warp: p of the current page
  ATTN_PROBE(0);
  const int r = blockIdx.x;             // cluster rank (cluster (DCL_CL,1,1), gridDim.x == DCL_CL)
  const int kh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < DCL_S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], HS ? DCL_CW : 1);
    }
    mbar_init(&merge_bar, (DCL_CL - 1) * (DCL_CW + 1));   // one arrive per warp of each peer
    fence_barrier_init();
  }
  __syncthreads();
  cluster_arrive_relaxed();            // matched by cluster_wait() before the record push
  const int32_t* trow = tables + (size_t)b * max_blocks;
  const int cur = __ldg(ctx_lens + b);      // written >= 2 launches back (decode_advance)
  const int L = cur + 1;                     // attention length incl. the current token
  const int npg = (L + 15) >> 4;
  const int pp = (npg + DCL_CL - 1) / DCL_CL;
  const int pg0 = r * pp;
  const int nmy = max(0, min(npg, pg0 + pp) - pg0);
  constexpr uint32_t kTile = DCL_PAGE * 2;   // bytes of one page of K (or V)

  if (warp == DCL_CW) {
    // ------------------------------------------------ producer (one lane)
    if (lane == 0) {
      auto issue = [&](int i) {
        const int st = i % DCL_S;
        const int blk = __ldg(trow + pg0 + i);
        const size_t src = ((size_t)blk * Hkv + kh) * DCL_PAGE;
        mbar_arrive_expect_tx(&full[st], 2 * kTile);
        bulk_g2s(ring + (size_t)(2 * st) * DCL_PAGE, kpool + src, kTile, &full[st]);
        bulk_g2s(ring + (size_t)(2 * st + 1) * DCL_PAGE, vpool + src, kTile, &full[st]);
      };
      const int pre = min(nmy, DCL_S);
      for (int i = 0; i < pre; ++i) issue(i);     // cached pages: before the PDL wait
      pdl_wait();
      for (int i = DCL_S; i < nmy; ++i) {
        mbar_wait_sleep(&empty[i % DCL_S], ((i / DCL_S) - 1) & 1);
        issue(i);
      }
      if (trig) pdl_launch_dependents();
    }
  } else {
    // ------------------------------------------------ consumers
    const int half = lane >> 4, hl = lane & 15;
    const float fpos = (float)cur;
    // RoPE angles of this lane's dims at position cur: ctx is known before
    // the dependency wait, so the sincos work overlaps the QKV projection
    float rsn[4], rcs[4];
    if (!alibi) rope_sincos4(rsn, rcs, 4 * hl, fpos, log2_theta);
    pdl_wait();                                   // q / current k,v from the QKV projection
    ATTN_PROBE(1);
    const __nv_bfloat16* qrow = qkv + (size_t)b * rs;
    // lane hl holds dims [4hl, 4hl+4) and [64+4hl, 64+4hl+4): its RoPE pairs
    const int g0 = HS ? warp * GW : 0;         // first head of this warp
    float q[GW][8];
    float sl[GW];
#pragma unroll
    for (int g = 0; g < GW; ++g) {
      const __nv_bfloat16* hp = qrow + (size_t)(kh * G + g0 + g) * DA_D;
      const uint2 ql = *reinterpret_cast<const uint2*>(hp + 4 * hl);
      const uint2 qh = *reinterpret_cast<const uint2*>(hp + 64 + 4 * hl);
      const float2 l0 = bf2_to_f2(ql.x), l1 = bf2_to_f2(ql.y);
      const float2 h0 = bf2_to_f2(qh.x), h1 = bf2_to_f2(qh.y);
      float lo[4] = {l0.x, l0.y, l1.x, l1.y}, hi[4] = {h0.x, h0.y, h1.x, h1.y};
      if (!alibi) {
        rope_apply4(lo, hi, rsn, rcs);
#pragma unroll
        for (int j = 0; j < 4; ++j) {            // rotated q is stored in bf16 (two-kernel path)
          lo[j] = __bfloat162float(__float2bfloat16(lo[j]));
          hi[j] = __bfloat162float(__float2bfloat16(hi[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        q[g][j] = lo[j] * scale_log2;
        q[g][4 + j] = hi[j] * scale_log2;
      }
      sl[g] = alibi ? alibi[kh * G + g0 + g] * 1.4426950408889634f : 0.f;
    }
    // the current token: its page's owner warp RoPEs k, appends k/v to the
    // pool (half 0: k, half 1: v) and keeps the rows to patch the staged page
    const int cpg = cur >> 4;
    const bool has_cur = cpg >= pg0 && cpg < pg0 + nmy;
    const bool own = has_cur && (HS ? warp == 0 : ((cpg - pg0) % DCL_CW) == warp);
    uint2 cur_lo = make_uint2(0, 0), cur_hi = make_uint2(0, 0);
    if (own) {
      const __nv_bfloat16* src = qrow + (size_t)(half == 0 ? H + kh : H + Hkv + kh) * DA_D;
      const uint2 a = *reinterpret_cast<const uint2*>(src + 4 * hl);
      const uint2 c = *reinterpret_cast<const uint2*>(src + 64 + 4 * hl);
      if (half == 0 && !alibi) {
        const float2 a0 = bf2_to_f2(a.x), a1 = bf2_to_f2(a.y);
        const float2 c0 = bf2_to_f2(c.x), c1 = bf2_to_f2(c.y);
        float lo[4] = {a0.x, a0.y, a1.x, a1.y}, hi[4] = {c0.x, c0.y, c1.x, c1.y};
        rope_apply4(lo, hi, rsn, rcs);
        cur_lo = make_uint2(f2_to_bf2(lo[0], lo[1]), f2_to_bf2(lo[2], lo[3]));
        cur_hi = make_uint2(f2_to_bf2(hi[0], hi[1]), f2_to_bf2(hi[2], hi[3]));
      } else {
        cur_lo = a;
        cur_hi = c;
      }
      const int slot = __ldg(trow + cpg) * 16 + (cur & 15);
      const size_t gdst = (((size_t)(slot >> 4) * Hkv + kh) * 16 + (slot & 15)) * DA_D;
      __nv_bfloat16* pool = half == 0 ? kpool : vpool;
      *reinterpret_cast<uint2*>(pool + gdst + 4 * hl) = cur_lo;
      *reinterpret_cast<uint2*>(pool + gdst + 64 + 4 * hl) = cur_hi;
    }
    float m[GW], l[GW], o[GW][4];
#pragma unroll
    for (int g = 0; g < GW; ++g) {
      m[g] = -INFINITY;
      l[g] = 0.f;
      o[g][0] = o[g][1] = o[g][2] = o[g][3] = 0.f;
    }
    ATTN_PROBE(2);
    for (int i = HS ? 0 : warp; i < nmy; i += HS ? 1 : DCL_CW) {
      const int st = i % DCL_S;
      mbar_wait(&full[st], (i / DCL_S) & 1);
      if (i == 0) ATTN_PROBE(3);
      __nv_bfloat16* ks = ring + (size_t)(2 * st) * DCL_PAGE;
      __nv_bfloat16* vs = ks + DCL_PAGE;
      const int t0 = (pg0 + i) * 16;
      if (pg0 + i == cpg) {                      // patch the current token's rows
        if (own) {
          __nv_bfloat16* row = (half == 0 ? ks : vs) + (cur - t0) * DA_D;
          *reinterpret_cast<uint2*>(row + 4 * hl) = cur_lo;
          *reinterpret_cast<uint2*>(row + 64 + 4 * hl) = cur_hi;
        }
        if constexpr (HS)      // every consumer warp reads this page: wait for the patch
          asm volatile("bar.sync 1, %0;" ::"n"(DCL_CW * 32) : "memory");
        else
          __syncwarp();
      }
      const int valid = min(16, L - t0);
      float sc[GW][8];
#pragma unroll
      for (int it = 0; it < 8; ++it) {          // token 2*it + half
        const int t = 2 * it + half;
        const __nv_bfloat16* kr = ks + t * DA_D;
        const uint2 a = *reinterpret_cast<const uint2*>(kr + 4 * hl);
        const uint2 c = *reinterpret_cast<const uint2*>(kr + 64 + 4 * hl);
        const float2 a0 = bf2_to_f2(a.x), a1 = bf2_to_f2(a.y);
        const float2 c0 = bf2_to_f2(c.x), c1 = bf2_to_f2(c.y);
        const float kf[8] = {a0.x, a0.y, a1.x, a1.y, c0.x, c0.y, c1.x, c1.y};
#pragma unroll
        for (int g = 0; g < GW; ++g) {
          float d = q[g][0] * kf[0];
#pragma unroll
          for (int j = 1; j < 8; ++j) d = fmaf(q[g][j], kf[j], d);
          sc[g][it] = d;
        }
      }
      // reduce-scatter across the 16 lanes of a half (xor 8, 4, 2, then 1):
      // the same pairwise sums as a full butterfly per token, but 8 shuffles
      // instead of 32 — lane hl ends with token 2*(hl >> 1) + half
#pragma unroll
      for (int g = 0; g < GW; ++g) {
        const bool b3 = hl & 8, b2 = hl & 4, b1 = hl & 2;
        float r4[4], r2[2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float keep = b3 ? sc[g][4 + j] : sc[g][j];
          const float send = b3 ? sc[g][j] : sc[g][4 + j];
          r4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float keep = b2 ? r4[2 + j] : r4[j];
          const float send = b2 ? r4[j] : r4[2 + j];
          r2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        float v;
        {
          const float keep = b1 ? r2[1] : r2[0];
          const float send = b1 ? r2[0] : r2[1];
          v = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        const int t = 2 * (hl >> 1) + half;
        v = t < valid ? fmaf(sl[g], (float)(t0 + t - cur), v) : -INFINITY;
        float mx = v;
#pragma unroll
        for (int sh = 2; sh < 32; sh <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, sh));
        const float mn = fmaxf(m[g], mx);
        const float corr = m[g] == -INFINITY ? 0.f : exp2f(m[g] - mn);
        const float e = exp2f(v - mn);
        float ps = (hl & 1) ? 0.f : e;          // each token once
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, sh);
        l[g] = l[g] * corr + ps;
        m[g] = mn;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[g][j] *= corr;
        // p of every token of the page to this warp's smem row (broadcast reads below)
        if (!(hl & 1)) pw[(warp * GW + g) * 16 + t] = e;
      }
      __syncwarp();
      // P.V: lane owns dims [4*lane, 4*lane+4)
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        float4 p4[GW];
#pragma unroll
        for (int g = 0; g < GW; ++g)
          p4[g] = *reinterpret_cast<const float4*>(pw + (warp * GW + g) * 16 + 4 * t4);
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const int t = 4 * t4 + tt;
          const uint2 vv = *reinterpret_cast<const uint2*>(vs + t * DA_D + 4 * lane);
          const float2 v0 = bf2_to_f2(vv.x), v1 = bf2_to_f2(vv.y);
#pragma unroll
          for (int g = 0; g < GW; ++g) {
            const float pt = tt == 0 ? p4[g].x : tt == 1 ? p4[g].y : tt == 2 ? p4[g].z : p4[g].w;
            o[g][0] = fmaf(pt, v0.x, o[g][0]);
            o[g][1] = fmaf(pt, v0.y, o[g][1]);
            o[g][2] = fmaf(pt, v1.x, o[g][2]);
            o[g][3] = fmaf(pt, v1.y, o[g][3]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    ATTN_PROBE(4);
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {          // heads this warp does not own: empty
      const int g = gg - g0;
      const bool mine = g >= 0 && g < GW;
      float* w = wst + ((size_t)warp * G + gg) * DCL_ST;
      float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
      float mv = -INFINITY, lv = 0.f;
#pragma unroll
      for (int h = 0; h < GW; ++h)
        if (h == g) {
          v4 = make_float4(o[h][0], o[h][1], o[h][2], o[h][3]);
          mv = m[h];
          lv = l[h];
        }
      *reinterpret_cast<float4*>(w + 4 * lane) = v4;
      if (lane == 0) {
        w[DA_D] = mine ? mv : -INFINITY;
        w[DA_D + 1] = mine ? lv : 0.f;
      }
    }
  }
  __syncthreads();
  // ---- combine the consumer warps (fixed order) into this CTA's record and
  // PUSH it into rank 0's inbox (st.shared::cluster); one release arrive on
  // rank 0's merge barrier per warp, then non-zero ranks exit at once
  ATTN_PROBE(5);
  cluster_wait();                      // rank 0's merge barrier is initialised
  const uint32_t inbox_local = smem_u32(inbox);
  for (int idx = threadIdx.x; idx < G * DA_D; idx += DCL_THREADS) {
    const int g = idx / DA_D, d = idx % DA_D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DCL_CW; ++w) M = fmaxf(M, wst[(w * G + g) * DCL_ST + DA_D]);
    float O = 0.f, Ls = 0.f;
#pragma unroll
    for (int w = 0; w < DCL_CW; ++w) {
      const float* ww = wst + (w * G + g) * DCL_ST;
      const float f = ww[DA_D] == -INFINITY ? 0.f : exp2f(ww[DA_D] - M);
      O = fmaf(f, ww[d], O);
      Ls = fmaf(f, ww[DA_D + 1], Ls);
    }
    const uint32_t dst = inbox_local + (uint32_t)(((r * G + g) * DCL_ST + d) * 4);
    if (r == 0) {
      inbox[(g * DCL_ST) + d] = O;
      if (d == 0) {
        inbox[g * DCL_ST + DA_D] = M;
        inbox[g * DCL_ST + DA_D + 1] = Ls;
      }
    } else {
      const uint32_t rd = mapa(dst, 0);
      st_dsmem(rd, O);
      if (d == 0) {
        st_dsmem(rd + (DA_D - d) * 4, M);
        st_dsmem(rd + (DA_D + 1 - d) * 4, Ls);
      }
    }
  }
  if (r != 0) {
    // each warp publishes its lanes' stores with one release arrive
    // (cumulative after __syncwarp): no cluster fence, no CTA barrier
    __syncwarp();
    if (lane == 0) mbar_arrive_remote(mapa(smem_u32(&merge_bar), 0));
    ATTN_PROBE(6);
    return;
  }
  ATTN_PROBE(6);
  __syncthreads();
  mbar_wait_cluster(&merge_bar, 0);    // every peer's record landed in the inbox
  ATTN_PROBE(7);
  __shared__ float fac[DCL_CL * G];
  __shared__ float ltot[G];
  for (int g = threadIdx.x; g < G; g += DCL_THREADS) {
    float M = -INFINITY;
#pragma unroll
    for (int p = 0; p < DCL_CL; ++p) M = fmaxf(M, inbox[(p * G + g) * DCL_ST + DA_D]);
    float Ls = 0.f;
#pragma unroll
    for (int p = 0; p < DCL_CL; ++p) {
      const float mp = inbox[(p * G + g) * DCL_ST + DA_D];
      const float f = mp == -INFINITY ? 0.f : exp2f(mp - M);
      fac[p * G + g] = f;
      Ls = fmaf(f, inbox[(p * G + g) * DCL_ST + DA_D + 1], Ls);
    }
    ltot[g] = Ls;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * DA_D; idx += DCL_THREADS) {
    const int g = idx / DA_D, d = idx % DA_D;
    float O = 0.f;
#pragma unroll
    for (int p = 0; p < DCL_CL; ++p) O = fmaf(fac[p * G + g], inbox[(p * G + g) * DCL_ST + d], O);
    out[((size_t)b * H + kh * G + g) * DA_D + d] = __float2bfloat16(O / ltot[g]);
  }
  ATTN_PROBE(8);
}

// ---------------------------------------------------------------- decode, MMA
// Tensor-core decode attention (block_size 16, partition 128): the G query
// heads of a kv group form the rows of a 16-row mma.sync A tile (rows >= G
// zero), so S = Q.K^T and O = P.V run as m16n8k16 MMAs straight from the
// staged pages (ldmatrix / ldmatrix.trans) instead of shuffle-reduced dot
// products — the GQA (G = 8) case was CUDA-core bound at ~0.1-0.9 TB/s.
// Warp w owns tokens [32w, 32w+32) of the partition (2 pages) and waits only
// for ITS pages (one K and one V mbarrier per warp), so compute starts while
// later pages are still landing; warps combine (max, sum, O) through shared
// memory, partitions through the fused split-K merge.
constexpr int DM_WARPS = 4, DM_PT = 128, DM_WT = 32, DM_QS = DA_D + 8;

constexpr int DC_MAXQT = 512;     // chunked prefill: up to 8192 query rows per chunk

// CLN > 0: the NP = CLN partitions of a (b, kv head) form one thread-block
// cluster and merge through rank 0's shared-memory inbox (push-merge, as the
// cluster-streaming kernel does) instead of global partials + ticket.
template <bool STEP, int WT, int CLN = 0>   // WT = tokens per warp (32: partition 128, 16: 64)
__global__ void __launch_bounds__(DM_WARPS * 32)
    attn_decode_mma_kernel(const __nv_bfloat16* __restrict__ qkv, int rs,
                           __nv_bfloat16* __restrict__ kpool, __nv_bfloat16* __restrict__ vpool,
                           const int32_t* __restrict__ tables, int max_blocks,
                           const int32_t* __restrict__ ctx_lens, const int32_t* __restrict__ pos,
                           const int32_t* __restrict__ slots, float log2_theta,
                           const float* __restrict__ alibi, int H, int Hkv, float scale_log2,
                           float* __restrict__ ws, int* __restrict__ tickets,
                           __nv_bfloat16* __restrict__ out, int trig) {
  constexpr int BS = 16;
  constexpr int PT = DM_WARPS * WT, PPW = WT / BS;   // partition tokens, pages per warp
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(dsm);          // [128][128]
  __nv_bfloat16* sv = sk + PT * DA_D;                               // [128][128]
  __nv_bfloat16* sq = sv + PT * DA_D;                               // [16][DM_QS]
  float* sml = reinterpret_cast<float*>(sq + 16 * DM_QS);              // [4][8][2]
  float* so = sml + DM_WARPS * 8 * 2;                                  // [4][G][128]
  float* inbox = so + DM_WARPS * (H / Hkv) * DA_D;         // CLN: rank 0 [CLN][G][DCL_ST]
  float* rec = inbox + CLN * (H / Hkv) * DCL_ST;           // CLN: this CTA's [G][DA_D + 2]
  __shared__ uint64_t kbar[DM_WARPS], vbar[DM_WARPS];
  __shared__ uint64_t merge_bar;
  __shared__ int s_last;
  __shared__ __align__(16) __nv_bfloat16 scur[2][DA_D];
  __shared__ float swf[DM_WARPS * 8], swM[8], swL[8];   // per (warp, head) combine factors
  ATTN_PROBE(0);
  const int p = blockIdx.x, kh = blockIdx.y, b = blockIdx.z;
  const int NP = gridDim.x;
  const int G = H / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  auto wsp = [&](int gh, int pp) {
    return ws + (((size_t)b * H + gh) * NP + pp) * (DA_D + 2);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < DM_WARPS; ++i) {
      mbar_init(&kbar[i], 1);
      mbar_init(&vbar[i], 1);
    }
    // one release arrive per warp of every other CTA (their records land
    // straight in this CTA's inbox from the warp-combine loop)
    if constexpr (CLN > 0) mbar_init(&merge_bar, (CLN - 1) * DM_WARPS);
    fence_barrier_init();
  }
  __syncthreads();
  if constexpr (CLN > 0) cluster_arrive_relaxed();   // matched before the record push
  const int32_t* trow = tables + (size_t)b * max_blocks;
  int L, cur;
  if constexpr (STEP) {
    const int c = __ldg(ctx_lens + b);
    L = c + 1;
    cur = c;
  } else {
    pdl_wait();
    L = ctx_lens[b];
    cur = pos ? pos[b] : -1;
  }
  const int t0 = p * PT;
  const int t1 = min(L, t0 + PT);
  const int ntok = t1 - t0;
  if (warp == 0 && ntok > 0) {
    // pages of cached tokens; page j feeds warp j/2's barriers
    const int cend = cur >= 0 ? min(t1, cur) : t1;
    const int nblk = (max(0, cend - t0) + BS - 1) / BS;
    constexpr uint32_t tile = BS * DA_D * 2;
    if (lane < DM_WARPS) {
      const int np = min(max(nblk - PPW * lane, 0), PPW);
      mbar_arrive_expect_tx(&kbar[lane], tile * np);
      mbar_arrive_expect_tx(&vbar[lane], tile * np);
    }
    __syncwarp();
    if (lane < nblk) {
      const int blk = __ldg(trow + t0 / BS + lane);
      const size_t gofs = ((size_t)blk * Hkv + kh) * BS * DA_D;
      bulk_g2s(sk + (size_t)lane * BS * DA_D, kpool + gofs, tile, &kbar[lane / PPW]);
      bulk_g2s(sv + (size_t)lane * BS * DA_D, vpool + gofs, tile, &vbar[lane / PPW]);
    }
  }
  // RoPE angles of this thread's dims (i0 = (tid % 16) * 4 in the q tile and
  // the current-token rows below) at position cur, before the dependency wait
  float rsn[4], rcs[4];
  if (STEP && cur >= 0 && !alibi) rope_sincos4(rsn, rcs, (threadIdx.x & 15) * 4, (float)cur, log2_theta);
  if constexpr (STEP) pdl_wait();
  ATTN_PROBE(1);

  if (ntok > 0) {
    const int qpos = cur >= 0 ? cur : L - 1;
    const __nv_bfloat16* qrow = qkv + (size_t)b * rs;
    const float fpos = (float)cur;
    // q tile: rows = the group's heads (RoPE'd, rounded to bf16), rows >= G zero
    for (int i = threadIdx.x; i < 16 * (DA_D / 8); i += DM_WARPS * 32) {
      const int gi = i / (DA_D / 8), i0 = (i % (DA_D / 8)) * 4;
      uint2 lo2 = make_uint2(0, 0), hi2 = make_uint2(0, 0);
      if (gi < G) {
        const __nv_bfloat16* hp = qrow + (kh * G + gi) * DA_D;
        const uint2 ql = *reinterpret_cast<const uint2*>(hp + i0);
        const uint2 qh = *reinterpret_cast<const uint2*>(hp + 64 + i0);
        if (cur >= 0 && !alibi) {
          const float2 l0 = bf2_to_f2(ql.x), l1 = bf2_to_f2(ql.y);
          const float2 h0 = bf2_to_f2(qh.x), h1 = bf2_to_f2(qh.y);
          float lo[4] = {l0.x, l0.y, l1.x, l1.y}, hi[4] = {h0.x, h0.y, h1.x, h1.y};
          if (STEP)
            rope_apply4(lo, hi, rsn, rcs);        // i0 == (tid % 16) * 4
          else
            rope4(lo, hi, i0, fpos, log2_theta);
          lo2 = make_uint2(f2_to_bf2(lo[0], lo[1]), f2_to_bf2(lo[2], lo[3]));
          hi2 = make_uint2(f2_to_bf2(hi[0], hi[1]), f2_to_bf2(hi[2], hi[3]));
        } else {
          lo2 = ql;
          hi2 = qh;
        }
      }
      *reinterpret_cast<uint2*>(sq + gi * DM_QS + i0) = lo2;
      *reinterpret_cast<uint2*>(sq + gi * DM_QS + 64 + i0) = hi2;
    }
    // current token: rotate k, append k/v to the pool, stage in smem
    const bool own_cur = cur >= t0 && cur < t1;
    if (own_cur && threadIdx.x < 16) {
      const int i0 = threadIdx.x * 4;
      const __nv_bfloat16* kp = qrow + (H + kh) * DA_D;
      const __nv_bfloat16* vp = qrow + (H + Hkv + kh) * DA_D;
      const uint2 kl = *reinterpret_cast<const uint2*>(kp + i0);
      const uint2 khi = *reinterpret_cast<const uint2*>(kp + 64 + i0);
      const float2 a0 = bf2_to_f2(kl.x), a1 = bf2_to_f2(kl.y);
      const float2 c0 = bf2_to_f2(khi.x), c1 = bf2_to_f2(khi.y);
      float lo[4] = {a0.x, a0.y, a1.x, a1.y}, hi[4] = {c0.x, c0.y, c1.x, c1.y};
      if (!alibi) {
        if (STEP)
          rope_apply4(lo, hi, rsn, rcs);          // tid < 16: i0 == tid * 4
        else
          rope4(lo, hi, i0, fpos, log2_theta);
      }
      const int slot = STEP ? __ldg(trow + cur / BS) * BS + (cur & (BS - 1)) : slots[b];
      const size_t go = (((size_t)(slot / BS) * Hkv + kh) * BS + (slot & (BS - 1))) * DA_D;
      const uint2 klo = make_uint2(f2_to_bf2(lo[0], lo[1]), f2_to_bf2(lo[2], lo[3]));
      const uint2 khh = make_uint2(f2_to_bf2(hi[0], hi[1]), f2_to_bf2(hi[2], hi[3]));
      const uint2 vlo = *reinterpret_cast<const uint2*>(vp + i0);
      const uint2 vhi = *reinterpret_cast<const uint2*>(vp + 64 + i0);
      *reinterpret_cast<uint2*>(kpool + go + i0) = klo;
      *reinterpret_cast<uint2*>(kpool + go + 64 + i0) = khh;
      *reinterpret_cast<uint2*>(vpool + go + i0) = vlo;
      *reinterpret_cast<uint2*>(vpool + go + 64 + i0) = vhi;
      *reinterpret_cast<uint2*>(&scur[0][i0]) = klo;
      *reinterpret_cast<uint2*>(&scur[0][64 + i0]) = khh;
      *reinterpret_cast<uint2*>(&scur[1][i0]) = vlo;
      *reinterpret_cast<uint2*>(&scur[1][64 + i0]) = vhi;
    }
    __syncthreads();
    ATTN_PROBE(2);

    const int wt0 = warp * WT;
    const bool cur_here = own_cur && cur - t0 >= wt0 && cur - t0 < wt0 + WT;
    if (wt0 < ntok) {   // warp-uniform
      mbar_wait(&kbar[warp], 0);
      ATTN_PROBE(3);
      if (cur_here && lane < 16)
        reinterpret_cast<uint4*>(sk + (size_t)(cur - t0) * DA_D)[lane] =
            reinterpret_cast<const uint4*>(scur[0])[lane];
      __syncwarp();
      // S = Q K^T (16 heads-rows x 32 tokens)
      float s[WT / 8][4];
#pragma unroll
      for (int i = 0; i < WT / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      const uint32_t sq_u = smem_u32(sq), sk_u = smem_u32(sk), sv_u = smem_u32(sv);
#pragma unroll
      for (int kk = 0; kk < DA_D / 16; ++kk) {
        uint32_t qf[4];
        ldsm_x4(sq_u + ((lane & 15) * DM_QS + (kk * 2 + (lane >> 4)) * 8) * 2, qf[0], qf[1],
                qf[2], qf[3]);
#pragma unroll
        for (int np = 0; np < WT / 16; ++np) {
          const int key = wt0 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int chunk = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sk_u + (key * DA_D + chunk * 8) * 2, b0, b1, b2, b3);
          mma_bf16(s[2 * np], qf, b0, b1);
          mma_bf16(s[2 * np + 1], qf, b2, b3);
        }
      }
      // row g = head g of the group (rows g+8 are padding)
      const float sl = (alibi && g < G) ? alibi[kh * G + g] * 1.4426950408889634f : 0.f;
      float m = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < WT / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int tok = wt0 + nt * 8 + 2 * t + e;
          const float v = tok < ntok ? fmaf(sl, (float)(t0 + tok - qpos), s[nt][e] * scale_log2)
                                     : -INFINITY;
          s[nt][e] = v;
          m = fmaxf(m, v);
        }
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      float l = 0.f;
      uint32_t pf[WT / 16][4];
#pragma unroll
      for (int nt = 0; nt < WT / 8; ++nt) {
        const float e0 = exp2f(s[nt][0] - m), e1 = exp2f(s[nt][1] - m);
        l += e0 + e1;
        const uint32_t pk = f2_to_bf2(e0, e1);
        if ((nt & 1) == 0) {
          pf[nt >> 1][0] = pk;
          pf[nt >> 1][1] = 0u;
        } else {
          pf[nt >> 1][2] = pk;
          pf[nt >> 1][3] = 0u;
        }
      }
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      mbar_wait(&vbar[warp], 0);
      ATTN_PROBE(4);
      if (cur_here && lane < 16)
        reinterpret_cast<uint4*>(sv + (size_t)(cur - t0) * DA_D)[lane] =
            reinterpret_cast<const uint4*>(scur[1])[lane];
      // rows past the context hold stale smem / unwritten pool bytes: P is 0
      // there, but 0 * NaN is not, so zero them
      for (int i = max(ntok - wt0, 0) * 16 + lane; i < WT * 16; i += 32)
        reinterpret_cast<uint4*>(sv + (size_t)wt0 * DA_D)[i] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      // O = P V (16 x 128)
      float o[16][4];
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < WT / 16; ++ks) {
#pragma unroll
        for (int dp = 0; dp < 8; ++dp) {
          const int key = wt0 + ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int chunk = dp * 2 + (lane >> 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sv_u + (key * DA_D + chunk * 8) * 2, b0, b1, b2, b3);
          mma_bf16(o[2 * dp], pf[ks], b0, b1);
          mma_bf16(o[2 * dp + 1], pf[ks], b2, b3);
        }
      }
      if (g < G) {
        float* dst = so + ((size_t)warp * G + g) * DA_D;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(dst + nt * 8 + 2 * t) = make_float2(o[nt][0], o[nt][1]);
        if (t == 0) {
          sml[(warp * 8 + g) * 2] = m;
          sml[(warp * 8 + g) * 2 + 1] = l;
        }
      }
    } else if (t == 0 && g < G) {
      sml[(warp * 8 + g) * 2] = -INFINITY;
      sml[(warp * 8 + g) * 2 + 1] = 0.f;
    }
    __syncthreads();
    ATTN_PROBE(5);
    if (trig) pdl_launch_dependents();
    // cluster form: rank 0's merge barrier is initialised (cluster_arrive at
    // the start) before any record is pushed into its inbox
    if constexpr (CLN > 0) cluster_wait();
    const uint32_t inbox0 = CLN > 0 ? mapa(smem_u32(inbox), 0) : 0u;
    // combine the warps' partial softmax states: the per-(warp, head)
    // factors once, then one FMA per warp and element
    if (threadIdx.x < G) {
      const int gi = threadIdx.x;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < DM_WARPS; ++w) M = fmaxf(M, sml[(w * 8 + gi) * 2]);
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < DM_WARPS; ++w) {
        const float mw = sml[(w * 8 + gi) * 2];
        const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
        swf[w * 8 + gi] = f;
        if (mw != -INFINITY) l += f * sml[(w * 8 + gi) * 2 + 1];
      }
      swM[gi] = M;
      swL[gi] = l;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * DA_D; i += DM_WARPS * 32) {
      const int gi = i / DA_D, d = i % DA_D;
      const float M = swM[gi], l = swL[gi];
      float o = 0.f;
#pragma unroll
      for (int w = 0; w < DM_WARPS; ++w) {
        if (sml[(w * 8 + gi) * 2] == -INFINITY) continue;   // warp had no tokens
        o += swf[w * 8 + gi] * so[((size_t)w * G + gi) * DA_D + d];
      }
      if (CLN == 0 && NP == 1) {
        out[((size_t)b * H + kh * G + gi) * DA_D + d] = __float2bfloat16(o / l);
        continue;
      }
      if constexpr (CLN > 0) {
        // this partition's record goes straight into rank 0's inbox
        const uint32_t slot = (uint32_t)(p * G + gi) * DCL_ST;
        if (p == 0) {
          inbox[slot + d] = o;
          if (d == 0) {
            inbox[slot + DA_D] = M;
            inbox[slot + DA_D + 1] = l;
          }
        } else {
          st_dsmem(inbox0 + (slot + d) * 4u, o);
          if (d == 0) {
            st_dsmem(inbox0 + (slot + DA_D) * 4u, M);
            st_dsmem(inbox0 + (slot + DA_D + 1) * 4u, l);
          }
        }
        continue;
      }
      float* wo = wsp(kh * G + gi, p);
      wo[d] = o;
      if (d == 0) {
        wo[DA_D] = M;
        wo[DA_D + 1] = l;
      }
    }
    if (CLN == 0 && NP == 1) return;
  } else {
    if (trig) pdl_launch_dependents();
    if constexpr (CLN > 0) {
      cluster_wait();
      const uint32_t inbox0 = mapa(smem_u32(inbox), 0);
      for (int i = threadIdx.x; i < G * (DA_D + 2); i += DM_WARPS * 32) {
        const int gi = i / (DA_D + 2), d = i % (DA_D + 2);
        const uint32_t slot = (uint32_t)(p * G + gi) * DCL_ST + d;
        const float v = d == DA_D ? -INFINITY : 0.f;
        if (p == 0)
          inbox[slot] = v;
        else
          st_dsmem(inbox0 + slot * 4u, v);
      }
    } else if (threadIdx.x < G) {
      float* w = wsp(kh * G + threadIdx.x, p);
      w[DA_D] = -INFINITY;
      w[DA_D + 1] = 0.f;
    }
  }
  if constexpr (CLN > 0) {
    // ---- records are in rank 0's inbox; every warp of ranks > 0 publishes
    // its stores with one release arrive (cumulative over the warp's lanes
    // after __syncwarp), rank 0 merges
    __syncwarp();
    ATTN_PROBE(6);
    if (p != 0) {
      if (lane == 0) mbar_arrive_remote(mapa(smem_u32(&merge_bar), 0));
      ATTN_PROBE(7);
      return;
    }
    __syncthreads();
    mbar_wait_cluster(&merge_bar, 0);
    ATTN_PROBE(7);
    float* fac = rec;                     // [CLN][G] merge factors
    float* ltot = rec + CLN * G;          // [G]
    if (G * CLN <= DM_WARPS * 32) {
      // one (head, partition) per thread; CLN consecutive lanes per head
      const int i = threadIdx.x, gi = i / CLN, q = i % CLN;
      const bool on = i < G * CLN;
      const float mq = on ? inbox[(q * G + gi) * DCL_ST + DA_D] : -INFINITY;
      float Mx = mq;
#pragma unroll
      for (int o = CLN / 2; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
      const float f = (!on || mq == -INFINITY) ? 0.f : exp2f(mq - Mx);
      float Ls = on ? f * inbox[(q * G + gi) * DCL_ST + DA_D + 1] : 0.f;
#pragma unroll
      for (int o = CLN / 2; o > 0; o >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, o);
      if (on) {
        fac[q * G + gi] = f;
        if (q == 0) ltot[gi] = Ls;
      }
    } else if (threadIdx.x < G) {
      const int gi = threadIdx.x;
      float Mx = -INFINITY;
      for (int q = 0; q < CLN; ++q) Mx = fmaxf(Mx, inbox[(q * G + gi) * DCL_ST + DA_D]);
      float Ls = 0.f;
      for (int q = 0; q < CLN; ++q) {
        const float mq = inbox[(q * G + gi) * DCL_ST + DA_D];
        const float f = mq == -INFINITY ? 0.f : exp2f(mq - Mx);
        fac[q * G + gi] = f;
        Ls = fmaf(f, inbox[(q * G + gi) * DCL_ST + DA_D + 1], Ls);
      }
      ltot[gi] = Ls;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * DA_D / 4; i += DM_WARPS * 32) {
      const int gi = i / (DA_D / 4), d = (i % (DA_D / 4)) * 4;
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (int q = 0; q < CLN; ++q) {
        const float f = fac[q * G + gi];
        const float4 v = *reinterpret_cast<const float4*>(inbox + (q * G + gi) * DCL_ST + d);
        o.x = fmaf(f, v.x, o.x); o.y = fmaf(f, v.y, o.y);
        o.z = fmaf(f, v.z, o.z); o.w = fmaf(f, v.w, o.w);
      }
      const float il = ltot[gi];
      *reinterpret_cast<uint2*>(out + ((size_t)b * H + kh * G + gi) * DA_D + d) =
          make_uint2(f2_to_bf2(o.x / il, o.y / il), f2_to_bf2(o.z / il, o.w / il));
    }
    ATTN_PROBE(8);
    return;
  }
  // ---- fused split-K merge: the last CTA of (b, kh) combines the partitions
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* tk = tickets + (size_t)b * Hkv + kh;
    const int prev = atomicAdd(tk, 1);
    s_last = prev == NP - 1;
    if (s_last) *tk = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  decode_merge(ws + (size_t)b * H * NP * (DA_D + 2), NP, G, kh, H, reinterpret_cast<float*>(dsm),
               out + (size_t)b * H * DA_D, DM_WARPS * 32);
}

// ---------------------------------------------------------------- chunked prefill
// Causal attention of a prompt CHUNK whose keys live in the paged pool (the
// chunk's own K/V were written there by the QKV GEMM epilogue, earlier chunks'
// by earlier calls): CTA (key partition p, head h, 16-query tile t) computes
// S = Q_t . K_p^T and O = P . V_p with mma.sync exactly like the decode MMA
// kernel, but the 16 A-tile rows are 16 consecutive query positions of one
// head, each with its own causal bound; partitions merge per row through the
// workspace (last CTA of (h, t), fixed order).
template <int DUMMY>
__global__ void __launch_bounds__(DM_WARPS * 32)
    attn_chunk_kernel(const __nv_bfloat16* __restrict__ qkv, int rs, int C, int q_start,
                      const __nv_bfloat16* __restrict__ kpool,
                      const __nv_bfloat16* __restrict__ vpool, const int32_t* __restrict__ trow,
                      int H, int Hkv, float scale_log2, const float* __restrict__ alibi,
                      float* __restrict__ ws, int* __restrict__ tickets,
                      __nv_bfloat16* __restrict__ out) {
  constexpr int BS = 16;
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(dsm);          // [128][128]
  __nv_bfloat16* sv = sk + DM_PT * DA_D;                               // [128][128]
  __nv_bfloat16* sq = sv + DM_PT * DA_D;                               // [16][DM_QS]
  float* sml = reinterpret_cast<float*>(sq + 16 * DM_QS);              // [4][16][2]
  float* so = sml + DM_WARPS * 16 * 2;                                 // [4][16][128]
  __shared__ uint64_t kbar[DM_WARPS], vbar[DM_WARPS];
  __shared__ int s_last;
  const int p = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int NP = gridDim.x;
  const int kh = h / (H / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = qt * 16;                                  // first chunk row of the tile
  const int nrows = min(16, C - r0);
  const int qmax = q_start + r0 + nrows - 1;               // last query position
  const int t0 = p * DM_PT;
  const int L = qmax + 1;                                  // keys this tile may see
  const int t1 = min(L, t0 + DM_PT);
  const int ntok = t1 - t0;
  // partial of (row, partition): ws[((h * nq + qt) * 16 + row) * NP + p][DA_D + 2]
  const int nq = gridDim.z;
  auto wsp = [&](int row, int pp) {
    return ws + ((((size_t)h * nq + qt) * 16 + row) * NP + pp) * (DA_D + 2);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < DM_WARPS; ++i) {
      mbar_init(&kbar[i], 1);
      mbar_init(&vbar[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();          // the chunk's K/V pages and q come from the QKV GEMM
  if (warp == 0 && ntok > 0) {
    const int nblk = (ntok + BS - 1) / BS;
    constexpr uint32_t tile = BS * DA_D * 2;
    if (lane < DM_WARPS) {
      const int np = min(max(nblk - 2 * lane, 0), 2);
      mbar_arrive_expect_tx(&kbar[lane], tile * np);
      mbar_arrive_expect_tx(&vbar[lane], tile * np);
    }
    __syncwarp();
    if (lane < nblk) {
      const int blk = __ldg(trow + t0 / BS + lane);
      const size_t gofs = ((size_t)blk * Hkv + kh) * BS * DA_D;
      bulk_g2s(sk + (size_t)lane * BS * DA_D, kpool + gofs, tile, &kbar[lane >> 1]);
      bulk_g2s(sv + (size_t)lane * BS * DA_D, vpool + gofs, tile, &vbar[lane >> 1]);
    }
  }
  if (ntok > 0) {
    // q tile: 16 consecutive query rows of head h (already RoPE'd), rows past C zero
    for (int i = threadIdx.x; i < 16 * (DA_D / 8); i += DM_WARPS * 32) {
      const int rr = i / (DA_D / 8), c8 = (i % (DA_D / 8)) * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (rr < nrows) v = *reinterpret_cast<const uint4*>(qkv + (size_t)(r0 + rr) * rs + h * DA_D + c8);
      *reinterpret_cast<uint4*>(sq + rr * DM_QS + c8) = v;
    }
    __syncthreads();
    const int wt0 = warp * DM_WT;
    if (wt0 < ntok) {
      mbar_wait(&kbar[warp], 0);
      float s[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      const uint32_t sq_u = smem_u32(sq), sk_u = smem_u32(sk), sv_u = smem_u32(sv);
#pragma unroll
      for (int kk = 0; kk < DA_D / 16; ++kk) {
        uint32_t qf[4];
        ldsm_x4(sq_u + ((lane & 15) * DM_QS + (kk * 2 + (lane >> 4)) * 8) * 2, qf[0], qf[1],
                qf[2], qf[3]);
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          const int key = wt0 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int chunk = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sk_u + (key * DA_D + chunk * 8) * 2, b0, b1, b2, b3);
          mma_bf16(s[2 * np], qf, b0, b1);
          mma_bf16(s[2 * np + 1], qf, b2, b3);
        }
      }
      // rows g (c0,c1) and g+8 (c2,c3): query positions q_start + r0 + row
      const float sl = alibi ? alibi[h] * 1.4426950408889634f : 0.f;
      float m[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int row = g + 8 * hr;
        const int qpos = q_start + r0 + row;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int tok = wt0 + nt * 8 + 2 * t + e;
            const int kpos = t0 + tok;
            const float v = (tok < ntok && kpos <= qpos && row < nrows)
                                ? fmaf(sl, (float)(kpos - qpos), s[nt][2 * hr + e] * scale_log2)
                                : -INFINITY;
            s[nt][2 * hr + e] = v;
            m[hr] = fmaxf(m[hr], v);
          }
        m[hr] = fmaxf(m[hr], __shfl_xor_sync(0xffffffffu, m[hr], 1));
        m[hr] = fmaxf(m[hr], __shfl_xor_sync(0xffffffffu, m[hr], 2));
      }
      float l[2] = {0.f, 0.f};
      uint32_t pf[2][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        float e0 = m[0] == -INFINITY ? 0.f : exp2f(s[nt][0] - m[0]);
        float e1 = m[0] == -INFINITY ? 0.f : exp2f(s[nt][1] - m[0]);
        float e2 = m[1] == -INFINITY ? 0.f : exp2f(s[nt][2] - m[1]);
        float e3 = m[1] == -INFINITY ? 0.f : exp2f(s[nt][3] - m[1]);
        l[0] += e0 + e1;
        l[1] += e2 + e3;
        const uint32_t pk0 = f2_to_bf2(e0, e1), pk1 = f2_to_bf2(e2, e3);
        if ((nt & 1) == 0) {
          pf[nt >> 1][0] = pk0;
          pf[nt >> 1][1] = pk1;
        } else {
          pf[nt >> 1][2] = pk0;
          pf[nt >> 1][3] = pk1;
        }
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 1);
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 2);
      }
      mbar_wait(&vbar[warp], 0);
      for (int i = max(ntok - wt0, 0) * 16 + lane; i < DM_WT * 16; i += 32)
        reinterpret_cast<uint4*>(sv + (size_t)wt0 * DA_D)[i] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      float o[16][4];
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
        for (int dp = 0; dp < 8; ++dp) {
          const int key = wt0 + ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int chunk = dp * 2 + (lane >> 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sv_u + (key * DA_D + chunk * 8) * 2, b0, b1, b2, b3);
          mma_bf16(o[2 * dp], pf[ks], b0, b1);
          mma_bf16(o[2 * dp + 1], pf[ks], b2, b3);
        }
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int row = g + 8 * hr;
        float* dst = so + ((size_t)warp * 16 + row) * DA_D;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(dst + nt * 8 + 2 * t) =
              make_float2(o[nt][2 * hr], o[nt][2 * hr + 1]);
        if (t == 0) {
          sml[(warp * 16 + row) * 2] = m[hr];
          sml[(warp * 16 + row) * 2 + 1] = l[hr];
        }
      }
    } else if (t == 0) {
      sml[(warp * 16 + g) * 2] = -INFINITY;
      sml[(warp * 16 + g) * 2 + 1] = 0.f;
      sml[(warp * 16 + g + 8) * 2] = -INFINITY;
      sml[(warp * 16 + g + 8) * 2 + 1] = 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 16 * DA_D; i += DM_WARPS * 32) {
      const int row = i / DA_D, d = i % DA_D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < DM_WARPS; ++w) M = fmaxf(M, sml[(w * 16 + row) * 2]);
      float o = 0.f, l = 0.f;
#pragma unroll
      for (int w = 0; w < DM_WARPS; ++w) {
        const float mw = sml[(w * 16 + row) * 2];
        if (mw == -INFINITY) continue;
        const float f = exp2f(mw - M);
        o += f * so[((size_t)w * 16 + row) * DA_D + d];
        l += f * sml[(w * 16 + row) * 2 + 1];
      }
      float* wo = wsp(row, p);
      wo[d] = o;
      if (d == 0) {
        wo[DA_D] = M;
        wo[DA_D + 1] = l;
      }
    }
  } else {
    for (int row = threadIdx.x; row < 16; row += DM_WARPS * 32) {
      float* w = wsp(row, p);
      w[DA_D] = -INFINITY;
      w[DA_D + 1] = 0.f;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* tk = tickets + (size_t)h * DC_MAXQT + qt;
    const int prev = atomicAdd(tk, 1);
    s_last = prev == NP - 1;
    if (s_last) *tk = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // merge the partitions of the tile's rows (rows = "heads" of decode_merge)
  // with out row stride H * DA_D: write through a [16][H*128] view
  float* sf = reinterpret_cast<float*>(dsm);
  const int tid = threadIdx.x;
  const float* base = ws + (((size_t)h * nq + qt) * 16) * NP * (DA_D + 2);
  for (int i = tid; i < 16 * NP; i += DM_WARPS * 32) {
    const int row = i / NP, pp = i % NP;
    const float* w = base + ((size_t)row * NP + pp) * (DA_D + 2);
    sf[i] = __ldcg(w + DA_D);
    sf[16 * NP + 16 + i] = __ldcg(w + DA_D + 1);
  }
  __syncthreads();
  for (int row = warp; row < 16; row += DM_WARPS) {
    float M = -INFINITY;
    for (int pp = lane; pp < NP; pp += 32) M = fmaxf(M, sf[row * NP + pp]);
    M = warp_max(M);
    float Ls = 0.f;
    for (int pp = lane; pp < NP; pp += 32) {
      const float mm = sf[row * NP + pp];
      const float f = mm == -INFINITY ? 0.f : exp2f(mm - M);
      Ls += f * sf[16 * NP + 16 + row * NP + pp];
      sf[row * NP + pp] = f;
    }
    Ls = warp_sum(Ls);
    if (lane == 0) sf[16 * NP + row] = Ls;
  }
  __syncthreads();
  for (int i = tid; i < nrows * (DA_D / 4); i += DM_WARPS * 32) {
    const int row = i / (DA_D / 4), d4 = i % (DA_D / 4);
    const float* b = base + (size_t)row * NP * (DA_D + 2) + d4 * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int pp = 0; pp < NP; ++pp) {
      const float f = sf[row * NP + pp];
      const float2 x0 = __ldcg(reinterpret_cast<const float2*>(b + (size_t)pp * (DA_D + 2)));
      const float2 x1 = __ldcg(reinterpret_cast<const float2*>(b + (size_t)pp * (DA_D + 2) + 2));
      acc.x = fmaf(f, x0.x, acc.x); acc.y = fmaf(f, x0.y, acc.y);
      acc.z = fmaf(f, x1.x, acc.z); acc.w = fmaf(f, x1.y, acc.w);
    }
    const float inv = 1.f / sf[16 * NP + row];
    __nv_bfloat16* dst = out + (size_t)(r0 + row) * H * DA_D + h * DA_D + d4 * 4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(f2_to_bf2(acc.x * inv, acc.y * inv),
                                                f2_to_bf2(acc.z * inv, acc.w * inv));
  }
}

}  // namespace swb

using namespace swb;

extern "C" int swb_attn_prefill(const void* qkv, int row_stride, const int32_t* cu_seqlens,
                                int num_seqs, int max_seqlen, int H, int Hkv, int dh,
                                float scale, void* out, uintptr_t stream) {
  SWB_REQUIRE(qkv && cu_seqlens && out, "swb_attn_prefill: null pointer");
  SWB_REQUIRE(dh == PA_D, "swb_attn_prefill: dh must be 128 (got %d)", dh);
  SWB_REQUIRE(H > 0 && Hkv > 0 && H % Hkv == 0, "swb_attn_prefill: bad heads");
  SWB_REQUIRE(row_stride % 8 == 0, "swb_attn_prefill: row_stride %% 8");
  SWB_REQUIRE(num_seqs >= 0 && max_seqlen >= 0, "swb_attn_prefill: bad sizes");
  if (num_seqs == 0 || max_seqlen == 0) return SWB_OK;
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(attn_prefill_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, PA_SMEM));
    attr[dev] = true;
  }
  const int tiles = (max_seqlen + PA_BQ - 1) / PA_BQ;
  dim3 grid(num_seqs * tiles, H);
  {
    const cudaError_t le_ = launch(attn_prefill_kernel, dim3(grid), dim3(PA_THREADS), PA_SMEM, (cudaStream_t)stream,
        
      reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride, cu_seqlens, tiles, H, Hkv,
      scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(out));
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch attn_prefill_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("attn_prefill_kernel");
}

extern "C" size_t swb_attn_decode_workspace(int B, int H, int max_ctx, int partition,
                                            int dh) {
  if (B <= 0 || H <= 0 || max_ctx <= 0 || partition <= 0) return 0;
  const size_t np = (max_ctx + partition - 1) / partition;
  // partials [B][H][NP][dh+2] fp32 + merge tickets [B][H] int32 (zeroed by caller)
  return (size_t)B * H * np * (dh + 2) * sizeof(float) + (size_t)B * H * sizeof(int);
}

template <bool STEP>
static int launch_attn_decode(const void* qkv, int row_stride, void* k_layer, void* v_layer,
                              const int32_t* block_tables, int max_blocks,
                              const int32_t* ctx_lens, const int32_t* positions,
                              const int32_t* slots, float theta, const float* alibi_slopes,
                              int B, int H, int Hkv, int dh, int block_size, float scale,
                              int max_ctx, int partition, void* workspace, void* out,
                              uintptr_t stream, const char* fn) {
  SWB_REQUIRE(qkv && k_layer && v_layer && block_tables && ctx_lens && workspace && out,
              "%s: null pointer", fn);
  SWB_REQUIRE(dh == DA_D, "%s: dh must be 128", fn);
  SWB_REQUIRE(H > 0 && Hkv > 0 && H % Hkv == 0 && H / Hkv <= DA_MAXG,
              "%s: GQA group must be <= %d", fn, DA_MAXG);
  SWB_REQUIRE(B > 0 && max_ctx > 0 && block_size > 0 && partition > 0 &&
                  partition <= DA_MAXPART,
              "%s: bad sizes (partition must be 1..%d)", fn, DA_MAXPART);
  SWB_REQUIRE((block_size & (block_size - 1)) == 0 && partition % block_size == 0,
              "%s: block_size must be a power of two dividing partition", fn);
  SWB_REQUIRE(!STEP || alibi_slopes || theta > 1.f, "%s: theta", fn);
  SWB_REQUIRE(row_stride % 8 == 0, "%s: row_stride %% 8", fn);
  const int G = H / Hkv;
  const int NP = (max_ctx + partition - 1) / partition;
  // 8 warps when a GQA group shares the pass (more FMAs per staged byte)
  const int nw = G >= 4 ? 8 : 4;
  const size_t merge_scratch = sizeof(float) * (2 * (size_t)G * NP + G);
  const size_t smem = std::max(merge_scratch,
                               (size_t)partition * DA_D * 2 * 2 +
                                   sizeof(float) * ((size_t)G * DA_D + (size_t)G * partition +
                                                    (size_t)nw * G * DA_D + 2 * G));
  SWB_REQUIRE(smem <= 160 * 1024, "%s: max_ctx %d needs too many partitions", fn, max_ctx);
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(attn_decode_kernel<STEP, 4>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    SWB_CUDA(cudaFuncSetAttribute(attn_decode_kernel<STEP, 8>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr[dev] = true;
  }
  float* ws = reinterpret_cast<float*>(workspace);
  int* tickets = reinterpret_cast<int*>(ws + (size_t)B * H * NP * (DA_D + 2));
#ifdef SWB_ATTN_PROBE
  if (const char* pe = std::getenv("SWB_ATTN_PROBE_ADDR")) {
    unsigned long long* pp = reinterpret_cast<unsigned long long*>(std::strtoull(pe, nullptr, 0));
    cudaMemcpyToSymbolAsync(g_attn_probe, &pp, sizeof(pp), 0, cudaMemcpyHostToDevice,
                            (cudaStream_t)stream);
  }
#endif
  static const bool mma_on = [] {
    const char* e = std::getenv("SWB_ATTN_MMA");
    return !(e && e[0] == '0');
  }();
  // cluster-streaming kernel for MHA / small groups in the decode graph
  // (SWB_ATTN_CL=0 keeps the split-K kernel below; SWB_ATTN_CL_MAXB bounds
  // the batch it takes)
  static const int cl_maxb = [] {
    const char* e = std::getenv("SWB_ATTN_CL");
    if (e && e[0] == '0') return 0;
    // measured (7B, ctx 1100, decode step): B=1 2.68 -> 2.51 ms, B=8 4.65 ->
    // 4.57, but B=32 8.54 -> 8.87 (8192 single-wave clusters vs the split-K
    // kernel's 64-token partitions)
    const char* m = std::getenv("SWB_ATTN_CL_MAXB");
    return m ? std::atoi(m) : 16;
  }();
  // GQA groups (G = 4, 8) only with SWB_ATTN_CL_MAXB_GQA > 0 (A/B): the
  // consumer warps split the group's heads (G/4 each) and all walk every
  // page; CUDA-core dot products for 8 heads per page do not beat the
  // tensor-core split-K kernel.  (Splitting pages instead, every warp
  // carrying 8 heads, was FMA/shuffle-bound: 24.1 vs 12.8 us.)
  // measured (head split, B=1): 70B-TP2 ctx 1100 12.7 vs 12.4 us, ctx 8000
  // 58 vs 25 us, 70B TP4 step unchanged (8.48 ms) — so off by default
  const int cl_maxb_gqa = [] {            // read per call: tests switch it
    const char* e = std::getenv("SWB_ATTN_CL_MAXB_GQA");
    return e ? std::atoi(e) : 0;
  }();
  const int gi = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : G == 8 ? 3 : -1;
  if (STEP && gi >= 0 && block_size == 16 &&
      B <= (G <= 2 ? cl_maxb : std::min(cl_maxb, cl_maxb_gqa))) {
    // cluster x consumer-warp shape: SWB_ATTN_CL_CFG = "8x4" | "8x8" | "16x4" | "16x8";
    // ring depth: SWB_ATTN_CL_S = 8 (default) | 12
    static const int cfg_env = [] {
      const char* e = std::getenv("SWB_ATTN_CL_CFG");
      if (!e) return -1;
      if (!strcmp(e, "8x8")) return 1;
      if (!strcmp(e, "16x4")) return 2;
      if (!strcmp(e, "16x8")) return 3;
      if (!strcmp(e, "4x4")) return 4;
      return 0;
    }();
    // default 8x4; 4x4 when 8-CTA clusters would not fit one wave at 3
    // CTAs per SM (7B B=2: 512 CTAs > 444 slots)
    const int cfg_id = cfg_env >= 0 ? cfg_env : (B * Hkv * 8 > 3 * kNumSMs ? 4 : 0);
    static const int s_env = [] {
      const char* e = std::getenv("SWB_ATTN_CL_S");
      return e ? std::atoi(e) : 0;
    }();
    const int CL = cfg_id == 4 ? 4 : cfg_id >= 2 ? 16 : 8, CW = (cfg_id == 1 || cfg_id == 3) && G <= 2 ? 8 : 4;
    const int pages_per_cta = ((max_ctx + 15) / 16 + CL - 1) / CL;
    // 12 stages prefetch a 1100-token context whole before the PDL wait (7B
    // B=1 standalone 6.7 -> 6.0 us) but at 2 CTAs/SM the step loses (2.51 ->
    // 2.60 ms: less room for the next kernel's early CTAs); default 8
    (void)pages_per_cta;
    const int si = s_env == 12 ? 1 : 0;
    const int S = si ? 12 : 8;
    using KFn = void (*)(const __nv_bfloat16*, int, __nv_bfloat16*, __nv_bfloat16*,
                         const int32_t*, int, const int32_t*, float, const float*, int, int,
                         float, __nv_bfloat16*, int);
#define SWB_CLK(g, s) {attn_decode_cl_kernel<g, 8, 4, s>, attn_decode_cl_kernel<g, 8, 8, s>, \
                       attn_decode_cl_kernel<g, 16, 4, s>, attn_decode_cl_kernel<g, 16, 8, s>, \
                       attn_decode_cl_kernel<g, 4, 4, s>}
#define SWB_CLK4(g, s) {attn_decode_cl_kernel<g, 8, 4, s>, attn_decode_cl_kernel<g, 8, 4, s>, \
                        attn_decode_cl_kernel<g, 16, 4, s>, attn_decode_cl_kernel<g, 16, 4, s>, \
                        attn_decode_cl_kernel<g, 4, 4, s>}
    // GQA (head split across the 4 consumer warps): 4 warps in every shape
    static const KFn table[4][2][5] = {{SWB_CLK(1, 8), SWB_CLK(1, 12)},
                                       {SWB_CLK(2, 8), SWB_CLK(2, 12)},
                                       {SWB_CLK4(4, 8), SWB_CLK4(4, 12)},
                                       {SWB_CLK4(8, 8), SWB_CLK4(8, 12)}};
#undef SWB_CLK4
#undef SWB_CLK
    const KFn kern = table[gi][si][cfg_id];
    const size_t smem_c = dcl_smem(G, CW, S, CL);
    static bool attr_c[64][40] = {};
    const int ai = gi * 10 + si * 5 + cfg_id;
    if (dev < 64 && !attr_c[dev][ai]) {
      SWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_c));
      if (CL > 8)
        SWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr_c[dev][ai] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, Hkv, B);
    cfg.blockDim = dim3((CW + 1) * 32);
    cfg.dynamicSmemBytes = smem_c;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const float l2t = !alibi_slopes ? log2f(theta) : 0.f;
    const float sc = scale * 1.4426950408889634f;
    const int trig = pdl_early_trigger() ? 1 : 0;
    const cudaError_t lc = cudaLaunchKernelEx(
        &cfg, kern, reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride,
        reinterpret_cast<__nv_bfloat16*>(k_layer), reinterpret_cast<__nv_bfloat16*>(v_layer),
        block_tables, max_blocks, ctx_lens, l2t, alibi_slopes, H, Hkv, sc,
        reinterpret_cast<__nv_bfloat16*>(out), trig);
    if (lc != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch attn_decode_cl_kernel: %s",
                           cudaGetErrorString(lc));
    return swb_check_launch("attn_decode_cl_kernel");
  }
  // tensor-core kernel for GQA groups (measured: 70B-TP2 B=8 17.0 vs 19.5 us,
  // B=32 54 vs 63 us); for MHA (G=1) the CUDA-core kernel is ahead (7B B=1
  // 10.0 vs 13.9 us: the unswizzled 256-byte page rows cost the MMA kernel
  // 8-way ldmatrix conflicts that only pay off when G rows share them)
  if (mma_on && G >= 4 && block_size == 16 && (partition == 128 || partition == 64)) {
    static bool attr_m[64] = {false};
    if (dev < 64 && !attr_m[dev]) {
      SWB_CUDA(cudaFuncSetAttribute(attn_decode_mma_kernel<STEP, 32>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      SWB_CUDA(cudaFuncSetAttribute(attn_decode_mma_kernel<STEP, 16>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      attr_m[dev] = true;
    }
    const size_t msm = std::max(merge_scratch,
                                (size_t)2 * partition * DA_D * 2 + 16 * DM_QS * 2 +
                                    sizeof(float) * (DM_WARPS * 8 * 2 + (size_t)DM_WARPS * G * DA_D));
    // cluster form (decode graph, 128-token partitions): the NP partitions of
    // a (b, kv head) are one cluster of 8 or 16 CTAs merging through DSMEM —
    // no global partials / ticket / fences (SWB_ATTN_MMA_CL_MAXB bounds B)
    const int mcl_maxb = [] {
      const char* e = std::getenv("SWB_ATTN_MMA_CL_MAXB");
      return e ? std::atoi(e) : 2;
    }();
    if (STEP && partition == 128 && B <= mcl_maxb && NP <= 16) {
      const int CLN = NP <= 8 ? 8 : 16;
      auto kern = CLN == 8 ? attn_decode_mma_kernel<STEP, 32, 8> : attn_decode_mma_kernel<STEP, 32, 16>;
      const size_t csm = (size_t)2 * partition * DA_D * 2 + 16 * DM_QS * 2 +
                         sizeof(float) * (DM_WARPS * 8 * 2 + (size_t)DM_WARPS * G * DA_D +
                                          (size_t)CLN * G * DCL_ST + (size_t)G * (DA_D + 2));
      static bool attr_mc[64][2] = {};
      if (dev < 64 && !attr_mc[dev][CLN == 16]) {
        SWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      160 * 1024));
        if (CLN > 8)
          SWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_mc[dev][CLN == 16] = true;
      }
      SWB_REQUIRE(csm <= 160 * 1024, "%s: cluster MMA smem", fn);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CLN, Hkv, B);
      cfg.blockDim = dim3(DM_WARPS * 32);
      cfg.dynamicSmemBytes = csm;
      cfg.stream = (cudaStream_t)stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CLN;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      const cudaError_t lc = cudaLaunchKernelEx(
          &cfg, kern, reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride,
          reinterpret_cast<__nv_bfloat16*>(k_layer), reinterpret_cast<__nv_bfloat16*>(v_layer),
          block_tables, max_blocks, ctx_lens, positions, slots,
          !alibi_slopes ? log2f(theta) : 0.f, alibi_slopes, H, Hkv,
          scale * 1.4426950408889634f, ws, tickets, reinterpret_cast<__nv_bfloat16*>(out),
          pdl_early_trigger() ? 1 : 0);
      if (lc != cudaSuccess)
        return swb_set_error(SWB_ERR_CUDA, "launch attn_decode_mma_kernel (cluster): %s",
                             cudaGetErrorString(lc));
      return swb_check_launch("attn_decode_mma_kernel");
    }
    const cudaError_t lm = launch(
        partition == 128 ? attn_decode_mma_kernel<STEP, 32> : attn_decode_mma_kernel<STEP, 16>,
        dim3(NP, Hkv, B), dim3(DM_WARPS * 32), msm,
        (cudaStream_t)stream, reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride,
        reinterpret_cast<__nv_bfloat16*>(k_layer), reinterpret_cast<__nv_bfloat16*>(v_layer),
        block_tables, max_blocks, ctx_lens, positions, slots,
        (STEP || positions) && !alibi_slopes ? log2f(theta) : 0.f, alibi_slopes, H, Hkv,
        scale * 1.4426950408889634f, ws, tickets, reinterpret_cast<__nv_bfloat16*>(out),
        pdl_early_trigger() ? 1 : 0);
    if (lm != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch attn_decode_mma_kernel: %s",
                           cudaGetErrorString(lm));
    return swb_check_launch("attn_decode_mma_kernel");
  }
  const cudaError_t le = launch(
      nw == 8 ? attn_decode_kernel<STEP, 8> : attn_decode_kernel<STEP, 4>, dim3(NP, Hkv, B),
      dim3(nw * 32), smem, (cudaStream_t)stream,
      reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride,
      reinterpret_cast<__nv_bfloat16*>(k_layer), reinterpret_cast<__nv_bfloat16*>(v_layer),
      block_tables, max_blocks, ctx_lens, positions, slots,
      (STEP || positions) && !alibi_slopes ? log2f(theta) : 0.f, alibi_slopes, H, Hkv,
      block_size, scale * 1.4426950408889634f, partition, ws, tickets,
      reinterpret_cast<__nv_bfloat16*>(out), pdl_early_trigger() ? 1 : 0);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch attn_decode_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("attn_decode_kernel");
}

extern "C" int swb_attn_decode(const void* qkv, int row_stride, void* k_layer, void* v_layer,
                               const int32_t* block_tables, int max_blocks,
                               const int32_t* ctx_lens, const int32_t* positions,
                               const int32_t* slots, float theta, const float* alibi_slopes,
                               int B, int H, int Hkv, int dh, int block_size, float scale,
                               int max_ctx, int partition, void* workspace, void* out,
                               uintptr_t stream) {
  SWB_REQUIRE((positions == nullptr) == (slots == nullptr),
              "swb_attn_decode: positions and slots go together");
  SWB_REQUIRE(!positions || alibi_slopes || theta > 1.f, "swb_attn_decode: theta");
  return launch_attn_decode<false>(qkv, row_stride, k_layer, v_layer, block_tables, max_blocks,
                                   ctx_lens, positions, slots, theta, alibi_slopes, B, H, Hkv,
                                   dh, block_size, scale, max_ctx, partition, workspace, out,
                                   stream, "swb_attn_decode");
}

extern "C" int swb_attn_decode_step(const void* qkv, int row_stride, void* k_layer,
                                    void* v_layer, const int32_t* block_tables, int max_blocks,
                                    const int32_t* ctx, float theta,
                                    const float* alibi_slopes, int B, int H, int Hkv, int dh,
                                    int block_size, float scale, int max_ctx, int partition,
                                    void* workspace, void* out, uintptr_t stream) {
  return launch_attn_decode<true>(qkv, row_stride, k_layer, v_layer, block_tables, max_blocks,
                                  ctx, nullptr, nullptr, theta, alibi_slopes, B, H, Hkv, dh,
                                  block_size, scale, max_ctx, partition, workspace, out, stream,
                                  "swb_attn_decode_step");
}

// workspace: merge tickets [H][DC_MAXQT] ints first (fixed offsets, so calls
// with different chunk lengths share one zeroed workspace), then the partials
extern "C" size_t swb_attn_chunk_workspace(int C, int H, int max_ctx) {
  if (C <= 0 || H <= 0 || max_ctx <= 0) return 0;
  const size_t nq = (C + 15) / 16, np = (max_ctx + DM_PT - 1) / DM_PT;
  return (size_t)H * DC_MAXQT * sizeof(int) +
         (size_t)H * nq * 16 * np * (DA_D + 2) * sizeof(float);
}

extern "C" int swb_attn_chunk(const void* qkv, int row_stride, int C, int q_start,
                              const void* k_layer, const void* v_layer, const int32_t* table_row,
                              int H, int Hkv, int dh, int block_size, float scale,
                              const float* alibi_slopes, int max_ctx, void* workspace, void* out,
                              uintptr_t stream) {
  SWB_REQUIRE(qkv && k_layer && v_layer && table_row && workspace && out,
              "swb_attn_chunk: null pointer");
  SWB_REQUIRE(dh == DA_D && block_size == 16, "swb_attn_chunk: dh 128 and block_size 16 only");
  SWB_REQUIRE(H > 0 && Hkv > 0 && H % Hkv == 0, "swb_attn_chunk: bad heads");
  SWB_REQUIRE(C > 0 && q_start >= 0 && q_start + C <= max_ctx, "swb_attn_chunk: bad chunk");
  SWB_REQUIRE(row_stride % 8 == 0, "swb_attn_chunk: row_stride %% 8");
  const int nq = (C + 15) / 16;
  const int NP = (q_start + C + DM_PT - 1) / DM_PT;          // partitions the chunk can see
  const size_t smem = std::max((size_t)2 * DM_PT * DA_D * 2 + 16 * DM_QS * 2 +
                                   sizeof(float) * (DM_WARPS * 16 * 2 + (size_t)DM_WARPS * 16 * DA_D),
                               sizeof(float) * (2 * 16 * (size_t)NP + 16));
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(attn_chunk_kernel<0>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr[dev] = true;
  }
  SWB_REQUIRE(smem <= 160 * 1024, "swb_attn_chunk: context too long");
  SWB_REQUIRE(nq <= DC_MAXQT, "swb_attn_chunk: C=%d > %d rows", C, 16 * DC_MAXQT);
  int* tickets = reinterpret_cast<int*>(workspace);
  float* ws = reinterpret_cast<float*>(tickets + (size_t)H * DC_MAXQT);
  const cudaError_t le = launch(
      attn_chunk_kernel<0>, dim3(NP, H, nq), dim3(DM_WARPS * 32), smem, (cudaStream_t)stream,
      reinterpret_cast<const __nv_bfloat16*>(qkv), row_stride, C, q_start,
      reinterpret_cast<const __nv_bfloat16*>(k_layer),
      reinterpret_cast<const __nv_bfloat16*>(v_layer), table_row, H, Hkv,
      scale * 1.4426950408889634f, alibi_slopes, ws, tickets,
      reinterpret_cast<__nv_bfloat16*>(out));
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch attn_chunk_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("attn_chunk_kernel");
}
