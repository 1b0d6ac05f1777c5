// Causal varlen prefill attention on the 5th-generation tensor cores.
//
// One CTA = 128 query rows of one head (GQA: kv head = h / G), head_dim 128.
//   warp 0  TMA producer: Q once, then K_j / V_j tiles (128 keys x 128 d) into
//           2-stage rings, 128B-swizzled boxes of 64 columns.
//   warp 1  one thread issues tcgen05.mma:
//             S_j  = Q . K_j^T   (M=128, N=128, K=128; both operands K-major)
//                    into one of two TMEM score buffers (double-buffered so
//                    S_{j+1} runs while the softmax warps work on S_j)
//             O   += P_j . V_j   (A = P from smem, K-major over keys;
//                    B = V MN-major: d contiguous, exactly as it sits in the
//                    qkv rows) into a TMEM accumulator
//   warps 2-5  softmax: thread = query row (TMEM lane), reads its 128 scores
//           with tcgen05.ld, applies the causal mask, online max/sum with
//           exp2, writes its P row (bf16, swizzled) to smem, rescales its O
//           row in TMEM (tcgen05.ld/st) when the running max moved, and at the
//           end normalises O and stores it.
// TMEM: S0 cols [0,128), S1 [128,256), O [256,384).
//
// Replaces (with swb_attn_prefill's FA2 kernel) the attention share of the
// prompt-phase cost PerfModel.prompt_time (reference perf.py:119-123).
#include <cudaTypedefs.h>

#include "common.cuh"

namespace swb {

int make_tmap_rows(CUtensorMap* map, const void* base, int rows, int K, int box_rows);

constexpr int TA_BM = 128, TA_BN = 128, TA_D = 128;
constexpr int TA_TILE = TA_BM * TA_D * 2;          // 32 KB: 128 rows x 128 bf16
constexpr int TA_HALF = TA_TILE / 2;               // one 64-column swizzled block
constexpr int TA_OFF_Q = 0;
constexpr int TA_OFF_K = TA_OFF_Q + TA_TILE;       // 2 stages
constexpr int TA_OFF_V = TA_OFF_K + 2 * TA_TILE;   // 2 stages
constexpr int TA_OFF_P = TA_OFF_V + 2 * TA_TILE;
constexpr int TA_OFF_BAR = TA_OFF_P + TA_TILE;
constexpr int TA_SMEM = TA_OFF_BAR + 256 + 1024;   // + alignment slack
constexpr int TA_THREADS = 192;

// K-major SW128 descriptor (rows of 128 B, 8-row groups 1 KB apart)
__device__ __forceinline__ uint64_t desc_k(uint32_t addr) { return umma_desc_k_sw128(addr); }
// MN-major SW128 descriptor: 64-element (128 B) atoms along N, 8-row K groups
// 1 KB apart (SBO), next 64-element N block LBO bytes away
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// bf16 x bf16 -> f32, M=128 N=128, A K-major, B K-major (b_mn=0) or MN-major
__host__ __device__ constexpr uint32_t idesc_attn(bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(TA_BN >> 3) << 17) | ((uint32_t)(TA_BM >> 4) << 24);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ALIBI: scores get slope_h * (key - query) (BLOOM; softmax-equivalent to
// the slope * key form), slopes given per head of this rank.
template <bool ALIBI>
__global__ void __launch_bounds__(TA_THREADS, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tm, const int32_t* cu,
                           int tiles_per_seq, int H, int Hkv, float scale_log2,
                           const float* __restrict__ alibi, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TA_OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_free = bars + 11;  // [2]
  uint64_t* p_ready = bars + 13;
  uint64_t* o_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (H, tiles * seqs), x fastest: the hardware hands out CTAs in order,
  // so every head's heaviest (last, causal) query tiles of every sequence go
  // first and the light ones fill the SMs that free up — a longest-first
  // schedule of the triangular work (1 CTA per SM by smem/TMEM)
  const int nseq = gridDim.y / tiles_per_seq;
  const int seq = blockIdx.y % nseq;
  const int qt = tiles_per_seq - 1 - blockIdx.y / nseq;
  const int h = blockIdx.x, kh = h / (H / Hkv);
  pdl_wait();
  const int s0 = cu[seq], len = cu[seq + 1] - s0;
  const int q0 = qt * TA_BM;
  if (q0 >= len) return;
  const int nkv = (min(q0 + TA_BM, len) - 1) / TA_BN + 1;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < 15; ++i) mbar_init(&bars[i], 1);
    mbar_init(&s_free[0], 4);
    mbar_init(&s_free[1], 4);
    mbar_init(p_ready, 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;

  const int qcol = h * TA_D, kcol = (H + kh) * TA_D, vcol = (H + Hkv + kh) * TA_D;
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(q_full, TA_TILE);
      tma_load_2d(smem + TA_OFF_Q, &tm, q_full, qcol, s0 + q0);
      tma_load_2d(smem + TA_OFF_Q + TA_HALF, &tm, q_full, qcol + 64, s0 + q0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait_sleep(&k_empty[st], ((j >> 1) - 1) & 1);
        uint8_t* kb = smem + TA_OFF_K + st * TA_TILE;
        mbar_arrive_expect_tx(&k_full[st], TA_TILE);
        tma_load_2d(kb, &tm, &k_full[st], kcol, s0 + j * TA_BN);
        tma_load_2d(kb + TA_HALF, &tm, &k_full[st], kcol + 64, s0 + j * TA_BN);
        if (j >= 2) mbar_wait_sleep(&v_empty[st], ((j >> 1) - 1) & 1);
        uint8_t* vb = smem + TA_OFF_V + st * TA_TILE;
        mbar_arrive_expect_tx(&v_full[st], TA_TILE);
        tma_load_2d(vb, &tm, &v_full[st], vcol, s0 + j * TA_BN);
        tma_load_2d(vb + TA_HALF, &tm, &v_full[st], vcol + 64, s0 + j * TA_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------- MMA issuer
      constexpr uint32_t id_s = idesc_attn(false), id_o = idesc_attn(true);
      const uint32_t qa = smem_u32(smem + TA_OFF_Q), pa = smem_u32(smem + TA_OFF_P);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_free[st], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + TA_OFF_K + st * TA_TILE);
#pragma unroll
        for (int kk = 0; kk < TA_D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * TA_HALF + (kk & 3) * 32;
          tc_mma_f16(t_s[st], desc_k(qa + off), desc_k(ka + off), id_s, kk != 0);
        }
        tc_commit(&s_full[st]);
        tc_commit(&k_empty[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(p_ready, j & 1);
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(smem + TA_OFF_V + st * TA_TILE);
#pragma unroll
        for (int kk = 0; kk < TA_BN / 16; ++kk) {
          // keys 16kk..16kk+15: P column block kk/4 (+32 B per 16 keys);
          // V rows 16kk.. (16 keys x 128 B = 2 KB per step)
          const uint32_t poff = (kk >> 2) * TA_HALF + (kk & 3) * 32;
          tc_mma_f16(t_o, desc_k(pa + poff), desc_mn(va + kk * 2048, TA_HALF), id_o,
                     (j | kk) != 0);
        }
        tc_commit(o_done);
        tc_commit(&v_empty[st]);
      }
    }
  } else {
    // ------------------------------------------------- softmax warps
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;          // query row in the tile
    const int qrow = q0 + r;                    // position in the sequence
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint8_t* prow = smem + TA_OFF_P;
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = ALIBI ? alibi[h] * 1.4426950408889634f : 0.f;
    const float sc = ALIBI ? 1.f : scale_log2;   // scores already scaled under ALIBI
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_s[st] + lane_off + c * 32, sv[c]);
      tc_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[st]);
      // causal mask (keys beyond the row, incl. keys beyond len) + row max
      const int k0 = j * TA_BN;
      if (ALIBI) {    // move to the log2 domain here: t = s*scale + slope*(k - q)
        const float base = sl2 * (float)(k0 - qrow);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            sv[c][i] = __float_as_uint(fmaf(__uint_as_float(sv[c][i]), scale_log2,
                                            fmaf(sl2, (float)(c * 32 + i), base)));
      }
      float mx = -INFINITY;
      if (k0 + TA_BN - 1 > q0) {      // tile touches the diagonal (block-uniform)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float v = __uint_as_float(sv[c][i]);
            if (k0 + c * 32 + i > qrow) v = -INFINITY;
            sv[c][i] = __float_as_uint(v);
            mx = fmaxf(mx, v);
          }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(sv[c][i]));
      }
      const float m_new = fmaxf(m_run, mx);
      const float msc = m_new == -INFINITY ? 0.f : m_new * sc;
      const float corr = m_run == -INFINITY ? 0.f : exp2f(m_run * sc - msc);
      float rs = 0.f;
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = exp2f(__uint_as_float(sv[c][2 * i]) * sc - msc);
          const float p1 = exp2f(__uint_as_float(sv[c][2 * i + 1]) * sc - msc);
          rs += p0 + p1;
          pk[c][i] = f2_to_bf2(p0, p1);
        }
      l_run = l_run * corr + rs;
      // previous P . V must be done before P is overwritten / O is rescaled
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
      }
      // P row r: 128 keys = 2 column blocks of 64 keys, 16 B chunks swizzled
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int key8 = c * 4 + q4;          // 8-key chunk index 0..15
          const int blk = key8 >> 3, ch = key8 & 7;
          uint4* dst = reinterpret_cast<uint4*>(prow + blk * TA_HALF + r * 128 +
                                                ((ch ^ (r & 7)) << 4));
          *dst = make_uint4(pk[c][4 * q4], pk[c][4 * q4 + 1], pk[c][4 * q4 + 2],
                            pk[c][4 * q4 + 3]);
        }
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {   // warp-uniform: tcgen05.ld/st are .sync.aligned
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t ov[32];
          tmem_ld32(t_o + lane_off + c * 32, ov);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
          tmem_st32(t_o + lane_off + c * 32, ov);
        }
        tc_wait_st();
      }
      m_run = m_new;
      fence_async_smem();   // P (generic-proxy stores) visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    // ---- epilogue: O / l -> bf16 -> out
    mbar_wait(o_done, (nkv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l_run;
    const bool ok = qrow < len;
    __nv_bfloat16* orow = out + (size_t)(s0 + qrow) * (H * TA_D) + h * TA_D;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld32(t_o + lane_off + c * 32, ov);
      tc_wait_ld();
      if (ok) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(
              f2_to_bf2(__uint_as_float(ov[8 * i + 0]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
              f2_to_bf2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
              f2_to_bf2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
              f2_to_bf2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <bool ALIBI>
static int launch_tc(const CUtensorMap& tm, const int32_t* cu, int num_seqs, int tiles, int H,
                     int Hkv, float scale, const float* alibi, void* out, cudaStream_t stream) {
  static bool attr[64] = {false};
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    SWB_CUDA(cudaFuncSetAttribute(attn_prefill_tc_kernel<ALIBI>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, TA_SMEM));
    attr[dev] = true;
  }
  const cudaError_t le = launch(attn_prefill_tc_kernel<ALIBI>, dim3(H, num_seqs * tiles),
                                dim3(TA_THREADS), TA_SMEM, stream, tm, cu, tiles, H, Hkv,
                                scale * 1.4426950408889634f, alibi,
                                reinterpret_cast<__nv_bfloat16*>(out));
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch attn_prefill_tc_kernel: %s",
                         cudaGetErrorString(le));
  return swb_check_launch("attn_prefill_tc_kernel");
}

int launch_attn_prefill_tc(const void* qkv, int row_stride, int total_rows, const int32_t* cu,
                           int num_seqs, int max_seqlen, int H, int Hkv, float scale,
                           const float* alibi, void* out, cudaStream_t stream) {
  CUtensorMap tm;
  // the whole qkv matrix as one K-major operand: rows = tokens, 64-col boxes
  const int st = make_tmap_rows(&tm, qkv, total_rows, row_stride, 128);
  if (st) return st;
  const int tiles = (max_seqlen + TA_BM - 1) / TA_BM;
  if (alibi) return launch_tc<true>(tm, cu, num_seqs, tiles, H, Hkv, scale, alibi, out, stream);
  return launch_tc<false>(tm, cu, num_seqs, tiles, H, Hkv, scale, nullptr, out, stream);
}

}  // namespace swb

using namespace swb;

extern "C" int swb_attn_prefill_tc(const void* qkv, int row_stride, int total_rows,
                                   const int32_t* cu_seqlens, int num_seqs, int max_seqlen,
                                   int H, int Hkv, int dh, float scale,
                                   const float* alibi_slopes, void* out, uintptr_t stream) {
  SWB_REQUIRE(qkv && cu_seqlens && out, "swb_attn_prefill_tc: null pointer");
  SWB_REQUIRE(dh == TA_D, "swb_attn_prefill_tc: dh must be 128 (got %d)", dh);
  SWB_REQUIRE(H > 0 && Hkv > 0 && H % Hkv == 0, "swb_attn_prefill_tc: bad heads");
  SWB_REQUIRE(row_stride % 8 == 0 && row_stride >= (H + 2 * Hkv) * dh,
              "swb_attn_prefill_tc: bad row_stride %d", row_stride);
  SWB_REQUIRE((((uintptr_t)qkv | (uintptr_t)out) & 15) == 0,
              "swb_attn_prefill_tc: pointers must be 16-byte aligned");
  SWB_REQUIRE(num_seqs >= 0 && max_seqlen >= 0 && total_rows >= 0,
              "swb_attn_prefill_tc: bad sizes");
  if (num_seqs == 0 || max_seqlen == 0 || total_rows == 0) return SWB_OK;
  return launch_attn_prefill_tc(qkv, row_stride, total_rows, cu_seqlens, num_seqs, max_seqlen,
                                H, Hkv, scale, alibi_slopes, out, (cudaStream_t)stream);
}
