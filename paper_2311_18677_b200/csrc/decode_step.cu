// One whole token-phase iteration in ONE persistent kernel (batch <= 8).
//
// The decode step of a Llama-style model is a chain of weight-streaming
// GEMVs separated by all-to-all dependencies (each output needs the whole
// input vector).  Launching them as separate kernels leaves HBM idle for
// several microseconds at every boundary (launch, pipeline fill, tail).  Here
// one CTA per SM (cooperative launch) runs the whole step:
//
//   warp 16 (producer): one lane streams EVERY weight matrix of the step —
//     L x [Wqkv, Wo, Wgu, Wd] then the LM head — through a 4-stage ring of
//     32 KB stages (4 rows x 4096 columns, 1-D cp.async.bulk, L2 evict-first)
//     in exactly the order the consumers use them.  It never waits on a
//     phase boundary, so the next matrix's first bytes are already on chip
//     while the consumers cross a grid barrier.
//   warps 0..15 (consumers): execute the phases
//       P0  prepare positions/slots, embed the current tokens
//       per layer:
//         A   QKV GEMV with the pre-attention RMSNorm fused (x fp32 -> bf16 h)
//         B   paged attention, one work item per (seq, kv head, 64-token
//             partition): current token's RoPE + KV append, cp.async gather
//             of the partition through the block table, split-K partials,
//             last-CTA merge (atomic ticket)
//         C   O GEMV + residual add into x
//         D   gate/up GEMV with the pre-MLP RMSNorm and SwiGLU fused
//         E   down GEMV + residual add into x
//       F   LM-head GEMV with the final RMSNorm fused (fp32 logits)
//       G   greedy argmax + step advance (token ring, context length)
//     with a grid-wide barrier between dependent phases (atomic counter,
//     acquire polling, bounded by a watchdog that traps instead of hanging).
//
// GEMV consumer layout: warp w owns columns [256w, 256w+256) of every stage
// for all 4 rows of a work item, lane = 8 columns (one 16-byte shared load per
// row); per-item partials are shuffle-reduced and combined across warps
// through shared memory.  Numerics match the multi-kernel path (swb_rmsnorm
// rounding, fp32 accumulation, bf16 activations).
//
// Replaces PerfModel.token_iter_time (reference perf.py:125-132) as one
// launch; the bookkeeping of Machine.complete_iteration (machine.py:263-266)
// happens on the device.
#include "common.cuh"

namespace swb {

constexpr int DS_CWARPS = 16;                    // consumer warps
constexpr int DS_THREADS = (DS_CWARPS + 1) * 32;  // + producer warp
constexpr int DS_ROWS = 4;                       // weight rows per item
constexpr int DS_KC = DS_CWARPS * 256;           // 4096 columns per stage
constexpr int DS_ROW_BYTES = DS_KC * 2;          // 8 KB
constexpr int DS_STAGE_BYTES = DS_ROWS * DS_ROW_BYTES;  // 32 KB
constexpr int DS_STAGES = 5;
constexpr int DS_CHUNK = 64;                     // attention chunk (tokens)
constexpr int DS_D = 128;                        // head dim
constexpr int DS_MAXG = 4;                       // GQA group supported here
constexpr int DS_MAXB = 8;                       // batch supported here

// shared memory carve-up (bytes).  The attention phase does not stream
// weights, so its scratch ALIASES the weight ring: the producer holds back the
// O-projection prefetch until the attention phase has released the ring
// (attn_done barrier), which buys a deeper ring for every GEMV phase.
constexpr int DS_OFF_RING = 0;
constexpr int DS_RING_BYTES = DS_STAGES * DS_STAGE_BYTES;                   // 160 KB
constexpr int DS_CAP = 288;                      // tokens per attention load wave
constexpr int DS_OFF_K = DS_OFF_RING;              // [CAP][128] bf16
constexpr int DS_OFF_V = DS_OFF_K + DS_CAP * DS_D * 2;                      // [CAP][128] bf16
constexpr int DS_OFF_SACC = DS_OFF_K;              // [16][G][128] f32, aliases K after scores
constexpr int DS_OFF_CUR = DS_OFF_V + DS_CAP * DS_D * 2;                    // cur k, v bf16
constexpr int DS_OFF_SQ = DS_OFF_CUR + 2 * DS_D * 2;                        // [G][128] f32
constexpr int DS_OFF_SS = DS_OFF_SQ + DS_MAXG * DS_D * 4;                   // [G][CAP] f32
constexpr int DS_OFF_SSTAT = DS_OFF_SS + DS_MAXG * DS_CAP * 4;              // m, l, scale [G]
constexpr int DS_ATTN_END = DS_OFF_SSTAT + DS_MAXG * 4 * 4;
constexpr int DS_HS_BYTES = 48 * 1024;             // staged GEMV input h (bf16 M x K)
constexpr int DS_OFF_HS = DS_OFF_RING + DS_RING_BYTES;
constexpr int DS_OFF_BAR = DS_OFF_HS + DS_HS_BYTES;                         // mbarriers
constexpr int DS_OFF_PART = DS_OFF_BAR + (2 * DS_STAGES + 2) * 8;           // [2][16][4][8] f32
constexpr int DS_OFF_RSTD = DS_OFF_PART + 2 * DS_CWARPS * DS_ROWS * DS_MAXB * 4;
constexpr int DS_OFF_MISC = DS_OFF_RSTD + 64;                               // ints / flags
constexpr int DS_SMEM = DS_OFF_MISC + 128 + 128;
static_assert(DS_ATTN_END <= DS_RING_BYTES, "attention scratch must fit in the ring");
static_assert((DS_CWARPS * DS_MAXG * DS_D + DS_CWARPS * DS_MAXG) * 4 <= DS_CAP * DS_D * 2,
              "sacc + wave-reduction scratch alias the K buffer");
static_assert(DS_SMEM <= 227 * 1024, "smem budget");
static_assert(DS_SMEM <= 227 * 1024, "smem budget");

// attention partitions: about one (seq, kv head, partition) item per CTA, and
// never more than DS_CAP tokens per item when the context allows
__host__ __device__ inline int ds_num_parts(int B, int Hkv, int max_ctx, int grid) {
  int np = grid / (B * Hkv);
  const int need = (max_ctx + DS_CAP - 1) / DS_CAP;
  const int maxnp = (max_ctx + 15) / 16;
  if (np < need) np = need;
  if (np > maxnp) np = maxnp;
  return np < 1 ? 1 : np;
}

struct DSWork {
  float* part;            // attention partials [B][H][NP][130]
  int* tickets;           // [B][Hkv]
  unsigned* barrier;      // grid barrier counter (zeroed before each launch)
  unsigned long long* trace;  // CTA 0 timestamps per barrier (diagnostics)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cbar() {  // consumer-only named barrier
  asm volatile("bar.sync 1, %0;" ::"n"(DS_CWARPS * 32) : "memory");
}

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& epoch,
                                          unsigned long long* trace = nullptr) {
  cbar();
  if (threadIdx.x == 0) {
    if (trace && blockIdx.x == 0 && epoch < 1024) trace[2 * epoch] = globaltimer();
    epoch += 1;
    const unsigned target = epoch * gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    const long long t0 = clock64();
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(64);
      if (clock64() - t0 > 8000000000LL) __trap();  // watchdog (~4 s): fail, never hang
    }
    __threadfence();
    if (trace && blockIdx.x == 0 && epoch <= 1024) trace[2 * epoch - 1] = globaltimer();
  }
  cbar();
}

__device__ __forceinline__ uint64_t ds_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void ds_bulk(void* dst, const void* src, uint32_t bytes,
                                        uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void ds_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

__device__ __forceinline__ int ds_row(int item, int j, bool swiglu) {
  if (!swiglu) return item * DS_ROWS + j;
  const int o = item * 2 + (j & 1);
  return (o >> 7) * 256 + (o & 127) + (j >= 2 ? 128 : 0);
}

struct MatDesc {
  const __nv_bfloat16* w;
  int N, K;
  bool swiglu;
};

// ------------------------------------------------------------- producer
__device__ void produce_matrix(const MatDesc& m, uint8_t* ring, uint64_t* full,
                               uint64_t* empty, int& it, uint64_t pol) {
  const int items = (m.N + DS_ROWS - 1) / DS_ROWS;
  const int nk = (m.K + DS_KC - 1) / DS_KC;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % DS_STAGES;
      if (it >= DS_STAGES) mbar_wait_sleep(&empty[s], ((it / DS_STAGES) - 1) & 1);
      const int k0 = kc * DS_KC;
      const uint32_t bytes = (uint32_t)min(DS_KC, m.K - k0) * 2;
      uint32_t total = 0;
      for (int j = 0; j < DS_ROWS; ++j)
        if (ds_row(item, j, m.swiglu) < m.N) total += bytes;
      mbar_arrive_expect_tx(&full[s], total);
      uint8_t* st = ring + s * DS_STAGE_BYTES;
      for (int j = 0; j < DS_ROWS; ++j) {
        const int row = ds_row(item, j, m.swiglu);
        if (row < m.N)
          ds_bulk(st + j * DS_ROW_BYTES, m.w + (size_t)row * m.K + k0, bytes, &full[s], pol);
      }
    }
  }
}

// ------------------------------------------------------------- consumers
// out = epi(h . W^T); h = x (bf16) or rmsnorm(x fp32, nw) when nw != nullptr
template <int MB>
__device__ void consume_matrix(const MatDesc& m, const void* xin, const __nv_bfloat16* nw,
                               float eps, int M, int epi, void* out, float* resid,
                               uint8_t* smem, uint64_t* full, uint64_t* empty, int& it,
                               int& parity) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* part = reinterpret_cast<float*>(smem + DS_OFF_PART);
  float* rstd = reinterpret_cast<float*>(smem + DS_OFF_RSTD);
  const float* xf = reinterpret_cast<const float*>(xin);
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(xin);
  const int K = m.K, N = m.N;
  // Stage the GEMV input h (bf16, M x K) in shared memory once per phase:
  // RMSNorm applied on the way (bit-identical to swb_rmsnorm) when nw is set.
  // The attention scratch region is idle during GEMV phases.
  __nv_bfloat16* hs = reinterpret_cast<__nv_bfloat16*>(smem + DS_OFF_HS);
  const bool staged = (size_t)M * K * 2 <= (size_t)DS_HS_BYTES;
  if (nw) {
    for (int b = 0; b < M; ++b) {
      float ss = 0.f;
      for (int k = threadIdx.x * 4; k < K; k += DS_CWARPS * 32 * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xf + (size_t)b * K + k);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
      ss = warp_sum(ss);
      if (lane == 0) part[warp * DS_MAXB + b] = ss;
    }
    cbar();
    if (threadIdx.x < M) {
      float ss = 0.f;
      for (int w = 0; w < DS_CWARPS; ++w) ss += part[w * DS_MAXB + threadIdx.x];
      rstd[threadIdx.x] = rsqrtf(ss / (float)K + eps);
    }
    cbar();
  }
  if (staged) {
    for (int i = threadIdx.x; i < M * K / 8; i += DS_CWARPS * 32) {
      const int b = (i * 8) / K, k = (i * 8) % K;
      uint4 h;
      if (nw) {
        const float r = rstd[b];
        const uint4 wq = *reinterpret_cast<const uint4*>(nw + k);
        const float2 n0 = bf2_to_f2(wq.x), n1 = bf2_to_f2(wq.y), n2 = bf2_to_f2(wq.z),
                     n3 = bf2_to_f2(wq.w);
        const float4 a = *reinterpret_cast<const float4*>(xf + (size_t)b * K + k);
        const float4 c = *reinterpret_cast<const float4*>(xf + (size_t)b * K + k + 4);
        h = make_uint4(f2_to_bf2(a.x * r * n0.x, a.y * r * n0.y),
                       f2_to_bf2(a.z * r * n1.x, a.w * r * n1.y),
                       f2_to_bf2(c.x * r * n2.x, c.y * r * n2.y),
                       f2_to_bf2(c.z * r * n3.x, c.w * r * n3.y));
      } else {
        h = *reinterpret_cast<const uint4*>(xb + (size_t)b * K + k);
      }
      *reinterpret_cast<uint4*>(hs + (size_t)b * K + k) = h;
    }
    cbar();
  }
  const int items = (N + DS_ROWS - 1) / DS_ROWS;
  const int nk = (K + DS_KC - 1) / DS_KC;
  for (int item = blockIdx.x; item < items; item += gridDim.x, ++parity) {
    float acc[DS_ROWS][MB];
#pragma unroll
    for (int j = 0; j < DS_ROWS; ++j)
#pragma unroll
      for (int b = 0; b < MB; ++b) acc[j][b] = 0.f;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int s = it % DS_STAGES;
      const int k = kc * DS_KC + warp * 256 + lane * 8;
      uint4 xq[MB];
      if (k < K) {
        if (staged) {
#pragma unroll
          for (int b = 0; b < MB; ++b)
            if (b < M) xq[b] = *reinterpret_cast<const uint4*>(hs + (size_t)b * K + k);
        } else if (nw) {
          const uint4 wq = *reinterpret_cast<const uint4*>(nw + k);
          const float2 n0 = bf2_to_f2(wq.x), n1 = bf2_to_f2(wq.y), n2 = bf2_to_f2(wq.z),
                       n3 = bf2_to_f2(wq.w);
#pragma unroll
          for (int b = 0; b < MB; ++b) {
            if (b >= M) break;
            const float r = rstd[b];
            const float4 a = *reinterpret_cast<const float4*>(xf + (size_t)b * K + k);
            const float4 c = *reinterpret_cast<const float4*>(xf + (size_t)b * K + k + 4);
            xq[b] = make_uint4(f2_to_bf2(a.x * r * n0.x, a.y * r * n0.y),
                               f2_to_bf2(a.z * r * n1.x, a.w * r * n1.y),
                               f2_to_bf2(c.x * r * n2.x, c.y * r * n2.y),
                               f2_to_bf2(c.z * r * n3.x, c.w * r * n3.y));
          }
        } else {
#pragma unroll
          for (int b = 0; b < MB; ++b)
            if (b < M) xq[b] = *reinterpret_cast<const uint4*>(xb + (size_t)b * K + k);
        }
      }
      mbar_wait(&full[s], (it / DS_STAGES) & 1);
      if (k < K) {
        const uint8_t* st = smem + DS_OFF_RING + s * DS_STAGE_BYTES + (warp * 256 + lane * 8) * 2;
        uint4 wv[DS_ROWS];
#pragma unroll
        for (int j = 0; j < DS_ROWS; ++j)
          wv[j] = *reinterpret_cast<const uint4*>(st + j * DS_ROW_BYTES);
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          if (b >= M) break;
          const float2 x0 = bf2_to_f2(xq[b].x), x1 = bf2_to_f2(xq[b].y),
                       x2 = bf2_to_f2(xq[b].z), x3 = bf2_to_f2(xq[b].w);
#pragma unroll
          for (int j = 0; j < DS_ROWS; ++j) {
            const float2 w0 = bf2_to_f2(wv[j].x), w1 = bf2_to_f2(wv[j].y),
                         w2 = bf2_to_f2(wv[j].z), w3 = bf2_to_f2(wv[j].w);
            float a = acc[j][b];
            a = fmaf(x0.x, w0.x, a); a = fmaf(x0.y, w0.y, a);
            a = fmaf(x1.x, w1.x, a); a = fmaf(x1.y, w1.y, a);
            a = fmaf(x2.x, w2.x, a); a = fmaf(x2.y, w2.y, a);
            a = fmaf(x3.x, w3.x, a); a = fmaf(x3.y, w3.y, a);
            acc[j][b] = a;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    float* pb = part + (parity & 1) * DS_CWARPS * DS_ROWS * DS_MAXB;
#pragma unroll
    for (int j = 0; j < DS_ROWS; ++j)
#pragma unroll
      for (int b = 0; b < MB; ++b) {
        if (b >= M) break;
        const float v = warp_sum(acc[j][b]);
        if (lane == 0) pb[(warp * DS_ROWS + j) * DS_MAXB + b] = v;
      }
    cbar();
    if (warp == 0) {
      // lane e = b*4 + j  (M*4 <= 32)
      const int b = lane >> 2, j = lane & 3;
      const bool active = b < M;
      float v = 0.f;
      if (active) {
#pragma unroll
        for (int w = 0; w < DS_CWARPS; ++w)
          v += pb[(w * DS_ROWS + j) * DS_MAXB + b];
      }
      const float u = __shfl_down_sync(0xffffffffu, v, 2);
      if (active) {
        if (m.swiglu) {
          const int nout = N >> 1, oi = item * 2 + j;
          if (j < 2 && oi < nout)
            reinterpret_cast<__nv_bfloat16*>(out)[(size_t)b * nout + oi] =
                __float2bfloat16(v / (1.f + __expf(-v)) * u);
        } else {
          const int r = ds_row(item, j, false);
          if (r < N) {
            const size_t idx = (size_t)b * N + r;
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
}

__device__ __forceinline__ void ds_rope4(float* a, float* b, int i0, float pos, float l2t) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float inv_freq = exp2f(-l2t * (float)(2 * (i0 + j)) / (float)DS_D);
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    const float x = a[j], y = b[j];
    a[j] = x * cs - y * sn;
    b[j] = y * cs + x * sn;
  }
}

// ---------------------------------------------------- attention phase
// Item = (sequence b, kv head kh, partition p), about one per CTA.  The ring
// memory is idle here (the producer waits on attn_done), so a partition of up
// to DS_CAP tokens is gathered in ONE cp.async wave (K and V through the block
// table), then scored, soft-maxed and reduced with a handful of barriers; a
// longer partition loops over waves with an online-softmax rescale.  The
// current token's rotated k and its v are written to the pool once and
// patched into the wave that holds it.  Each item publishes (o, m, l); the
// last CTA of (b, kh) merges the partitions.
__device__ void attention_phase(const swb_decode_params& P, int layer, const DSWork& W,
                                uint8_t* smem, float scale_log2, float l2t, uint64_t* attn_bar,
                                int& attn_phase_bit) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = P.n_heads, Hkv = P.n_kv_heads, G = H / Hkv, bs = P.block_size;
  const int lbs = __ffs(bs) - 1;                    // block size is a power of two
  const int NP = ds_num_parts(P.batch, Hkv, P.max_ctx, gridDim.x);
  const int part = ((P.max_ctx + NP - 1) / NP + 15) / 16 * 16;
  const int qkv_cols = (H + 2 * Hkv) * DS_D;
  __nv_bfloat16* kpool = reinterpret_cast<__nv_bfloat16*>(
      static_cast<char*>(P.k_base) + (size_t)layer * P.layer_stride_bytes);
  __nv_bfloat16* vpool = reinterpret_cast<__nv_bfloat16*>(
      static_cast<char*>(P.v_base) + (size_t)layer * P.layer_stride_bytes);
  const __nv_bfloat16* qkv = reinterpret_cast<const __nv_bfloat16*>(P.qkv);
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem + DS_OFF_K);
  __nv_bfloat16* sv = reinterpret_cast<__nv_bfloat16*>(smem + DS_OFF_V);
  __nv_bfloat16* curk = reinterpret_cast<__nv_bfloat16*>(smem + DS_OFF_CUR);
  __nv_bfloat16* curv = curk + DS_D;
  float* sq = reinterpret_cast<float*>(smem + DS_OFF_SQ);
  float* ss = reinterpret_cast<float*>(smem + DS_OFF_SS);
  float* sacc = reinterpret_cast<float*>(smem + DS_OFF_SACC);
  float* sm_ = reinterpret_cast<float*>(smem + DS_OFF_SSTAT);   // running max [G]
  float* sl_ = sm_ + DS_MAXG;                                     // running sum [G]
  float* sc_ = sl_ + DS_MAXG;                                     // wave rescale [G]
  int* s_last = reinterpret_cast<int*>(smem + DS_OFF_MISC);
  const int n_items = P.batch * Hkv * NP;
  auto tp = [&](int k) {
    if (W.trace && blockIdx.x == 0 && threadIdx.x == 0 && layer < 100)
      W.trace[1024 + layer * 8 + k] = globaltimer();
  };
  tp(0);
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int b = item / (Hkv * NP), rem = item % (Hkv * NP);
    const int kh = rem / NP, p = rem % NP;
    const int ctx = P.attn_len[b];
    const int cur = ctx - 1;
    const int t0 = p * part, t1 = min(ctx, t0 + part);
    float* wsb = W.part + (((size_t)b * H) * NP) * (DS_D + 2);
    auto wsp = [&](int gh, int pp) { return wsb + ((size_t)gh * NP + pp) * (DS_D + 2); };
    if (t0 >= t1) {
      if (threadIdx.x < G) {
        float* w = wsp(kh * G + threadIdx.x, p);
        w[DS_D] = -INFINITY;
        w[DS_D + 1] = 0.f;
      }
    } else {
      const int32_t* trow = P.block_tables + (size_t)b * P.max_blocks;
      const __nv_bfloat16* qrow = qkv + (size_t)b * qkv_cols;
      const float fpos = (float)cur;
      tp(7);
      if (threadIdx.x < G * 16) {
        const int gi = threadIdx.x / 16, i0 = (threadIdx.x % 16) * 4;
        const __nv_bfloat16* hp = qrow + (kh * G + gi) * DS_D;
        float lo[4], hi[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          lo[j] = __bfloat162float(hp[i0 + j]);
          hi[j] = __bfloat162float(hp[64 + i0 + j]);
        }
        ds_rope4(lo, hi, i0, fpos, l2t);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sq[gi * DS_D + i0 + j] = __bfloat162float(__float2bfloat16(lo[j])) * scale_log2;
          sq[gi * DS_D + 64 + i0 + j] = __bfloat162float(__float2bfloat16(hi[j])) * scale_log2;
        }
      } else if (threadIdx.x >= 128 && threadIdx.x < 144 && cur >= t0 && cur < t1) {
        const int i0 = (threadIdx.x - 128) * 4;
        const __nv_bfloat16* kp = qrow + (H + kh) * DS_D;
        const __nv_bfloat16* vp = qrow + (H + Hkv + kh) * DS_D;
        float lo[4], hi[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          lo[j] = __bfloat162float(kp[i0 + j]);
          hi[j] = __bfloat162float(kp[64 + i0 + j]);
        }
        ds_rope4(lo, hi, i0, fpos, l2t);
        const int slot = P.slots[b];
        const size_t g = (((size_t)(slot / bs) * Hkv + kh) * bs + slot % bs) * DS_D;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const __nv_bfloat16 kl = __float2bfloat16(lo[j]), khv = __float2bfloat16(hi[j]);
          kpool[g + i0 + j] = kl;
          kpool[g + 64 + i0 + j] = khv;
          curk[i0 + j] = kl;
          curk[64 + i0 + j] = khv;
          vpool[g + i0 + j] = vp[i0 + j];
          vpool[g + 64 + i0 + j] = vp[64 + i0 + j];
          curv[i0 + j] = vp[i0 + j];
          curv[64 + i0 + j] = vp[64 + i0 + j];
        }
      }
      tp(6);
      if (threadIdx.x < G) {
        sm_[threadIdx.x] = -INFINITY;
        sl_[threadIdx.x] = 0.f;
      }
      float acc[DS_MAXG][4];
#pragma unroll
      for (int gi = 0; gi < DS_MAXG; ++gi) acc[gi][0] = acc[gi][1] = acc[gi][2] = acc[gi][3] = 0.f;
      float* wred = sacc + DS_CWARPS * DS_MAXG * DS_D;   // [16][G] partial max / sum
      float lsum[DS_MAXG] = {0.f, 0.f, 0.f, 0.f};
      for (int w0 = t0; w0 < t1; w0 += DS_CAP) {          // load waves
        const int ntok = min(DS_CAP, t1 - w0);
        // one thread gathers the wave with 4 KB bulk copies: each (block, kv
        // head) tile of 16 tokens is contiguous in the pool
        if (warp == 0) {
          // lanes fetch their block ids in parallel, then each issues its tiles
          const int nblk = (ntok + bs - 1) >> lbs;
          const uint32_t tile = (uint32_t)bs * DS_D * 2;
          if (lane == 0) mbar_arrive_expect_tx(attn_bar, 2 * tile * nblk);
          __syncwarp();
          const uint64_t pol = ds_policy();
          for (int j = lane; j < nblk; j += 32) {
            const int blk = __ldg(trow + ((w0 >> lbs) + j));
            const size_t g = ((size_t)blk * Hkv + kh) * bs * DS_D;
            ds_bulk(sk + (size_t)j * bs * DS_D, kpool + g, tile, attn_bar, pol);
            ds_bulk(sv + (size_t)j * bs * DS_D, vpool + g, tile, attn_bar, pol);
          }
        }
        tp(1);
        mbar_wait(attn_bar, attn_phase_bit);
        attn_phase_bit ^= 1;
        if (cur >= w0 && cur < w0 + ntok && threadIdx.x < 32) {   // patch the current token
          const int tt = cur - w0;
          if (threadIdx.x < 16)
            reinterpret_cast<uint4*>(sk + tt * DS_D)[threadIdx.x] =
                reinterpret_cast<const uint4*>(curk)[threadIdx.x];
          else
            reinterpret_cast<uint4*>(sv + tt * DS_D)[threadIdx.x - 16] =
                reinterpret_cast<const uint4*>(curv)[threadIdx.x - 16];
        }
        cbar();
        tp(2);
        {  // scores: half-warp per token, 4 tokens in flight per half-warp
          const int half = lane >> 4, hl = lane & 15;
          for (int tb = (warp * 2 + half); tb < ntok + 3 * DS_CWARPS * 2; tb += 4 * DS_CWARPS * 2) {
            float kf[4][8];
            bool valid[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int tt = tb + u * DS_CWARPS * 2;
              valid[u] = tt < ntok;
              const uint4 kv =
                  *reinterpret_cast<const uint4*>(sk + (valid[u] ? tt : 0) * DS_D + hl * 8);
              float2 a = bf2_to_f2(kv.x), c2 = bf2_to_f2(kv.y), e = bf2_to_f2(kv.z),
                     f = bf2_to_f2(kv.w);
              kf[u][0] = a.x; kf[u][1] = a.y; kf[u][2] = c2.x; kf[u][3] = c2.y;
              kf[u][4] = e.x; kf[u][5] = e.y; kf[u][6] = f.x; kf[u][7] = f.y;
            }
            for (int gi = 0; gi < G; ++gi) {
              const float4 q0 = *reinterpret_cast<const float4*>(sq + gi * DS_D + hl * 8);
              const float4 q1 = *reinterpret_cast<const float4*>(sq + gi * DS_D + hl * 8 + 4);
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
                for (int u = 0; u < 4; ++u)
                  if (valid[u]) ss[gi * DS_CAP + tb + u * DS_CWARPS * 2] = d[u];
              }
            }
          }
        }
        cbar();
        // wave max per head: every warp reduces a token slice, then all combine
        for (int gi = 0; gi < G; ++gi) {
          float mx = -INFINITY;
          for (int i = warp * 32 + lane; i < ntok; i += DS_CWARPS * 32)
            mx = fmaxf(mx, ss[gi * DS_CAP + i]);
          mx = warp_max(mx);
          if (lane == 0) wred[warp * DS_MAXG + gi] = mx;
        }
        cbar();
        float corr[DS_MAXG], mnew[DS_MAXG];
#pragma unroll
        for (int gi = 0; gi < DS_MAXG; ++gi) {
          if (gi >= G) break;
          float mx = -INFINITY;
          for (int w = 0; w < DS_CWARPS; ++w) mx = fmaxf(mx, wred[w * DS_MAXG + gi]);
          const float mold = sm_[gi];
          mnew[gi] = fmaxf(mold, mx);
          corr[gi] = mold == -INFINITY ? 0.f : exp2f(mold - mnew[gi]);
          acc[gi][0] *= corr[gi]; acc[gi][1] *= corr[gi];
          acc[gi][2] *= corr[gi]; acc[gi][3] *= corr[gi];
          lsum[gi] *= corr[gi];
        }
        // P.V with the exponentials computed on the fly; lsum per warp
        for (int tt = warp; tt < ntok; tt += DS_CWARPS) {
          const uint2 vv = *reinterpret_cast<const uint2*>(sv + tt * DS_D + lane * 4);
          const float2 v0 = bf2_to_f2(vv.x), v1 = bf2_to_f2(vv.y);
#pragma unroll
          for (int gi = 0; gi < DS_MAXG; ++gi) {
            if (gi >= G) break;
            const float pw = exp2f(ss[gi * DS_CAP + tt] - mnew[gi]);
            lsum[gi] += pw;
            acc[gi][0] = fmaf(pw, v0.x, acc[gi][0]);
            acc[gi][1] = fmaf(pw, v0.y, acc[gi][1]);
            acc[gi][2] = fmaf(pw, v1.x, acc[gi][2]);
            acc[gi][3] = fmaf(pw, v1.y, acc[gi][3]);
          }
        }
        cbar();  // K/V/scores/wred reused by the next wave (or by sacc below)
        if (threadIdx.x < G) sm_[threadIdx.x] = mnew[threadIdx.x];
        tp(3);
      }
      // cross-warp reduction (sacc aliases the K buffer)
#pragma unroll
      for (int gi = 0; gi < DS_MAXG; ++gi) {
        if (gi >= G) break;
        *reinterpret_cast<float4*>(sacc + ((size_t)warp * G + gi) * DS_D + lane * 4) =
            make_float4(acc[gi][0], acc[gi][1], acc[gi][2], acc[gi][3]);
      }
      if (lane == 0) {
#pragma unroll
        for (int gi = 0; gi < DS_MAXG; ++gi)
          if (gi < G) wred[warp * DS_MAXG + gi] = lsum[gi];
      }
      cbar();
      if (threadIdx.x < G * DS_D) {
        const int gi = threadIdx.x / DS_D, d = threadIdx.x % DS_D;
        float v = 0.f;
        for (int w = 0; w < DS_CWARPS; ++w) v += sacc[((size_t)w * G + gi) * DS_D + d];
        float* wo = wsp(kh * G + gi, p);
        wo[d] = v;
        if (d == 0) {
          float l = 0.f;
          for (int w = 0; w < DS_CWARPS; ++w) l += wred[w * DS_MAXG + gi];
          wo[DS_D] = sm_[gi];
          wo[DS_D + 1] = l;
        }
      }
    }
    // last CTA of (b, kh) merges the partitions
    tp(4);
    __threadfence();
    cbar();
    if (threadIdx.x == 0) {
      int* t = W.tickets + (size_t)b * Hkv + kh;
      const int prev = atomicAdd(t, 1);
      *s_last = prev == NP - 1;
      if (*s_last) *t = 0;
    }
    cbar();
    if (*s_last) {
      __threadfence();
      if (threadIdx.x < G * DS_D) {
        const int gi = threadIdx.x / DS_D, d = threadIdx.x % DS_D;
        const int gh = kh * G + gi;
        float mx = -INFINITY;
        for (int pp = 0; pp < NP; ++pp) mx = fmaxf(mx, __ldcg(wsp(gh, pp) + DS_D));
        float l = 0.f, o = 0.f;
        for (int pp = 0; pp < NP; ++pp) {
          const float* w = wsp(gh, pp);
          const float mp = __ldcg(w + DS_D);
          if (mp == -INFINITY) continue;
          const float f = exp2f(mp - mx);
          l += __ldcg(w + DS_D + 1) * f;
          o += __ldcg(w + d) * f;
        }
        reinterpret_cast<__nv_bfloat16*>(P.attn)[((size_t)b * H + gh) * DS_D + d] =
            __float2bfloat16(o / l);
      }
    }
    cbar();  // scratch reuse by the next item
    tp(5);
  }
}

template <int MB>
__global__ void __launch_bounds__(DS_THREADS, 1)
    decode_step_kernel(const swb_decode_params P, const DSWork W) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DS_OFF_BAR);
  uint64_t* empty = full + DS_STAGES;
  uint64_t* attn_done = empty + DS_STAGES;
  uint64_t* attn_bar = attn_done + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = P.num_layers, d = P.d_model;
  const int qkv_cols = (P.n_heads + 2 * P.n_kv_heads) * DS_D;
  const int hd = P.n_heads * DS_D;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], DS_CWARPS);
    }
    mbar_init(attn_done, 1);
    mbar_init(attn_bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) reinterpret_cast<int*>(smem + DS_OFF_MISC)[threadIdx.x] = 0;
  __syncthreads();
  const swb_decode_layer* layers = P.layers;

  if (warp == DS_CWARPS) {
    // ================================ producer: every matrix of the step
    if (lane == 0) {
      const uint64_t pol = ds_policy();
      int it = 0;
      for (int l = 0; l < L; ++l) {
        const swb_decode_layer ly = layers[l];
        produce_matrix({(const __nv_bfloat16*)ly.wqkv, qkv_cols, d, false}, smem, full, empty,
                       it, pol);
        mbar_wait_sleep(attn_done, l & 1);   // ring memory is attention scratch until then
        produce_matrix({(const __nv_bfloat16*)ly.wo, d, hd, false}, smem, full, empty, it, pol);
        produce_matrix({(const __nv_bfloat16*)ly.wgu, 2 * P.ffn, d, true}, smem, full, empty,
                       it, pol);
        produce_matrix({(const __nv_bfloat16*)ly.wd, d, P.ffn, false}, smem, full, empty, it,
                       pol);
      }
      produce_matrix({(const __nv_bfloat16*)P.lm_head, P.vocab, d, false}, smem, full, empty,
                     it, pol);
    }
    return;
  }

  // ================================== consumers
  const int B = P.batch;
  unsigned epoch = 0;
  int it = 0, parity = 0, attn_bit = 0;
  const float l2t = log2f(P.rope_theta);
  const float scale_log2 = rsqrtf((float)DS_D) * 1.4426950408889634f;
  // P0: positions / slots / attention lengths, embedding of the current tokens
  if (blockIdx.x == 0 && threadIdx.x < B) {
    const int b = threadIdx.x;
    const int c = P.ctx[b];
    P.pos[b] = c;
    P.slots[b] = P.block_tables[(size_t)b * P.max_blocks + c / P.block_size] * P.block_size +
                 c % P.block_size;
    P.attn_len[b] = c + 1;
  }
  {
    const __nv_bfloat16* E = reinterpret_cast<const __nv_bfloat16*>(P.embed);
    const int chunks = B * d / 8;
    for (int i = blockIdx.x * DS_CWARPS * 32 + threadIdx.x; i < chunks;
         i += gridDim.x * DS_CWARPS * 32) {
      const int b = (i * 8) / d, c = (i * 8) % d;
      const uint4 v = *reinterpret_cast<const uint4*>(E + (size_t)P.cur_tok[b] * d + c);
      float4* dst = reinterpret_cast<float4*>(P.x + (size_t)b * d + c);
      const float2 a = bf2_to_f2(v.x), e = bf2_to_f2(v.y), f = bf2_to_f2(v.z), g = bf2_to_f2(v.w);
      dst[0] = make_float4(a.x, a.y, e.x, e.y);
      dst[1] = make_float4(f.x, f.y, g.x, g.y);
    }
  }
  grid_sync(W.barrier, epoch, W.trace);
  for (int l = 0; l < L; ++l) {
    const swb_decode_layer ly = layers[l];
    consume_matrix<MB>({(const __nv_bfloat16*)ly.wqkv, qkv_cols, d, false}, P.x,
                       (const __nv_bfloat16*)ly.attn_norm, P.norm_eps, B, SWB_EPI_BF16, P.qkv,
                       nullptr, smem, full, empty, it, parity);
    grid_sync(W.barrier, epoch, W.trace);
    attention_phase(P, l, W, smem, scale_log2, l2t, attn_bar, attn_bit);  // ends with cbar
    if (threadIdx.x == 0) mbar_arrive(attn_done);      // ring free: prefetch Wo
    grid_sync(W.barrier, epoch, W.trace);
    consume_matrix<MB>({(const __nv_bfloat16*)ly.wo, d, hd, false}, P.attn, nullptr, 0.f, B,
                       SWB_EPI_RESID_F32, P.x, P.x, smem, full, empty, it, parity);
    grid_sync(W.barrier, epoch, W.trace);
    consume_matrix<MB>({(const __nv_bfloat16*)ly.wgu, 2 * P.ffn, d, true}, P.x,
                       (const __nv_bfloat16*)ly.mlp_norm, P.norm_eps, B, SWB_EPI_SWIGLU, P.act,
                       nullptr, smem, full, empty, it, parity);
    grid_sync(W.barrier, epoch, W.trace);
    consume_matrix<MB>({(const __nv_bfloat16*)ly.wd, d, P.ffn, false}, P.act, nullptr, 0.f, B,
                       SWB_EPI_RESID_F32, P.x, P.x, smem, full, empty, it, parity);
    grid_sync(W.barrier, epoch, W.trace);
  }
  consume_matrix<MB>({(const __nv_bfloat16*)P.lm_head, P.vocab, d, false}, P.x,
                     (const __nv_bfloat16*)P.final_norm, P.norm_eps, B, SWB_EPI_F32, P.logits,
                     nullptr, smem, full, empty, it, parity);
  grid_sync(W.barrier, epoch, W.trace);
  // G: greedy argmax (lowest index on ties) + advance, CTA b handles row b
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    const float* row = P.logits + (size_t)b * P.vocab;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < P.vocab; i += DS_CWARPS * 32) {
      const float v = __ldcg(row + i);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    float* sb = reinterpret_cast<float*>(smem + DS_OFF_SACC);
    int* si = reinterpret_cast<int*>(sb + DS_CWARPS);
    if (lane == 0) {
      sb[warp] = best;
      si[warp] = bi;
    }
    cbar();
    if (threadIdx.x == 0) {
      float bb = sb[0];
      int ii = si[0];
      for (int w = 1; w < DS_CWARPS; ++w)
        if (sb[w] > bb || (sb[w] == bb && si[w] < ii)) {
          bb = sb[w];
          ii = si[w];
        }
      P.cur_tok[b] = ii;
      const int s = P.step[b];
      if (s < P.ring_len) P.out_ring[(size_t)b * P.ring_len + s] = ii;
      P.step[b] = s + 1;
      P.ctx[b] += 1;
    }
  }
}

}  // namespace swb

using namespace swb;

extern "C" size_t swb_decode_step_workspace(const swb_decode_params* p) {
  if (!p || p->batch <= 0) return 0;
  const size_t NP = ds_num_parts(p->batch, p->n_kv_heads, p->max_ctx, kNumSMs);
  const size_t tick_bytes = ((size_t)p->batch * p->n_kv_heads * sizeof(int) + 127) / 128 * 128;
  return 2048 * 8 + 128 + tick_bytes +
         (size_t)p->batch * p->n_heads * NP * (DS_D + 2) * sizeof(float);
}

extern "C" int swb_decode_step(const swb_decode_params* p, uintptr_t stream) {
  SWB_REQUIRE(p, "swb_decode_step: null params");
  SWB_REQUIRE(p->batch >= 1 && p->batch <= DS_MAXB, "swb_decode_step: batch %d outside 1..%d",
              p->batch, DS_MAXB);
  SWB_REQUIRE(p->head_dim == DS_D, "swb_decode_step: head_dim must be 128");
  SWB_REQUIRE(p->n_heads % p->n_kv_heads == 0 && p->n_heads / p->n_kv_heads <= DS_MAXG,
              "swb_decode_step: GQA group must be <= %d", DS_MAXG);
  SWB_REQUIRE(p->d_model % 8 == 0 && p->ffn % 128 == 0 && p->vocab > 0,
              "swb_decode_step: bad model dims");
  SWB_REQUIRE(p->block_size > 0 && (p->block_size & (p->block_size - 1)) == 0,
              "swb_decode_step: block_size must be a power of two");
  SWB_REQUIRE(p->layers && p->embed && p->lm_head && p->final_norm && p->k_base && p->v_base &&
                  p->x && p->qkv && p->attn && p->act && p->logits && p->cur_tok && p->ctx &&
                  p->step && p->out_ring && p->pos && p->slots && p->attn_len &&
                  p->block_tables && p->workspace,
              "swb_decode_step: null pointer in params");
  const size_t NP = ds_num_parts(p->batch, p->n_kv_heads, p->max_ctx, kNumSMs);
  // workspace: trace [2048] u64 | barrier (128 B) | tickets | partials
  DSWork W;
  char* base = static_cast<char*>(p->workspace);
  W.trace = reinterpret_cast<unsigned long long*>(base);
  W.barrier = reinterpret_cast<unsigned*>(base + 2048 * 8);
  W.tickets = reinterpret_cast<int*>(base + 2048 * 8 + 128);
  const size_t tick_bytes = ((size_t)p->batch * p->n_kv_heads * sizeof(int) + 127) / 128 * 128;
  W.part = reinterpret_cast<float*>(base + 2048 * 8 + 128 + tick_bytes);
  (void)NP;
  cudaStream_t s = (cudaStream_t)stream;
  SWB_CUDA(cudaMemsetAsync(W.barrier, 0, sizeof(unsigned), s));
  int dev = 0;
  SWB_CUDA(cudaGetDevice(&dev));
  static bool attr[64][4] = {};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNumSMs);
  cfg.blockDim = dim3(DS_THREADS);
  cfg.dynamicSmemBytes = DS_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all 148 CTAs co-resident (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e;
#define DS_LAUNCH(MBV, IDX)                                                              \
  do {                                                                                   \
    if (dev < 64 && !attr[dev][IDX]) {                                                   \
      SWB_CUDA(cudaFuncSetAttribute(decode_step_kernel<MBV>,                             \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, DS_SMEM)); \
      attr[dev][IDX] = true;                                                             \
    }                                                                                    \
    e = cudaLaunchKernelEx(&cfg, decode_step_kernel<MBV>, *p, W);                        \
  } while (0)
  if (p->batch == 1)
    DS_LAUNCH(1, 0);
  else if (p->batch <= 2)
    DS_LAUNCH(2, 1);
  else if (p->batch <= 4)
    DS_LAUNCH(4, 2);
  else
    DS_LAUNCH(8, 3);
#undef DS_LAUNCH
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch decode_step_kernel: %s", cudaGetErrorString(e));
  return swb_check_launch("decode_step_kernel");
}
