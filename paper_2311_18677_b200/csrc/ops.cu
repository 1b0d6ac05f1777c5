// Element-wise / row-wise kernels of the prefill and decode layers, the
// RoPE + paged-KV write, the per-layer KV pack-and-push, completion flags and
// the graph-resident decode bookkeeping.
//
// KV block layout (per layer, K and V separately):
//     [num_blocks][Hkv][block_size][dh] bf16
// A token at logical position p of a sequence lives in physical slot
//     slot = block_table[p / block_size] * block_size + p % block_size.
// One (block, head) is block_size*dh*2 bytes contiguous (4 KB at bs=16,
// dh=128), which is the unit the decode-attention kernel streams.
#include <cudaTypedefs.h>

#include <cstring>

#include "common.cuh"

namespace swb {

// ------------------------------------------------------------------ embed
__global__ void embed_kernel(const int32_t* __restrict__ tokens,
                             const __nv_bfloat16* __restrict__ table,
                             float* __restrict__ x, int d) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int tok = tokens[r];
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)tok * d);
  float4* dst = reinterpret_cast<float4*>(x + (size_t)r * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    const uint4 v = src[c];
    const float2 a = bf2_to_f2(v.x), b = bf2_to_f2(v.y), e = bf2_to_f2(v.z),
                 f = bf2_to_f2(v.w);
    dst[2 * c] = make_float4(a.x, a.y, b.x, b.y);
    dst[2 * c + 1] = make_float4(e.x, e.y, f.x, f.y);
  }
}

// ---------------------------------------------------------------- rmsnorm
// LayerNorm (BLOOM): out = (x - mean) * rstd * w + b over fp32 rows, two
// passes over the (L1/L2-resident) row; bf16 or fp32 output (the embedding
// LayerNorm produces the fp32 residual stream, possibly in place).
// addend (optional, bf16 [rows of x]): x[src] += addend[src] first, written
// back (the TP prefill's bf16 all-reduce result joins the fp32 residual here).
// With several addends (the TP ranks' partials, copy-engine exchange) their
// fp32 sum in the given order is added: x += (p0 + p1 + ...).
struct Addends {
  const __nv_bfloat16* p[8];
  int n;
};
__device__ __forceinline__ float4 add_row4(float* x, const Addends& ad, size_t i4) {
  float4 v = reinterpret_cast<float4*>(x)[i4];
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < ad.n; ++k) {
    const uint2 a = reinterpret_cast<const uint2*>(ad.p[k])[i4];
    const float2 a0 = bf2_to_f2(a.x), a1 = bf2_to_f2(a.y);
    if (k == 0) {
      s = make_float4(a0.x, a0.y, a1.x, a1.y);
    } else {
      s.x += a0.x; s.y += a0.y; s.z += a1.x; s.w += a1.y;
    }
  }
  v.x += s.x; v.y += s.y; v.z += s.z; v.w += s.w;
  reinterpret_cast<float4*>(x)[i4] = v;
  return v;
}

__global__ void layernorm_kernel(const float* x, const int32_t* __restrict__ row_index,
                                 const __nv_bfloat16* __restrict__ w,
                                 const __nv_bfloat16* __restrict__ b, void* out, int d,
                                 float eps, int out_f32, const __grid_constant__ Addends addend) {
  pdl_wait();
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)src * d);
  __shared__ float red[32];
  __shared__ float stat[2];
  float s = 0.f;
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 v = addend.n ? add_row4(const_cast<float*>(x), addend, (size_t)src * (d / 4) + c)
                              : xr[c];
    s += (v.x + v.y) + (v.z + v.w);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) stat[0] = v / (float)d;
  }
  __syncthreads();
  const float mean = stat[0];
  float ss = 0.f;
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 v = xr[c];
    const float a0 = v.x - mean, a1 = v.y - mean, a2 = v.z - mean, a3 = v.w - mean;
    ss += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
  ss = warp_sum(ss);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) stat[1] = rsqrtf(v / (float)d + eps);
  }
  __syncthreads();
  const float rstd = stat[1];
  const uint2* wv = reinterpret_cast<const uint2*>(w);
  const uint2* bv = reinterpret_cast<const uint2*>(b);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 v = xr[c];
    const uint2 ww = wv[c], bb = bv[c];
    const float2 w0 = bf2_to_f2(ww.x), w1 = bf2_to_f2(ww.y);
    const float2 b0 = bf2_to_f2(bb.x), b1 = bf2_to_f2(bb.y);
    const float o0 = (v.x - mean) * rstd * w0.x + b0.x, o1 = (v.y - mean) * rstd * w0.y + b0.y;
    const float o2 = (v.z - mean) * rstd * w1.x + b1.x, o3 = (v.w - mean) * rstd * w1.y + b1.y;
    if (out_f32)
      reinterpret_cast<float4*>(out)[(size_t)r * (d / 4) + c] = make_float4(o0, o1, o2, o3);
    else
      reinterpret_cast<uint2*>(out)[(size_t)r * (d / 4) + c] =
          make_uint2(f2_to_bf2(o0, o1), f2_to_bf2(o2, o3));
  }
}

__global__ void rmsnorm_kernel(const float* x, const int32_t* __restrict__ row_index,
                               const __nv_bfloat16* __restrict__ w,
                               __nv_bfloat16* __restrict__ out, int d, float eps,
                               const __grid_constant__ Addends addend) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)src * d);
  float ss = 0.f;
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 v = addend.n ? add_row4(const_cast<float*>(x), addend, (size_t)src * (d / 4) + c)
                              : xr[c];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float rstd = rsqrtf(red[0] / (float)d + eps);
  const uint2* wv = reinterpret_cast<const uint2*>(w);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)r * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 v = xr[c];
    const uint2 ww = wv[c];
    const float2 w0 = bf2_to_f2(ww.x), w1 = bf2_to_f2(ww.y);
    o[c] = make_uint2(f2_to_bf2(v.x * rstd * w0.x, v.y * rstd * w0.y),
                      f2_to_bf2(v.z * rstd * w1.x, v.w * rstd * w1.y));
  }
}

// ----------------------------------------------------------------- argmax
__global__ void argmax_kernel(const float* __restrict__ logits, int V,
                              int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const float* row = logits + (size_t)blockIdx.x * V;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > best) {  // strided scan visits increasing i: first max kept
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
  __shared__ float sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sb[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = sb[0];
    int i0 = si[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sb[k] > b || (sb[k] == b && si[k] < i0)) {
        b = sb[k];
        i0 = si[k];
      }
    out[blockIdx.x] = i0;
  }
}

// ------------------------------------------------------ RoPE + KV write
// One CTA per row.  Thread t handles 4 consecutive rotary pairs (i..i+3 with
// partners i+dh/2..) of one q or k head; k heads are also written to the
// paged pool together with the matching v chunk.
__global__ void rope_kv_kernel(__nv_bfloat16* __restrict__ qkv, int row_stride,
                               const int32_t* __restrict__ positions, int H,
                               int Hkv, int dh, float log2_theta,
                               __nv_bfloat16* __restrict__ kpool,
                               __nv_bfloat16* __restrict__ vpool,
                               const int32_t* __restrict__ slots, int bs) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int half = dh >> 1;
  const int groups = half >> 2;  // 4 pairs per thread
  const float pos = (float)positions[r];
  __nv_bfloat16* row = qkv + (size_t)r * row_stride;
  const int total = (H + Hkv) * groups;
  int slot = 0;
  if (kpool) slot = slots[r];
  const int blk = slot / bs, off = slot % bs;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int head = t / groups;
    const int i0 = (t % groups) * 4;
    __nv_bfloat16* hp = row + head * dh;
    const uint2 lo = *reinterpret_cast<const uint2*>(hp + i0);
    const uint2 hi = *reinterpret_cast<const uint2*>(hp + half + i0);
    float a[4], b[4];
    {
      float2 t0 = bf2_to_f2(lo.x), t1 = bf2_to_f2(lo.y);
      a[0] = t0.x; a[1] = t0.y; a[2] = t1.x; a[3] = t1.y;
      t0 = bf2_to_f2(hi.x); t1 = bf2_to_f2(hi.y);
      b[0] = t0.x; b[1] = t0.y; b[2] = t1.x; b[3] = t1.y;
    }
    float ra[4], rb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (log2_theta > 0.f) {   // inv_freq = theta^(-2i/dh)
        rope_pair(a[j], b[j], i0 + j, pos, log2_theta, dh, ra[j], rb[j]);
      } else {  // no rotary embedding (ALiBi models): KV write only
        ra[j] = a[j];
        rb[j] = b[j];
      }
    }
    const uint2 nlo = make_uint2(f2_to_bf2(ra[0], ra[1]), f2_to_bf2(ra[2], ra[3]));
    const uint2 nhi = make_uint2(f2_to_bf2(rb[0], rb[1]), f2_to_bf2(rb[2], rb[3]));
    *reinterpret_cast<uint2*>(hp + i0) = nlo;
    *reinterpret_cast<uint2*>(hp + half + i0) = nhi;
    if (kpool && head >= H) {
      const int kh = head - H;
      const size_t base = (((size_t)blk * Hkv + kh) * bs + off) * dh;
      *reinterpret_cast<uint2*>(kpool + base + i0) = nlo;
      *reinterpret_cast<uint2*>(kpool + base + half + i0) = nhi;
      const __nv_bfloat16* vp = row + (H + Hkv + kh) * dh;
      *reinterpret_cast<uint2*>(vpool + base + i0) =
          *reinterpret_cast<const uint2*>(vp + i0);
      *reinterpret_cast<uint2*>(vpool + base + half + i0) =
          *reinterpret_cast<const uint2*>(vp + half + i0);
    }
  }
}

// ------------------------------------------------- KV pack-and-push (P2P)
// One warp per (row, K-or-V) unit: the row's Hkv*dh bf16 are contiguous in
// the source (the rotated qkv activations of one finished layer); lane l
// moves 16-byte chunks l, l+32, ... .  Each lane first issues all of its
// loads (up to 16 x 16 B in flight), then its stores, which land in the
// destination pool's paged blocks — a peer GPU's HBM mapped through CUDA
// IPC — as coalesced 256-byte NVLink writes per head.
constexpr int PUSH_UNROLL = 16;
// blockIdx.y = layer: the serialized mode pushes every layer of a finished
// prompt in one launch (layer strides in elements; 0 for the per-layer mode).
__global__ void __launch_bounds__(256)
    kv_push_kernel(const __nv_bfloat16* __restrict__ qkv, int rows, int row_stride,
                   int k_col, int v_col, int Hkv, int dh, __nv_bfloat16* __restrict__ dk,
                   __nv_bfloat16* __restrict__ dv, const int32_t* __restrict__ slots, int bs,
                   size_t src_layer_stride, size_t dst_layer_stride) {
  pdl_trigger();
  pdl_wait();
  qkv += blockIdx.y * src_layer_stride;
  dk += blockIdx.y * dst_layer_stride;
  dv += blockIdx.y * dst_layer_stride;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int cph = dh >> 3;                 // 16-byte chunks per head
  const int chunks = Hkv * cph;            // per row, per K or V
  for (int u = gw; u < rows * 2; u += nw) {
    const int r = u >> 1, is_v = u & 1;
    const __nv_bfloat16* src = qkv + (size_t)r * row_stride + (is_v ? v_col : k_col);
    const int slot = slots[r];
    const size_t dbase = (((size_t)(slot / bs) * Hkv) * bs + slot % bs) * dh;
    __nv_bfloat16* dst = (is_v ? dv : dk) + dbase;
    for (int c0 = 0; c0 < chunks; c0 += 32 * PUSH_UNROLL) {
      uint4 v[PUSH_UNROLL];
#pragma unroll
      for (int j = 0; j < PUSH_UNROLL; ++j) {
        const int c = c0 + j * 32 + lane;
        if (c < chunks) v[j] = ld_nc_v4(src + c * 8);
      }
#pragma unroll
      for (int j = 0; j < PUSH_UNROLL; ++j) {
        const int c = c0 + j * 32 + lane;
        if (c < chunks) {
          const int h = c / cph, w = c % cph;
          st_v4(dst + (size_t)h * bs * dh + w * 8, v[j]);
        }
      }
    }
  }
}

// Hand-off record of a finished prompt batch in the token machine's table
// (host-mapped shared memory or peer memory), per request i: word 1 = its
// first token (first[row[i]]), word 2 = the batch's group key, word 3 = how
// many records of this table the batch writes (the token machine admits a
// group only when all of it landed); the per-request flags (word 0) follow
// as stream memory operations (swb_kv_handoff).
constexpr int HANDOFF_MAX = 64;
struct HandoffBatch {
  int seq[HANDOFF_MAX];
  int row[HANDOFF_MAX];
};
__global__ void handoff_token_kernel(const int32_t* __restrict__ first, int n,
                                     HandoffBatch b, int key, char* base, int stride) {
  pdl_trigger();
  pdl_wait();
  const int i = threadIdx.x;
  if (i < n) {
    int32_t* rec = reinterpret_cast<int32_t*>(base + (size_t)b.seq[i] * stride);
    asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(rec + 1), "r"(first[b.row[i]])
                 : "memory");
    asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(rec + 2), "r"(key) : "memory");
    asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(rec + 3), "r"(n) : "memory");
  }
}

// ------------------------------------------ vocab-parallel greedy argmax
// TP pools split the LM head by vocabulary rows: rank r scores rows
// [offset, offset + V) and publishes its candidate (max logit, global index)
// in its slot of a [rows][tp][2] fp32 buffer (other slots zero) that the
// pool's all-reduce (a sum) turns into every rank's candidates; the pick
// takes the max, lowest global index on ties (= argmax over the full vocab).
__global__ void argmax_shard_kernel(const float* __restrict__ logits, int V, int offset,
                                    int rank, int tp, float* __restrict__ cand) {
  pdl_trigger();
  pdl_wait();
  const float* row = logits + (size_t)blockIdx.x * V;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
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
  __shared__ float sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sb[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (int)(blockDim.x >> 5) ? sb[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < (int)(blockDim.x >> 5) ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
  }
  float* c = cand + (size_t)blockIdx.x * tp * 2;
  if (threadIdx.x < tp) {
    const bool mine = (int)threadIdx.x == rank;
    c[2 * threadIdx.x] = mine ? best : 0.f;
    c[2 * threadIdx.x + 1] = mine ? (float)(bi + offset) : 0.f;
  }
}

__global__ void argmax_pick_kernel(const float* __restrict__ cand, int rows, int tp,
                                   int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float* c = cand + (size_t)r * tp * 2;
  float best = c[0];
  int bi = (int)c[1];
  for (int k = 1; k < tp; ++k) {        // ranks hold increasing index ranges
    if (c[2 * k] > best) {
      best = c[2 * k];
      bi = (int)c[2 * k + 1];
    }
  }
  out[r] = bi;
}

// -------------------------------------------------- decode bookkeeping
__global__ void decode_advance_kernel(const int32_t* __restrict__ next_tok,
                                      int32_t* __restrict__ cur_tok,
                                      int32_t* __restrict__ ctx,
                                      int32_t* __restrict__ step,
                                      int32_t* __restrict__ ring, int ring_len,
                                      int B) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int t = next_tok[b];
  cur_tok[b] = t;
  const int s = step[b];
  if (s < ring_len) ring[(size_t)b * ring_len + s] = t;
  step[b] = s + 1;
  ctx[b] += 1;
}

__global__ void slots_from_table_kernel(const int32_t* table_row, int start,
                                        int n, int bs, int32_t* slots) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = start + i;
  slots[i] = table_row[p / bs] * bs + p % bs;
}

}  // namespace swb

using namespace swb;

#define STREAM ((cudaStream_t)stream)

extern "C" int swb_embed(const int32_t* tokens, const void* table, float* x,
                         int rows, int d, uintptr_t stream) {
  SWB_REQUIRE(tokens && table && x, "swb_embed: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 8 == 0, "swb_embed: bad shape");
  if (rows == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(embed_kernel, dim3(rows), dim3(256), 0, STREAM,
        
      tokens, reinterpret_cast<const __nv_bfloat16*>(table), x, d);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch embed_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("embed_kernel");
}

static Addends one_addend(const void* a) {
  Addends ad;
  memset(&ad, 0, sizeof(ad));
  ad.p[0] = reinterpret_cast<const __nv_bfloat16*>(a);
  ad.n = a ? 1 : 0;
  return ad;
}

extern "C" int swb_add_rmsnorm(float* x, const void* addend, const int32_t* row_index,
                               const void* w, void* out, int rows, int d, float eps,
                               uintptr_t stream) {
  SWB_REQUIRE(x && w && out, "swb_add_rmsnorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_add_rmsnorm: bad shape");
  if (rows == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(rmsnorm_kernel, dim3(rows), dim3(512), 0, STREAM,
      x, row_index, reinterpret_cast<const __nv_bfloat16*>(w),
      reinterpret_cast<__nv_bfloat16*>(out), d, eps, one_addend(addend));
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch rmsnorm_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("rmsnorm_kernel");
}

extern "C" int swb_rmsnorm(const float* x, const int32_t* row_index, const void* w,
                           void* out, int rows, int d, float eps, uintptr_t stream) {
  SWB_REQUIRE(x && w && out, "swb_rmsnorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_rmsnorm: bad shape");
  if (rows == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(rmsnorm_kernel, dim3(rows), dim3(512), 0, STREAM,
      x, row_index, reinterpret_cast<const __nv_bfloat16*>(w),
      reinterpret_cast<__nv_bfloat16*>(out), d, eps, one_addend(nullptr));
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch rmsnorm_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("rmsnorm_kernel");
}

extern "C" int swb_layernorm(const float* x, const int32_t* row_index, const void* w,
                             const void* b, void* out, int rows, int d, float eps, int out_f32,
                             uintptr_t stream) {
  SWB_REQUIRE(x && w && b && out, "swb_layernorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_layernorm: bad shape");
  SWB_REQUIRE(!row_index || !out_f32 || (const void*)x != out,
              "swb_layernorm: gathered rows cannot be normalised in place");
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(layernorm_kernel, dim3(rows), dim3(512), 0, STREAM, x,
                                row_index, reinterpret_cast<const __nv_bfloat16*>(w),
                                reinterpret_cast<const __nv_bfloat16*>(b), out, d, eps, out_f32,
                                one_addend(nullptr));
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch layernorm_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("layernorm_kernel");
}

extern "C" int swb_add_layernorm(float* x, const void* addend, const int32_t* row_index,
                                 const void* w, const void* b, void* out, int rows, int d,
                                 float eps, uintptr_t stream) {
  SWB_REQUIRE(x && addend && w && b && out, "swb_add_layernorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_add_layernorm: bad shape");
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(layernorm_kernel, dim3(rows), dim3(512), 0, STREAM, x,
                                row_index, reinterpret_cast<const __nv_bfloat16*>(w),
                                reinterpret_cast<const __nv_bfloat16*>(b), out, d, eps, 0,
                                one_addend(addend));
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch layernorm_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("layernorm_kernel");
}

static int parts_addends(const char* fn, const void* const* parts, int n, Addends* ad) {
  SWB_REQUIRE(parts && n >= 1 && n <= 8, "%s: 1..8 partials, got %d", fn, n);
  memset(ad, 0, sizeof(*ad));
  for (int k = 0; k < n; ++k) {
    SWB_REQUIRE(parts[k] && ((uintptr_t)parts[k] & 7) == 0, "%s: partial %d null or unaligned",
                fn, k);
    ad->p[k] = reinterpret_cast<const __nv_bfloat16*>(parts[k]);
  }
  ad->n = n;
  return SWB_OK;
}

extern "C" int swb_add_parts_rmsnorm(float* x, const void* const* parts, int n_parts,
                                     const int32_t* row_index, const void* w, void* out, int rows,
                                     int d, float eps, uintptr_t stream) {
  SWB_REQUIRE(x && w && out, "swb_add_parts_rmsnorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_add_parts_rmsnorm: bad shape");
  Addends ad;
  const int st = parts_addends("swb_add_parts_rmsnorm", parts, n_parts, &ad);
  if (st) return st;
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(rmsnorm_kernel, dim3(rows), dim3(512), 0, STREAM, x, row_index,
                                reinterpret_cast<const __nv_bfloat16*>(w),
                                reinterpret_cast<__nv_bfloat16*>(out), d, eps, ad);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch rmsnorm_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("rmsnorm_kernel");
}

extern "C" int swb_add_parts_layernorm(float* x, const void* const* parts, int n_parts,
                                       const int32_t* row_index, const void* w, const void* b,
                                       void* out, int rows, int d, float eps, uintptr_t stream) {
  SWB_REQUIRE(x && w && b && out, "swb_add_parts_layernorm: null pointer");
  SWB_REQUIRE(rows >= 0 && d > 0 && d % 4 == 0, "swb_add_parts_layernorm: bad shape");
  Addends ad;
  const int st = parts_addends("swb_add_parts_layernorm", parts, n_parts, &ad);
  if (st) return st;
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(layernorm_kernel, dim3(rows), dim3(512), 0, STREAM, x,
                                row_index, reinterpret_cast<const __nv_bfloat16*>(w),
                                reinterpret_cast<const __nv_bfloat16*>(b), out, d, eps, 0, ad);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch layernorm_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("layernorm_kernel");
}

extern "C" int swb_argmax(const float* logits, int rows, int V, int32_t* out,
                          uintptr_t stream) {
  SWB_REQUIRE(logits && out, "swb_argmax: null pointer");
  SWB_REQUIRE(rows >= 0 && V > 0, "swb_argmax: bad shape");
  if (rows == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(argmax_kernel, dim3(rows), dim3(1024), 0, STREAM,
        logits, V, out);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch argmax_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("argmax_kernel");
}

extern "C" int swb_rope_kv_write(void* qkv, int rows, int row_stride,
                                 const int32_t* positions, int H, int Hkv, int dh,
                                 float theta, void* k_layer, void* v_layer,
                                 const int32_t* slots, int block_size,
                                 uintptr_t stream) {
  SWB_REQUIRE(qkv && positions, "swb_rope_kv_write: null pointer");
  SWB_REQUIRE(dh % 8 == 0 && H > 0 && Hkv > 0 && H % Hkv == 0,
              "swb_rope_kv_write: bad heads H=%d Hkv=%d dh=%d", H, Hkv, dh);
  SWB_REQUIRE(row_stride >= (H + 2 * Hkv) * dh, "swb_rope_kv_write: row_stride");
  SWB_REQUIRE((k_layer == nullptr) == (v_layer == nullptr),
              "swb_rope_kv_write: k/v pools must both be set or both null");
  SWB_REQUIRE(!k_layer || (slots && block_size > 0), "swb_rope_kv_write: slots");
  SWB_REQUIRE(theta > 1.f || theta == 0.f, "swb_rope_kv_write: theta (0 = no rotation)");
  if (rows == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(rope_kv_kernel, dim3(rows), dim3(256), 0, STREAM,
        
      reinterpret_cast<__nv_bfloat16*>(qkv), row_stride, positions, H, Hkv, dh,
      theta > 0.f ? log2f(theta) : 0.f, reinterpret_cast<__nv_bfloat16*>(k_layer),
      reinterpret_cast<__nv_bfloat16*>(v_layer), slots, block_size);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch rope_kv_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("rope_kv_kernel");
}

static int push_launch(const void* qkv, int rows, int row_stride, int k_col, int v_col,
                       int Hkv, int dh, void* dk, void* dv, const int32_t* dst_slots,
                       int block_size, int num_ctas, int layers, size_t src_layer_stride,
                       size_t dst_layer_stride, uintptr_t stream) {
  SWB_REQUIRE(qkv && dk && dv && dst_slots, "swb_kv_push: null pointer");
  SWB_REQUIRE(dh % 8 == 0 && Hkv > 0 && block_size > 0 && rows >= 0 && layers > 0,
              "swb_kv_push: bad shape");
  SWB_REQUIRE(row_stride % 8 == 0 && k_col % 8 == 0 && v_col % 8 == 0 &&
                  src_layer_stride % 8 == 0,
              "swb_kv_push: 16-byte alignment of rows/columns");
  if (rows == 0) return SWB_OK;
  int grid = num_ctas > 0 ? num_ctas : 64;
  const int need = (rows * 2 + 7) / 8;     // 8 warps per CTA, one (row, k|v) unit each
  if (need < grid) grid = need;
  const cudaError_t le_ = launch(kv_push_kernel, dim3(grid, layers), dim3(256), 0, STREAM,
      reinterpret_cast<const __nv_bfloat16*>(qkv), rows, row_stride, k_col, v_col,
      Hkv, dh, reinterpret_cast<__nv_bfloat16*>(dk), reinterpret_cast<__nv_bfloat16*>(dv),
      dst_slots, block_size, src_layer_stride, dst_layer_stride);
  if (le_ != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch kv_push_kernel: %s", cudaGetErrorString(le_));
  return swb_check_launch("kv_push_kernel");
}

extern "C" int swb_kv_push_layer(const void* qkv, int rows, int row_stride,
                                 int k_col, int v_col, int Hkv, int dh,
                                 void* dst_k_layer, void* dst_v_layer,
                                 const int32_t* dst_slots, int block_size,
                                 int num_ctas, uintptr_t stream) {
  return push_launch(qkv, rows, row_stride, k_col, v_col, Hkv, dh, dst_k_layer, dst_v_layer,
                     dst_slots, block_size, num_ctas, 1, 0, 0, stream);
}

extern "C" int swb_kv_push_layers(const void* qkv, size_t qkv_layer_stride, int layers,
                                  int rows, int row_stride, int k_col, int v_col, int Hkv,
                                  int dh, void* dst_k_layer0, void* dst_v_layer0,
                                  size_t dst_layer_stride_bytes, const int32_t* dst_slots,
                                  int block_size, int num_ctas, uintptr_t stream) {
  SWB_REQUIRE(dst_layer_stride_bytes % 16 == 0, "swb_kv_push_layers: layer stride alignment");
  return push_launch(qkv, rows, row_stride, k_col, v_col, Hkv, dh, dst_k_layer0, dst_v_layer0,
                     dst_slots, block_size, num_ctas, layers, qkv_layer_stride,
                     dst_layer_stride_bytes / sizeof(__nv_bfloat16), stream);
}

static PFN_cuStreamWriteValue32_v11070 write_value_fn() {
  static PFN_cuStreamWriteValue32_v11070 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
  }
  return fn;
}

extern "C" int swb_kv_handoff(const int32_t* first_tok, int n, const int32_t* rows,
                              const int32_t* seqs, const uint32_t* epochs, int group_key,
                              void* table, int stride_bytes, uintptr_t stream) {
  SWB_REQUIRE(first_tok && seqs && epochs && table, "swb_kv_handoff: null pointer");
  SWB_REQUIRE(n > 0 && n <= HANDOFF_MAX && stride_bytes >= 16 && stride_bytes % 4 == 0,
              "swb_kv_handoff: bad batch (n <= %d, stride >= 16)", HANDOFF_MAX);
  HandoffBatch b;
  for (int i = 0; i < n; ++i) {
    SWB_REQUIRE(seqs[i] >= 0, "swb_kv_handoff: negative slot");
    b.seq[i] = seqs[i];
    b.row[i] = rows ? rows[i] : i;
    SWB_REQUIRE(b.row[i] >= 0, "swb_kv_handoff: negative row");
  }
  const cudaError_t le = launch(handoff_token_kernel, dim3(1), dim3(HANDOFF_MAX), 0, STREAM,
                                first_tok, n, b, group_key, reinterpret_cast<char*>(table),
                                stride_bytes);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch handoff_token_kernel: %s", cudaGetErrorString(le));
  int rc = swb_check_launch("handoff_token_kernel");
  if (rc != SWB_OK) return rc;
  auto fn = write_value_fn();
  if (!fn) return swb_set_error(SWB_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  for (int i = 0; i < n; ++i) {
    // default flags: a full memory barrier precedes the store, so the pushed
    // KV pages and the first token are visible before the flag
    CUresult r = fn((CUstream)stream,
                    (CUdeviceptr)(reinterpret_cast<char*>(table) + (size_t)seqs[i] * stride_bytes),
                    epochs[i], CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS)
      return swb_set_error(SWB_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  }
  return SWB_OK;
}

extern "C" int swb_host_register(void* ptr, size_t bytes, void** dev_ptr) {
  SWB_REQUIRE(ptr && bytes && dev_ptr, "swb_host_register: null pointer");
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  e = cudaHostGetDevicePointer(dev_ptr, ptr, 0);
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  return SWB_OK;
}

extern "C" int swb_host_unregister(void* ptr) {
  SWB_REQUIRE(ptr, "swb_host_unregister: null pointer");
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
  return SWB_OK;
}

extern "C" int swb_decode_advance(const int32_t* next_tok, int32_t* cur_tok,
                                  int32_t* ctx, int32_t* step, int32_t* out_ring,
                                  int ring, int B, uintptr_t stream) {
  SWB_REQUIRE(next_tok && cur_tok && ctx && step && out_ring,
              "swb_decode_advance: null pointer");
  SWB_REQUIRE(B > 0 && ring > 0, "swb_decode_advance: bad shape");
  {
    const cudaError_t le_ = launch(decode_advance_kernel, dim3((B + 127) / 128), dim3(128), 0, STREAM,
        next_tok, cur_tok, ctx,
                                                             step, out_ring, ring, B);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch decode_advance_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("decode_advance_kernel");
}

extern "C" int swb_slots_from_table(const int32_t* table_row, int start, int n,
                                    int block_size, int32_t* slots, uintptr_t stream) {
  SWB_REQUIRE(table_row && slots, "swb_slots_from_table: null pointer");
  SWB_REQUIRE(start >= 0 && n >= 0 && block_size > 0, "swb_slots_from_table: bad args");
  if (n == 0) return SWB_OK;
  {
    const cudaError_t le_ = launch(slots_from_table_kernel, dim3((n + 255) / 256), dim3(256), 0, STREAM,
        table_row, start, n,
                                                               block_size, slots);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch slots_from_table_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("slots_from_table_kernel");
}

extern "C" int swb_argmax_shard(const float* logits, int rows, int V, int offset, int rank,
                                int tp, float* cand, uintptr_t stream) {
  SWB_REQUIRE(logits && cand, "swb_argmax_shard: null pointer");
  SWB_REQUIRE(rows >= 0 && V > 0 && offset >= 0 && tp >= 1 && tp <= 32 && rank >= 0 &&
                  rank < tp && offset + V < (1 << 24),
              "swb_argmax_shard: bad args (indices must stay exact in fp32)");
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(argmax_shard_kernel, dim3(rows), dim3(1024), 0, STREAM, logits,
                                V, offset, rank, tp, cand);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch argmax_shard_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("argmax_shard_kernel");
}

extern "C" int swb_argmax_pick(const float* cand, int rows, int tp, int32_t* out,
                               uintptr_t stream) {
  SWB_REQUIRE(cand && out, "swb_argmax_pick: null pointer");
  SWB_REQUIRE(rows >= 0 && tp >= 1 && tp <= 32, "swb_argmax_pick: bad args");
  if (rows == 0) return SWB_OK;
  const cudaError_t le = launch(argmax_pick_kernel, dim3((rows + 127) / 128), dim3(128), 0,
                                STREAM, cand, rows, tp, out);
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch argmax_pick_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("argmax_pick_kernel");
}
