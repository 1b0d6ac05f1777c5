// Tensor-parallel all-reduce over NVLink peer memory (the TP pools of the
// 70B / BLOOM configs: "all-reduce twice per layer").
//
// Each rank owns one device region, exported by CUDA IPC and mapped by every
// peer of its TP group:
//   [slot 0 | slot 1 | aux slot 2 | rx[3][MAXW] | flags[3][MAXW][MAXC] | counters[3][MAXC]
//    | push counters[3][MAXW] | receive epochs[3][MAXC]]
// The producing GEMM/GEMV writes its fp32 partial sums straight into a slot
// (rank 0 folds the residual in), so the all-reduce moves no extra copy:
//   CTA c of rank r   1. system-scope fence, then a store of its epoch into
//                        flags[slot][r][c] of every peer,
//                     2. spins (acquire, nanosleep back-off, watchdog) until
//                        every peer's flag for (slot, c) reached the epoch,
//                     3. sums chunk c of the slot over ranks 0..W-1 in rank
//                        order (bit-identical results on every rank) with
//                        16-byte L2-only loads over NVLink, writes `out`.
// Decode-size messages (<= 1 MB) use the push form instead: CTA c first
// stores chunk c of its own slot into rx[slot][r] of every peer (posted
// NVLink writes), releases the flag behind them, and after the handshake sums
// own slot + rx[slot][p] from local memory — one one-way trip instead of a
// flag trip plus a remote-read round trip; same floats, same order.
// Epochs are per-(slot, CTA) device counters, so the launch is CUDA-graph
// replayable.  Slots 0 and 1 alternate: a slot is rewritten only after the
// next all-reduce (other slot) completed on every rank, i.e. after all peers
// finished reading it.  Slot 2 (small, <= 1 MB) is the once-per-step
// reduction (the vocab-parallel greedy candidates): the slot 0/1 all-reduces
// between two of its uses order them the same way, and it keeps the 0/1
// alternation unbroken across steps (a step does an even number of those).
// Fused form (swb_gemv_bf16_tp + swb_tp_allreduce_recv_f32): the projection
// GEMV's epilogue stores its partial into the peers' rx[slot][rank] itself
// and each of its nsrc CTAs adds 1 to the peers' push counter[slot][rank]
// after a system fence; the receive kernel's CTA c waits until every peer's
// counter reached epoch * nsrc (its own per-CTA epoch) and sums from local
// memory — the separate copy-and-flag pass of the push form disappears.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace swb {

constexpr int TP_MAXW = 8;
constexpr int TP_NSLOT = 3;
constexpr int TP_MAXC = 256;
constexpr int TP_THREADS = 512;
constexpr unsigned TP_RECV_CTAS = 4;   // fused form's receive grid (fixed: see mode 3)
constexpr uint32_t kTpMagic = 0x53575450u;  // "SWTP"

struct TpIpcBlob {
  uint32_t magic;
  int rank, world, device;
  uint64_t slot_bytes;
  cudaIpcMemHandle_t mem;
};
static_assert(sizeof(TpIpcBlob) <= SWB_TP_IPC_BYTES, "blob too large");

struct TpArgs {
  const unsigned long long* my_ll;   // fused form: this rank's receive lines[slot] (source 0)
  long long ll_stride;               // words per source
  const uint32_t* my_pcnt;           // fused form: this rank's push counters[slot][src]
  uint32_t* my_rctr;                 // fused form: per-CTA receive epochs[slot][c]
  uint32_t nsrc;                     // fused form: producer CTAs per peer
  const float* peer_slot[TP_MAXW];   // slot base of every rank (own = local)
  float* peer_rx[TP_MAXW];           // push mode: rank p's rx[slot][this rank]
  const float* my_rx;                // push mode: this rank's rx[slot][0]
  long long rx_stride;               // floats between rx[slot][src] and rx[slot][src+1]
  uint32_t* peer_flags[TP_MAXW];     // flags region of every rank
  uint32_t* my_flags;
  uint32_t* my_ctr;
  float* out;
  long long n;
  int rank, world, slot;
};

__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tp_handshake(const TpArgs& a, int c, uint32_t e) {
  // thread 0 of CTA c: publish epoch e to every peer, wait for theirs.  One
  // system-scope fence orders the CTA's data before all the flags; the flag
  // stores themselves are relaxed so they go out back to back (a release
  // store per peer would wait for the previous flag's NVLink round trip).
  __threadfence_system();
  for (int p = 0; p < a.world; ++p)
    if (p != a.rank)
      st_relaxed_sys(a.peer_flags[p] + ((size_t)a.slot * TP_MAXW + a.rank) * TP_MAXC + c, e);
  const long long t0 = clock64();
  for (int p = 0; p < a.world; ++p) {
    if (p == a.rank) continue;
    const uint32_t* f = a.my_flags + ((size_t)a.slot * TP_MAXW + p) * TP_MAXC + c;
    int spins = 0;
    while ((int)(ld_acquire_sys(f) - e) < 0) {
      if (++spins > 64) __nanosleep(64);
      // a peer that never arrives (crashed rank) must not wedge the GPU
      if (clock64() - t0 > 40000000000ll) __trap();
    }
  }
}

// Rank-ordered sum of float4 element i over all ranks' slots.
__device__ __forceinline__ float4 tp_sum4(const TpArgs& a, long long i) {
  float4 v[TP_MAXW];
#pragma unroll
  for (int p = 0; p < TP_MAXW; ++p)
    if (p < a.world) v[p] = __ldcg(reinterpret_cast<const float4*>(a.peer_slot[p]) + i);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int p = 0; p < TP_MAXW; ++p)
    if (p < a.world) {
      s.x += v[p].x; s.y += v[p].y; s.z += v[p].z; s.w += v[p].w;
    }
  return s;
}

// mode 0, one-shot pull: every rank reads all ranks' slots and sums the whole
// vector (one handshake; (W-1)*n floats in over NVLink).
// mode 1, two-shot: reduce-scatter then all-gather through the slots (two
// handshakes; 2*(W-1)/W*n in) — large messages on W > 2.
// mode 2, one-shot push: decode-size messages (fit the rx buffers).
__global__ void __launch_bounds__(TP_THREADS) tp_allreduce_kernel(const TpArgs a, int mode,
                                                                   int trig) {
  const int c = blockIdx.x;
  if (mode != 3) {
    pdl_wait();  // the producer GEMM/GEMV must be complete before we publish
    // past our own wait: the next kernel may launch now and stream its static
    // weights (pre-wait) while this one waits on the peers' flags over NVLink
    if (trig) pdl_launch_dependents();
  }
  if (mode == 3) {
    // fused form: the peers' projection GEMVs pushed (value, epoch) words
    // into rx[slot][p]; the own GEMV's CTAs counted into pcnt[slot][rank].
    // Always TP_RECV_CTAS CTAs, so rc[slot][0] (the GEMV's epoch) and every
    // rc[slot][c] advance together.
    const long long n4 = a.n >> 2;
    const long long per = (n4 + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)c * per, hi = min(n4, lo + per);
    uint32_t* rc = a.my_rctr + a.slot * TP_MAXC + c;
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(rc) + 1;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
      // the own projection's outputs: wait for its CTA count, not its exit
      const uint32_t* f = a.my_pcnt + (size_t)a.slot * TP_MAXW + a.rank;
      const uint32_t target = e * a.nsrc;
      int spins = 0;
      while ((int)(ld_acquire_sys(f) - target) < 0) {
        if (++spins > 64) __nanosleep(32);
        if (clock64() - t0 > 40000000000ll) __trap();
      }
    }
    __syncthreads();
    // dependents may launch: their pre-wait code only streams static weights
    if (trig) pdl_launch_dependents();
    const float4* mine = reinterpret_cast<const float4*>(a.peer_slot[a.rank]);
    const unsigned long long* lines = a.my_ll;
    const long long lstride = a.ll_stride;
    float4* out4 = reinterpret_cast<float4*>(a.out);
    for (long long i = lo + threadIdx.x; i < hi; i += TP_THREADS) {
      float4 v[TP_MAXW];
#pragma unroll
      for (int p = 0; p < TP_MAXW; ++p) {
        if (p >= a.world) continue;
        if (p == a.rank) {
          v[p] = __ldcg(mine + i);
          continue;
        }
        const unsigned long long* l = lines + p * lstride + 4 * i;
        unsigned long long w0, w1, w2, w3;
        for (;;) {
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(w0), "=l"(w1) : "l"(l) : "memory");
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(w2), "=l"(w3) : "l"(l + 2) : "memory");
          if ((uint32_t)(w0 >> 32) == e && (uint32_t)(w1 >> 32) == e &&
              (uint32_t)(w2 >> 32) == e && (uint32_t)(w3 >> 32) == e)
            break;
          if (clock64() - t0 > 40000000000ll) __trap();
        }
        v[p] = make_float4(__uint_as_float((uint32_t)w0), __uint_as_float((uint32_t)w1),
                           __uint_as_float((uint32_t)w2), __uint_as_float((uint32_t)w3));
      }
      // same source order on every rank: identical sums everywhere
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < TP_MAXW; ++p)
        if (p < a.world) {
          sum.x += v[p].x; sum.y += v[p].y; sum.z += v[p].z; sum.w += v[p].w;
        }
      out4[i] = sum;
    }
    if (threadIdx.x == 0) *rc = e;   // after the __syncthreads above: every thread read rc
    return;
  }
  uint32_t* ctr = a.my_ctr + a.slot * TP_MAXC + c;
  uint32_t e = 0;
  if (threadIdx.x == 0) {
    e = *ctr + 1;
    if (mode != 2) tp_handshake(a, c, e);
  }
  __syncthreads();
  const long long n4 = a.n >> 2;
  float4* out4 = reinterpret_cast<float4*>(a.out);
  if (mode == 2) {
    // push: copy this CTA's chunk of the local partial into every peer's
    // rx[slot][rank] (posted NVLink stores), release the flag behind them,
    // then sum the chunk from local memory only (own slot + rx of each peer)
    // in rank order — the same floats in the same order as the pull form.
    const long long per = (n4 + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)c * per, hi = min(n4, lo + per);
    const float4* mine = reinterpret_cast<const float4*>(a.peer_slot[a.rank]);
    for (long long i = lo + threadIdx.x; i < hi; i += TP_THREADS) {
      const float4 v = __ldcg(mine + i);
      for (int p = 0; p < a.world; ++p)
        if (p != a.rank) reinterpret_cast<float4*>(a.peer_rx[p])[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) tp_handshake(a, c, e);
    __syncthreads();
    for (long long i = lo + threadIdx.x; i < hi; i += TP_THREADS) {
      float4 v[TP_MAXW];
#pragma unroll
      for (int p = 0; p < TP_MAXW; ++p)
        if (p < a.world)
          v[p] = p == a.rank ? __ldcg(mine + i)
                             : __ldcg(reinterpret_cast<const float4*>(a.my_rx + p * a.rx_stride) + i);
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < TP_MAXW; ++p)
        if (p < a.world) {
          s.x += v[p].x; s.y += v[p].y; s.z += v[p].z; s.w += v[p].w;
        }
      out4[i] = s;
    }
    if (threadIdx.x == 0) *ctr = e;
    return;
  }
  if (mode == 0) {
    const long long per = (n4 + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)c * per, hi = min(n4, lo + per);
    for (long long i = lo + threadIdx.x; i < hi; i += 2 * TP_THREADS) {
      const long long j = i + TP_THREADS;
      const float4 s0 = tp_sum4(a, i);
      if (j < hi) out4[j] = tp_sum4(a, j);
      out4[i] = s0;
    }
    if (threadIdx.x == 0) *ctr = e;
    return;
  }
  // ---- reduce-scatter: this rank owns part `rank` of W parts
  const long long pl = (n4 + a.world - 1) / a.world;
  const long long per = (pl + gridDim.x - 1) / gridDim.x;
  const long long c_lo = (long long)c * per, c_hi = min(pl, c_lo + per);
  float4* mine = reinterpret_cast<float4*>(const_cast<float*>(a.peer_slot[a.rank]));
  {
    const long long base = (long long)a.rank * pl;
    for (long long i = c_lo + threadIdx.x; i < c_hi && base + i < n4; i += TP_THREADS) {
      const float4 s = tp_sum4(a, base + i);
      out4[base + i] = s;
      mine[base + i] = s;          // peers gather the reduced part from here
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    e += 1;
    tp_handshake(a, c, e);
    *ctr = e;
  }
  __syncthreads();
  // ---- all-gather: the other parts, reduced, from their owners
  for (int p = 0; p < a.world; ++p) {
    if (p == a.rank) continue;
    const float4* src = reinterpret_cast<const float4*>(a.peer_slot[p]);
    const long long base = (long long)p * pl;
    for (long long i = c_lo + threadIdx.x; i < c_hi && base + i < n4; i += TP_THREADS)
      out4[base + i] = __ldcg(src + base + i);
  }
}

}  // namespace swb

using namespace swb;

struct swb_tp_comm {
  int rank, world, device;
  int nsrc[TP_NSLOT];               // producer CTAs of the last fused GEMV per slot
  long long nout[TP_NSLOT];         // its output count (the receive must match it)
  size_t slot_bytes;
  uint8_t* base;                    // own region
  uint8_t* peer_base[TP_MAXW];      // mapped regions (own at [rank])
  bool connected;
};

// push-mode receive buffers: rx[3 slots][TP_MAXW sources] of tp_rx_bytes each
static size_t tp_rx_bytes(size_t slot_bytes) { return std::min<size_t>(slot_bytes, 1 << 20); }
static size_t tp_slot_cap(size_t slot_bytes, int slot) {
  return slot < 2 ? slot_bytes : tp_rx_bytes(slot_bytes);
}
static size_t tp_slot_off(size_t slot_bytes, int slot) { return (size_t)slot * slot_bytes; }
static size_t tp_rx_off(size_t slot_bytes) {
  return 2 * slot_bytes + tp_rx_bytes(slot_bytes);
}
static size_t tp_flags_off(size_t slot_bytes) {
  return tp_rx_off(slot_bytes) + TP_NSLOT * TP_MAXW * tp_rx_bytes(slot_bytes);
}
static size_t tp_pcnt_off(size_t slot_bytes) {
  return tp_flags_off(slot_bytes) +
         sizeof(uint32_t) * (TP_NSLOT * TP_MAXW * TP_MAXC + TP_NSLOT * TP_MAXC);
}
// fused-form receive lines: (value, epoch) words, ll[3 slots][TP_MAXW sources],
// apart from the float rx buffers so no float payload can pose as an epoch
constexpr size_t TP_LL_BYTES = 128 << 10;   // 16384 outputs per source
static size_t tp_ll_off(size_t slot_bytes) {
  const size_t end = tp_pcnt_off(slot_bytes) +
                     sizeof(uint32_t) * (TP_NSLOT * TP_MAXW + TP_NSLOT * TP_MAXC);
  return (end + 255) & ~(size_t)255;
}
static size_t tp_region_bytes(size_t slot_bytes) {
  return tp_ll_off(slot_bytes) + TP_NSLOT * TP_MAXW * TP_LL_BYTES;
}

extern "C" int swb_tp_comm_create(int rank, int world, size_t slot_bytes, swb_tp_comm** out,
                                  void* ipc_out, size_t ipc_bytes) {
  SWB_REQUIRE(out && ipc_out, "swb_tp_comm_create: null pointer");
  SWB_REQUIRE(world >= 1 && world <= TP_MAXW && rank >= 0 && rank < world,
              "swb_tp_comm_create: rank %d / world %d outside 1..%d", rank, world, TP_MAXW);
  SWB_REQUIRE(slot_bytes > 0 && slot_bytes % 256 == 0,
              "swb_tp_comm_create: slot_bytes must be a positive multiple of 256");
  SWB_REQUIRE(ipc_bytes >= sizeof(TpIpcBlob), "swb_tp_comm_create: need %zu ipc bytes",
              sizeof(TpIpcBlob));
  swb_tp_comm* c = new swb_tp_comm();
  c->rank = rank;
  c->world = world;
  c->slot_bytes = slot_bytes;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e == cudaSuccess) e = cudaMalloc(&c->base, tp_region_bytes(slot_bytes));
  if (e == cudaSuccess) e = cudaMemset(c->base, 0, tp_region_bytes(slot_bytes));
  TpIpcBlob b;
  memset(&b, 0, sizeof(b));
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&b.mem, c->base);
  if (e != cudaSuccess) {
    if (c->base) cudaFree(c->base);
    delete c;
    return swb_set_error(SWB_ERR_CUDA, "swb_tp_comm_create: %s", cudaGetErrorString(e));
  }
  b.magic = kTpMagic;
  b.rank = rank;
  b.world = world;
  b.device = c->device;
  b.slot_bytes = slot_bytes;
  memcpy(ipc_out, &b, sizeof(b));
  for (int p = 0; p < TP_MAXW; ++p) c->peer_base[p] = nullptr;
  c->peer_base[rank] = c->base;
  *out = c;
  return SWB_OK;
}

extern "C" int swb_tp_comm_connect(swb_tp_comm* c, const void* blobs, size_t blob_stride) {
  SWB_REQUIRE(c && blobs, "swb_tp_comm_connect: null pointer");
  SWB_REQUIRE(!c->connected, "swb_tp_comm_connect: already connected");
  SWB_REQUIRE(blob_stride >= sizeof(TpIpcBlob), "swb_tp_comm_connect: short blob stride");
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    TpIpcBlob b;
    memcpy(&b, static_cast<const uint8_t*>(blobs) + p * blob_stride, sizeof(b));
    SWB_REQUIRE(b.magic == kTpMagic, "swb_tp_comm_connect: bad blob for rank %d", p);
    SWB_REQUIRE(b.rank == p && b.world == c->world && b.slot_bytes == c->slot_bytes,
                "swb_tp_comm_connect: rank %d blob does not match this group", p);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.mem, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "swb_tp_comm_connect: open rank %d: %s", p,
                           cudaGetErrorString(e));
    c->peer_base[p] = static_cast<uint8_t*>(ptr);
  }
  c->connected = true;
  return SWB_OK;
}

extern "C" int swb_tp_comm_destroy(swb_tp_comm* c) {
  if (!c) return SWB_OK;
  for (int p = 0; p < c->world; ++p)
    if (p != c->rank && c->peer_base[p]) cudaIpcCloseMemHandle(c->peer_base[p]);
  cudaFree(c->base);
  delete c;
  return SWB_OK;
}

extern "C" void* swb_tp_comm_slot(const swb_tp_comm* c, int slot) {
  if (!c || slot < 0 || slot >= TP_NSLOT) return nullptr;
  return c->base + tp_slot_off(c->slot_bytes, slot);
}

namespace swb {
int tp_push_targets(swb_tp_comm* c, int slot, int nsrc, long long n, TpPush* out) {
  SWB_REQUIRE(c && out, "tp_push_targets: null pointer");
  SWB_REQUIRE(n >= 0 && (size_t)n * 8 <= TP_LL_BYTES,
              "tp_push_targets: %lld outputs exceed the receive lines", n);
  SWB_REQUIRE(c->connected || c->world == 1, "tp_push_targets: not connected");
  SWB_REQUIRE(slot >= 0 && slot < TP_NSLOT, "tp_push_targets: bad slot");
  SWB_REQUIRE(c->world <= 8, "tp_push_targets: world > 8");
  const size_t ll_off = tp_ll_off(c->slot_bytes) + (size_t)slot * TP_MAXW * TP_LL_BYTES;
  const size_t pc_off = tp_pcnt_off(c->slot_bytes);
  memset(out, 0, sizeof(*out));
  out->world = c->world;
  out->rank = c->rank;
  out->own_cnt = reinterpret_cast<unsigned*>(c->base + pc_off) + (size_t)slot * TP_MAXW + c->rank;
  out->epoch = reinterpret_cast<const unsigned*>(c->base + pc_off) + TP_NSLOT * TP_MAXW +
               (size_t)slot * TP_MAXC;
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    out->rx[p] = reinterpret_cast<unsigned long long*>(c->peer_base[p] + ll_off +
                                                       (size_t)c->rank * TP_LL_BYTES);
  }
  c->nsrc[slot] = nsrc;
  c->nout[slot] = n;
  return SWB_OK;
}
}  // namespace swb

// SWB_TP_AR_TRIGGER=0: exit-time PDL trigger instead of right after the wait
static int tp_trigger() {
  static const int on = [] {
    const char* e = std::getenv("SWB_TP_AR_TRIGGER");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on;
}

static int tp_allreduce(swb_tp_comm* c, int slot, float* out, size_t n, uintptr_t stream,
                        bool recv);

extern "C" int swb_tp_allreduce_f32(swb_tp_comm* c, int slot, float* out, size_t n,
                                    uintptr_t stream) {
  return tp_allreduce(c, slot, out, n, stream, false);
}

extern "C" int swb_tp_allreduce_recv_f32(swb_tp_comm* c, int slot, float* out, size_t n,
                                         uintptr_t stream) {
  SWB_REQUIRE(c && c->world > 1, "swb_tp_allreduce_recv_f32: needs a TP group");
  SWB_REQUIRE(slot >= 0 && slot < TP_NSLOT && c->nsrc[slot] > 0,
              "swb_tp_allreduce_recv_f32: no fused projection on slot %d", slot);
  SWB_REQUIRE(n * 8 <= TP_LL_BYTES,
              "swb_tp_allreduce_recv_f32: n=%zu exceeds the receive lines", n);
  SWB_REQUIRE((long long)n == c->nout[slot],
              "swb_tp_allreduce_recv_f32: n=%zu but the fused projection on slot %d produced %lld",
              n, slot, c->nout[slot]);
  return tp_allreduce(c, slot, out, n, stream, true);
}

static int tp_allreduce(swb_tp_comm* c, int slot, float* out, size_t n, uintptr_t stream,
                        bool recv) {
  SWB_REQUIRE(c && out, "swb_tp_allreduce_f32: null pointer");
  SWB_REQUIRE(c->connected || c->world == 1, "swb_tp_allreduce_f32: not connected");
  SWB_REQUIRE(slot >= 0 && slot < TP_NSLOT, "swb_tp_allreduce_f32: slot must be 0, 1 or 2");
  SWB_REQUIRE(n % 4 == 0 && n * sizeof(float) <= tp_slot_cap(c->slot_bytes, slot),
              "swb_tp_allreduce_f32: n=%zu must be a multiple of 4 and fit slot %d", n, slot);
  SWB_REQUIRE((((uintptr_t)out) & 15) == 0, "swb_tp_allreduce_f32: out must be 16-byte aligned");
  if (n == 0) return SWB_OK;
  TpArgs a;
  memset(&a, 0, sizeof(a));
  const size_t flags_off = tp_flags_off(c->slot_bytes);
  const size_t rxb = tp_rx_bytes(c->slot_bytes);
  const size_t rx_off = tp_rx_off(c->slot_bytes) + (size_t)slot * TP_MAXW * rxb;
  for (int p = 0; p < c->world; ++p) {
    a.peer_slot[p] = reinterpret_cast<const float*>(c->peer_base[p] +
                                                    tp_slot_off(c->slot_bytes, slot));
    a.peer_rx[p] = reinterpret_cast<float*>(c->peer_base[p] + rx_off + (size_t)c->rank * rxb);
    a.peer_flags[p] = reinterpret_cast<uint32_t*>(c->peer_base[p] + flags_off);
  }
  a.my_rx = reinterpret_cast<const float*>(c->base + rx_off);
  a.rx_stride = (long long)(rxb / sizeof(float));
  a.my_flags = reinterpret_cast<uint32_t*>(c->base + flags_off);
  a.my_ctr = a.my_flags + TP_NSLOT * TP_MAXW * TP_MAXC;
  a.my_pcnt = reinterpret_cast<const uint32_t*>(c->base + tp_pcnt_off(c->slot_bytes));
  a.my_rctr = reinterpret_cast<uint32_t*>(c->base + tp_pcnt_off(c->slot_bytes)) +
              TP_NSLOT * TP_MAXW;
  a.my_ll = reinterpret_cast<const unsigned long long*>(
      c->base + tp_ll_off(c->slot_bytes) + (size_t)slot * TP_MAXW * TP_LL_BYTES);
  a.ll_stride = (long long)(TP_LL_BYTES / 8);
  a.nsrc = recv ? (uint32_t)c->nsrc[slot] : 0u;
  a.out = out;
  a.n = (long long)n;
  a.rank = c->rank;
  a.world = c->world;
  a.slot = slot;
  // ~16 KB of output per CTA, at most TP_MAXC CTAs (one wave)
  const long long ctas = std::min<long long>(TP_MAXC, std::max<long long>(1, (long long)n / 4096));
  // two-shot once the (W-1)x one-shot traffic outweighs a second handshake
  int mode = c->world > 2 && n >= (size_t)(1 << 18) ? 1 : 0;
  // small messages: push (posted NVLink stores + flag, local reads) instead
  // of pull (flag, then a remote-read round trip); SWB_TP_AR_PUSH=0 for A/B
  static const bool push_on = [] {
    const char* e = std::getenv("SWB_TP_AR_PUSH");
    return !(e && e[0] == '0');
  }();
  if (mode == 0 && push_on && c->world > 1 && n * sizeof(float) <= rxb) mode = 2;
  if (recv) mode = 3;
  const cudaError_t le = launch(tp_allreduce_kernel, dim3(recv ? TP_RECV_CTAS : (unsigned)ctas), dim3(TP_THREADS), 0,
                                (cudaStream_t)stream, a, mode, tp_trigger());
  if (le != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "launch tp_allreduce_kernel: %s", cudaGetErrorString(le));
  return swb_check_launch("tp_allreduce_kernel");
}
