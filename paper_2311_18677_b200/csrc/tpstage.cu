// Prefill partial exchange over the copy engines (TP > 1).
//
// The prefill's O / down projections leave each TP rank with a bf16 partial
// [rows, d]; the reference prices one all-reduce per projection (SURVEY
// §8(e)).  NCCL's all-reduce runs on the SMs and cannot overlap the
// persistent prefill GEMMs that hold every SM (70B TP4, 1500 tokens: 15.5 of
// 63.5 ms).  Here each rank instead hands its partial to every peer with a
// DMA copy (cudaMemcpyAsync into the peer's IPC-mapped receive buffer, on a
// side stream) followed by a stream-ordered flag write into the peer's flag
// word; the consumer stream waits for the peers' flags (cuStreamWaitValue32)
// and the next norm kernel adds own + received partials in rank order
// (swb_add_parts_rmsnorm / _layernorm).  The copy engines move the bytes
// while the tensor cores keep running (tools/ce_overlap_bench.py: a 16 MB
// copy hides completely behind a 1024 x 28672 x 8192 GEMM), so with the
// rows split into chunks the transfer of one chunk overlaps the next
// chunk's GEMMs.
//
// Region per rank: rx[n_bufs][world][bytes_per_src] followed by
// flags[n_bufs][SWB_TP_STAGE_MAXCH][world] (uint32 epochs).

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"

namespace {

constexpr int kStageMaxW = 8;
constexpr uint32_t kStageMagic = 0x53544731u;   // "STG1"

struct StageBlob {
  uint32_t magic;
  int rank, world, device, n_bufs;
  size_t bytes_per_src;
  cudaIpcMemHandle_t mem;
};
static_assert(sizeof(StageBlob) <= SWB_TP_STAGE_IPC_BYTES, "StageBlob outgrew the ABI blob");

PFN_cuStreamWriteValue32_v11070 stage_write_fn() {
  static PFN_cuStreamWriteValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    return cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
                       cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p)
               : nullptr;
  }();
  return fn;
}

PFN_cuStreamWaitValue32_v11070 stage_wait_fn() {
  static PFN_cuStreamWaitValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    return cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) ==
                       cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p)
               : nullptr;
  }();
  return fn;
}

}  // namespace

struct swb_tp_stage {
  int rank, world, device, n_bufs;
  size_t bytes_per_src;
  uint8_t* base;
  uint8_t* peer_base[kStageMaxW];
  bool connected;
};

static size_t stage_rx_off(const swb_tp_stage* s, int buf, int src) {
  return ((size_t)buf * s->world + src) * s->bytes_per_src;
}
static size_t stage_flag_off(const swb_tp_stage* s, int buf, int chunk, int src) {
  const size_t rx_end = (size_t)s->n_bufs * s->world * s->bytes_per_src;
  return rx_end + sizeof(uint32_t) * (((size_t)buf * SWB_TP_STAGE_MAXCH + chunk) * s->world + src);
}
static size_t stage_region_bytes(const swb_tp_stage* s) {
  return stage_flag_off(s, s->n_bufs, 0, 0);
}

extern "C" int swb_tp_stage_create(int rank, int world, size_t bytes_per_src, int n_bufs,
                                   swb_tp_stage** out, void* ipc_out, size_t ipc_bytes) {
  SWB_REQUIRE(out && ipc_out, "swb_tp_stage_create: null pointer");
  SWB_REQUIRE(world >= 2 && world <= kStageMaxW && rank >= 0 && rank < world,
              "swb_tp_stage_create: rank %d / world %d outside 2..%d", rank, world, kStageMaxW);
  SWB_REQUIRE(bytes_per_src > 0 && bytes_per_src % 256 == 0 && n_bufs >= 1 && n_bufs <= 8,
              "swb_tp_stage_create: bytes_per_src must be a positive multiple of 256, "
              "n_bufs 1..8");
  SWB_REQUIRE(ipc_bytes >= sizeof(StageBlob), "swb_tp_stage_create: need %zu ipc bytes",
              sizeof(StageBlob));
  SWB_REQUIRE(stage_write_fn() && stage_wait_fn(),
              "swb_tp_stage_create: stream memory operations unavailable");
  swb_tp_stage* s = new swb_tp_stage();
  s->rank = rank;
  s->world = world;
  s->n_bufs = n_bufs;
  s->bytes_per_src = bytes_per_src;
  s->base = nullptr;
  cudaError_t e = cudaGetDevice(&s->device);
  const size_t bytes = stage_region_bytes(s);
  if (e == cudaSuccess) e = cudaMalloc(&s->base, bytes);
  if (e == cudaSuccess) e = cudaMemset(s->base, 0, bytes);
  StageBlob b;
  memset(&b, 0, sizeof(b));
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&b.mem, s->base);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (s->base) cudaFree(s->base);
    delete s;
    return swb_set_error(SWB_ERR_CUDA, "swb_tp_stage_create: %s", cudaGetErrorString(e));
  }
  b.magic = kStageMagic;
  b.rank = rank;
  b.world = world;
  b.device = s->device;
  b.n_bufs = n_bufs;
  b.bytes_per_src = bytes_per_src;
  memcpy(ipc_out, &b, sizeof(b));
  for (int p = 0; p < kStageMaxW; ++p) s->peer_base[p] = nullptr;
  s->peer_base[rank] = s->base;
  s->connected = false;
  *out = s;
  return SWB_OK;
}

extern "C" int swb_tp_stage_connect(swb_tp_stage* s, const void* blobs, size_t blob_stride) {
  SWB_REQUIRE(s && blobs, "swb_tp_stage_connect: null pointer");
  SWB_REQUIRE(!s->connected, "swb_tp_stage_connect: already connected");
  SWB_REQUIRE(blob_stride >= sizeof(StageBlob), "swb_tp_stage_connect: short blob stride");
  for (int p = 0; p < s->world; ++p) {
    if (p == s->rank) continue;
    StageBlob b;
    memcpy(&b, static_cast<const uint8_t*>(blobs) + p * blob_stride, sizeof(b));
    SWB_REQUIRE(b.magic == kStageMagic, "swb_tp_stage_connect: bad blob for rank %d", p);
    SWB_REQUIRE(b.rank == p && b.world == s->world && b.n_bufs == s->n_bufs &&
                    b.bytes_per_src == s->bytes_per_src,
                "swb_tp_stage_connect: rank %d blob does not match this group", p);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.mem, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "swb_tp_stage_connect: open rank %d: %s", p,
                           cudaGetErrorString(e));
    s->peer_base[p] = static_cast<uint8_t*>(ptr);
  }
  s->connected = true;
  return SWB_OK;
}

extern "C" int swb_tp_stage_destroy(swb_tp_stage* s) {
  if (!s) return SWB_OK;
  for (int p = 0; p < s->world; ++p)
    if (p != s->rank && s->peer_base[p]) cudaIpcCloseMemHandle(s->peer_base[p]);
  cudaFree(s->base);
  delete s;
  return SWB_OK;
}

extern "C" void* swb_tp_stage_rx(const swb_tp_stage* s, int buf, int src) {
  if (!s || buf < 0 || buf >= s->n_bufs || src < 0 || src >= s->world) return nullptr;
  return s->base + stage_rx_off(s, buf, src);
}

extern "C" int swb_tp_stage_send(swb_tp_stage* s, int buf, int chunk, const void* src,
                                 size_t offset, size_t bytes, uint32_t epoch,
                                 uintptr_t stream) {
  SWB_REQUIRE(s && src, "swb_tp_stage_send: null pointer");
  SWB_REQUIRE(s->connected, "swb_tp_stage_send: not connected");
  SWB_REQUIRE(buf >= 0 && buf < s->n_bufs && chunk >= 0 && chunk < SWB_TP_STAGE_MAXCH,
              "swb_tp_stage_send: buffer %d / chunk %d out of range", buf, chunk);
  SWB_REQUIRE(offset + bytes <= s->bytes_per_src,
              "swb_tp_stage_send: %zu + %zu bytes exceed the %zu-byte receive buffer", offset,
              bytes, s->bytes_per_src);
  auto wr = stage_write_fn();
  for (int k = 1; k < s->world; ++k) {
    const int p = (s->rank + k) % s->world;      // staggered: not every rank on peer 0 first
    if (bytes) {
      const cudaError_t e = cudaMemcpyAsync(s->peer_base[p] + stage_rx_off(s, buf, s->rank) +
                                                offset,
                                            src, bytes, cudaMemcpyDeviceToDevice,
                                            (cudaStream_t)stream);
      if (e != cudaSuccess)
        return swb_set_error(SWB_ERR_CUDA, "swb_tp_stage_send: copy to rank %d: %s", p,
                             cudaGetErrorString(e));
    }
  }
  for (int k = 1; k < s->world; ++k) {
    const int p = (s->rank + k) % s->world;
    // default flags: the write follows the stream's prior work (the copies)
    // and is ordered after their data
    const CUresult r = wr((CUstream)stream,
                          (CUdeviceptr)(s->peer_base[p] + stage_flag_off(s, buf, chunk, s->rank)),
                          epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS)
      return swb_set_error(SWB_ERR_CUDA, "swb_tp_stage_send: flag write to rank %d (%d)", p,
                           (int)r);
  }
  return SWB_OK;
}

extern "C" int swb_tp_stage_wait(swb_tp_stage* s, int buf, int chunk, uint32_t epoch,
                                 uintptr_t stream) {
  SWB_REQUIRE(s, "swb_tp_stage_wait: null pointer");
  SWB_REQUIRE(buf >= 0 && buf < s->n_bufs && chunk >= 0 && chunk < SWB_TP_STAGE_MAXCH,
              "swb_tp_stage_wait: buffer %d / chunk %d out of range", buf, chunk);
  auto wt = stage_wait_fn();
  for (int p = 0; p < s->world; ++p) {
    if (p == s->rank) continue;
    const CUresult r = wt((CUstream)stream,
                          (CUdeviceptr)(s->base + stage_flag_off(s, buf, chunk, p)), epoch,
                          CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS)
      return swb_set_error(SWB_ERR_CUDA, "swb_tp_stage_wait: wait on rank %d (%d)", p, (int)r);
  }
  return SWB_OK;
}
