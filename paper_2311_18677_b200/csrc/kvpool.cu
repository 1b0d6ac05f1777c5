// Device-resident KV block pool and block-table manager (KV-cache manager).
//
// The reference keeps KV only as a byte count: Machine reserves each token
// task's *final* context at admission (machine.py:107-110, :216-223) and
// PerfModel prices it at kv_bytes_per_token (perf.py:134-141).  Here the pool
// is real HBM: per layer K and V arrays of [num_blocks][Hkv][bs][dh] bf16,
// int32 block tables [max_seqs][max_blocks_per_seq], and a free-block bitmap.
// Allocation is a single-CTA device kernel that hands out the n lowest free
// block ids (deterministic, so a CPU allocator model reproduces the table
// bit-for-bit) and writes the sequence's table row; freeing clears the bits.
// The host only mirrors the free-block count for admission decisions.
//
// The pool can be exported through CUDA IPC so that a prompt-pool process
// opens a non-owning view and pushes layer KV straight into these blocks.
#include <cstring>

#include "common.cuh"

struct swb_kv_pool {
  swb_kv_pool_info info;
  void* kv_alloc;      // K for all layers, then V for all layers
  int32_t* tables;
  uint32_t* bitmap;
  int device;
};

namespace swb {

constexpr uint32_t kIpcMagic = 0x53574231u;  // "SWB1"
struct IpcBlob {
  uint32_t magic;
  int32_t num_layers, num_blocks, Hkv, block_size, dh, max_seqs, max_blocks_per_seq;
  cudaIpcMemHandle_t kv;
  cudaIpcMemHandle_t tables;
};

// Lowest-free-first allocation of n blocks for one sequence (1 CTA, 1024 thr).
__global__ void __launch_bounds__(1024)
    block_alloc_kernel(uint32_t* __restrict__ bitmap, int num_blocks,
                       int32_t* __restrict__ table_row, int n) {
  pdl_trigger();
  pdl_wait();
  __shared__ int warp_tot[32];
  const int nwords = (num_blocks + 31) >> 5;
  const int per = (nwords + blockDim.x - 1) / blockDim.x;
  const int w0 = threadIdx.x * per;
  const int w1 = min(w0 + per, nwords);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) {
    uint32_t valid = 0xffffffffu;
    if (w == nwords - 1 && (num_blocks & 31)) valid = (1u << (num_blocks & 31)) - 1u;
    cnt += __popc(~bitmap[w] & valid);
  }
  // block-wide exclusive scan of cnt
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int v = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    warp_tot[lane] = s - v;  // exclusive warp offsets
  }
  __syncthreads();
  int rank = warp_tot[wid] + incl - cnt;
  for (int w = w0; w < w1 && rank < n; ++w) {
    uint32_t valid = 0xffffffffu;
    if (w == nwords - 1 && (num_blocks & 31)) valid = (1u << (num_blocks & 31)) - 1u;
    uint32_t freeb = ~bitmap[w] & valid;
    uint32_t take = 0;
    while (freeb && rank < n) {
      const int b = __ffs(freeb) - 1;
      freeb &= freeb - 1;
      take |= 1u << b;
      table_row[rank++] = w * 32 + b;
    }
    if (take) bitmap[w] |= take;
  }
}

__global__ void block_free_kernel(uint32_t* __restrict__ bitmap,
                                  int32_t* __restrict__ table_row, int n) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = table_row[i];
  if (b < 0) return;
  atomicAnd(&bitmap[b >> 5], ~(1u << (b & 31)));
  table_row[i] = -1;
}

}  // namespace swb

using namespace swb;

extern "C" int swb_kv_pool_create(int num_layers, int num_blocks, int Hkv,
                                  int block_size, int dh, int max_seqs,
                                  int max_blocks_per_seq, swb_kv_pool** out) {
  SWB_REQUIRE(out, "swb_kv_pool_create: null out");
  SWB_REQUIRE(num_layers > 0 && num_blocks > 0 && Hkv > 0 && block_size > 0 && dh > 0 &&
                  max_seqs > 0 && max_blocks_per_seq > 0,
              "swb_kv_pool_create: all sizes must be positive");
  SWB_REQUIRE(dh % 8 == 0, "swb_kv_pool_create: dh %% 8");
  *out = nullptr;
  const size_t block_bytes = (size_t)Hkv * block_size * dh * 2;
  const size_t layer_stride = block_bytes * num_blocks;
  const size_t kv_bytes = 2 * layer_stride * num_layers;
  swb_kv_pool* p = new swb_kv_pool();
  std::memset(p, 0, sizeof(*p));
  cudaGetDevice(&p->device);
  cudaError_t e = cudaMalloc(&p->kv_alloc, kv_bytes);
  if (e != cudaSuccess) {
    delete p;
    cudaGetLastError();
    return swb_set_error(SWB_ERR_CAPACITY, "KV pool of %zu bytes: %s", kv_bytes,
                         cudaGetErrorString(e));
  }
  const size_t tbytes = (size_t)max_seqs * max_blocks_per_seq * 4;
  const size_t nwords = ((size_t)num_blocks + 31) / 32;
  if (cudaMalloc(&p->tables, tbytes) != cudaSuccess ||
      cudaMalloc(&p->bitmap, nwords * 4) != cudaSuccess) {
    cudaFree(p->kv_alloc);
    if (p->tables) cudaFree(p->tables);
    delete p;
    cudaGetLastError();
    return swb_set_error(SWB_ERR_CAPACITY, "KV pool tables: out of memory");
  }
  cudaMemset(p->tables, 0xff, tbytes);
  cudaMemset(p->bitmap, 0, nwords * 4);
  swb_kv_pool_info& in = p->info;
  in.k_base = p->kv_alloc;
  in.v_base = static_cast<char*>(p->kv_alloc) + layer_stride * num_layers;
  in.layer_stride_bytes = layer_stride;
  in.block_bytes = block_bytes;
  in.block_tables = p->tables;
  in.bitmap = p->bitmap;
  in.num_layers = num_layers;
  in.num_blocks = num_blocks;
  in.Hkv = Hkv;
  in.block_size = block_size;
  in.dh = dh;
  in.max_seqs = max_seqs;
  in.max_blocks_per_seq = max_blocks_per_seq;
  in.free_blocks = num_blocks;
  in.is_peer_view = 0;
  SWB_CUDA(cudaDeviceSynchronize());
  *out = p;
  return SWB_OK;
}

extern "C" int swb_kv_pool_destroy(swb_kv_pool* p) {
  if (!p) return SWB_OK;
  if (p->info.is_peer_view) {
    cudaIpcCloseMemHandle(p->kv_alloc);
    cudaIpcCloseMemHandle(p->tables);
  } else {
    cudaFree(p->kv_alloc);
    cudaFree(p->tables);
    cudaFree(p->bitmap);
  }
  delete p;
  return SWB_OK;
}

extern "C" int swb_kv_pool_get_info(const swb_kv_pool* p, swb_kv_pool_info* out) {
  SWB_REQUIRE(p && out, "swb_kv_pool_get_info: null pointer");
  *out = p->info;
  return SWB_OK;
}

extern "C" int swb_block_alloc(swb_kv_pool* p, int seq, int n, uintptr_t stream) {
  SWB_REQUIRE(p, "swb_block_alloc: null pool");
  SWB_REQUIRE(!p->info.is_peer_view, "swb_block_alloc: peer views cannot allocate");
  SWB_REQUIRE(seq >= 0 && seq < p->info.max_seqs, "swb_block_alloc: seq %d out of range", seq);
  SWB_REQUIRE(n >= 0 && n <= p->info.max_blocks_per_seq,
              "swb_block_alloc: %d blocks exceeds max_blocks_per_seq %d", n,
              p->info.max_blocks_per_seq);
  if (n > p->info.free_blocks)
    return swb_set_error(SWB_ERR_CAPACITY, "swb_block_alloc: need %d blocks, %d free", n,
                         p->info.free_blocks);
  if (n == 0) return SWB_OK;
  p->info.free_blocks -= n;
  {
    const cudaError_t le_ = launch(block_alloc_kernel, dim3(1), dim3(1024), 0, (cudaStream_t)stream,
        
      p->bitmap, p->info.num_blocks, p->tables + (size_t)seq * p->info.max_blocks_per_seq, n);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch block_alloc_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("block_alloc_kernel");
}

extern "C" int swb_block_free(swb_kv_pool* p, int seq, int n, uintptr_t stream) {
  SWB_REQUIRE(p, "swb_block_free: null pool");
  SWB_REQUIRE(!p->info.is_peer_view, "swb_block_free: peer views cannot free");
  SWB_REQUIRE(seq >= 0 && seq < p->info.max_seqs, "swb_block_free: seq out of range");
  SWB_REQUIRE(n >= 0 && n <= p->info.max_blocks_per_seq, "swb_block_free: bad n");
  if (n == 0) return SWB_OK;
  p->info.free_blocks += n;
  {
    const cudaError_t le_ = launch(block_free_kernel, dim3((n + 255) / 256), dim3(256), 0, (cudaStream_t)stream,
        
      p->bitmap, p->tables + (size_t)seq * p->info.max_blocks_per_seq, n);
    if (le_ != cudaSuccess)
      return swb_set_error(SWB_ERR_CUDA, "launch block_free_kernel: %s", cudaGetErrorString(le_));
  }
  return swb_check_launch("block_free_kernel");
}

extern "C" int swb_kv_pool_ipc_export(const swb_kv_pool* p, void* handle_out,
                                      size_t handle_bytes) {
  SWB_REQUIRE(p && handle_out, "swb_kv_pool_ipc_export: null pointer");
  SWB_REQUIRE(handle_bytes >= sizeof(IpcBlob), "swb_kv_pool_ipc_export: need %zu bytes",
              sizeof(IpcBlob));
  SWB_REQUIRE(!p->info.is_peer_view, "swb_kv_pool_ipc_export: cannot re-export a view");
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kIpcMagic;
  b.num_layers = p->info.num_layers;
  b.num_blocks = p->info.num_blocks;
  b.Hkv = p->info.Hkv;
  b.block_size = p->info.block_size;
  b.dh = p->info.dh;
  b.max_seqs = p->info.max_seqs;
  b.max_blocks_per_seq = p->info.max_blocks_per_seq;
  SWB_CUDA(cudaIpcGetMemHandle(&b.kv, p->kv_alloc));
  SWB_CUDA(cudaIpcGetMemHandle(&b.tables, p->tables));
  std::memset(handle_out, 0, handle_bytes);
  std::memcpy(handle_out, &b, sizeof(b));
  return SWB_OK;
}

extern "C" int swb_kv_pool_ipc_open(const void* handle, size_t handle_bytes,
                                    swb_kv_pool** out) {
  SWB_REQUIRE(handle && out, "swb_kv_pool_ipc_open: null pointer");
  SWB_REQUIRE(handle_bytes >= sizeof(IpcBlob), "swb_kv_pool_ipc_open: short handle");
  IpcBlob b;
  std::memcpy(&b, handle, sizeof(b));
  SWB_REQUIRE(b.magic == kIpcMagic, "swb_kv_pool_ipc_open: bad magic");
  *out = nullptr;
  swb_kv_pool* p = new swb_kv_pool();
  std::memset(p, 0, sizeof(*p));
  cudaGetDevice(&p->device);
  cudaError_t e = cudaIpcOpenMemHandle(&p->kv_alloc, b.kv, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaSuccess) {
    void* t = nullptr;
    e = cudaIpcOpenMemHandle(&t, b.tables, cudaIpcMemLazyEnablePeerAccess);
    p->tables = static_cast<int32_t*>(t);
  }
  if (e != cudaSuccess) {
    if (p->kv_alloc) cudaIpcCloseMemHandle(p->kv_alloc);
    delete p;
    cudaGetLastError();
    return swb_set_error(SWB_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  }
  const size_t block_bytes = (size_t)b.Hkv * b.block_size * b.dh * 2;
  const size_t layer_stride = block_bytes * b.num_blocks;
  swb_kv_pool_info& in = p->info;
  in.k_base = p->kv_alloc;
  in.v_base = static_cast<char*>(p->kv_alloc) + layer_stride * b.num_layers;
  in.layer_stride_bytes = layer_stride;
  in.block_bytes = block_bytes;
  in.block_tables = p->tables;
  in.bitmap = nullptr;
  in.num_layers = b.num_layers;
  in.num_blocks = b.num_blocks;
  in.Hkv = b.Hkv;
  in.block_size = b.block_size;
  in.dh = b.dh;
  in.max_seqs = b.max_seqs;
  in.max_blocks_per_seq = b.max_blocks_per_seq;
  in.free_blocks = 0;
  in.is_peer_view = 1;
  *out = p;
  return SWB_OK;
}
