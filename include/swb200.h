/*
 * swb200.h — C-ABI of libswb200.so, the B200-native hot path of Splitwise
 * (arXiv 2311.18677): prompt-phase prefill, layer-wise KV push into a token
 * machine's paged KV blocks, and token-phase decode.
 *
 * The reference (`splitsim`, /root/reference/pkg) models this path with
 * latency lookups; every entry point below replaces one of those lookups (or
 * the byte accounting behind it) with real GPU work.  The reference-side
 * interface each one replaces is cited as file:line relative to
 * /root/reference/pkg/src/splitsim/.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types.  Device pointers are
 *    passed as `void*`/typed pointers; CUDA streams as `uintptr_t`
 *    (a cudaStream_t value, 0 = legacy default stream).
 *  - Every function returns an int status.  The Python host maps them onto
 *    the reference exception hierarchy (errors.py:4-31):
 *        SWB_ERR_INVALID  -> ValidationError     (errors.py:8)
 *        SWB_ERR_CAPACITY -> CapacityError       (errors.py:26)
 *        SWB_ERR_CONFIG   -> ConfigurationError  (errors.py:30)
 *        SWB_ERR_CUDA     -> RuntimeError (text from swb_last_error()).
 *  - All compute calls are asynchronous and stream ordered; none blocks the
 *    host except swb_sync_stream.  The library never allocates or frees
 *    caller memory, except the KV pools it creates (swb_kv_pool_create /
 *    swb_kv_pool_destroy).
 *  - Element types: activations/weights bf16, residual stream fp32,
 *    accumulation fp32, token ids / slots / block ids int32.
 */
#ifndef SWB200_H_
#define SWB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWB_OK 0
#define SWB_ERR_INVALID 1
#define SWB_ERR_CAPACITY 2
#define SWB_ERR_CUDA 3
#define SWB_ERR_CONFIG 4

#define SWB_ABI_VERSION 1

/* ---------------------------------------------------------------- meta */
int swb_abi_version(void);
/* Text of the last error raised on the calling host thread ("" if none). */
const char* swb_last_error(void);
/* Blocks the host until `stream` drains (the only blocking call). */
int swb_sync_stream(uintptr_t stream);

/* ------------------------------------------------------- dense GEMM (prefill)
 * out[M,N] = epilogue(A[M,K] . W[N,K]^T), bf16 operands, fp32 accumulate in
 * TMEM (tcgen05.mma, TMA-fed 128B-swizzled smem ring).  Replaces the prompt
 * cost lookup PerfModel.prompt_time (perf.py:119-123) for the linear layers.
 *   epilogue SWB_EPI_BF16     : out bf16 [M,N]
 *   epilogue SWB_EPI_F32      : out fp32 [M,N]
 *   epilogue SWB_EPI_RESID_F32: out fp32 [M,N] = resid fp32 [M,N] + acc
 *                               (out may alias resid)
 *   epilogue SWB_EPI_SWIGLU   : W rows are gate/up interleaved in 128-row
 *                               groups; out bf16 [M,N/2] = silu(gate)*up
 * Requirements: K % 8 == 0 (TMA row pitch), N % 16 == 0, pointers 16B aligned.
 */
#define SWB_EPI_BF16 0
#define SWB_EPI_F32 1
#define SWB_EPI_RESID_F32 2
#define SWB_EPI_SWIGLU 3
/*   epilogue SWB_EPI_GELU     : out bf16 [M,N] = gelu_tanh(acc + bias)
 *                               (BLOOM's MLP up projection) */
#define SWB_EPI_GELU 4
int swb_gemm_bf16(const void* a, const void* w, void* out, const void* resid,
                  int M, int N, int K, int epilogue, uintptr_t stream);
/* With a per-output-feature bf16 bias [N] (may be NULL) added to the fp32
 * accumulator before the epilogue (BLOOM's biased linears); not with
 * SWB_EPI_SWIGLU. */
int swb_gemm_bf16_bias(const void* a, const void* w, void* out,
                       const void* resid, const void* bias, int M, int N,
                       int K, int epilogue, uintptr_t stream);

/* QKV projection of a prefill with the RoPE / KV-write step fused into the
 * GEMM epilogue: qkv bf16 [M, (H+2Hkv)*128] = a . w^T (+ bias), then the q
 * and k heads of row r are rotated at positions[r] (theta <= 1: no rotation,
 * ALiBi models; rope_table may be NULL) and, when slots is given, row r's k/v heads are written to
 * pool slot slots[r] — bit-identical to swb_gemm_bf16_bias(EPI_BF16) followed
 * by swb_rope_kv_write.  Replaces the same prompt-phase lookup
 * (PerfModel.prompt_time, perf.py:119-123). */
int swb_gemm_qkv_rope(const void* a, const void* w, void* qkv, const void* bias,
                      int M, int N, int K, const int32_t* positions, float theta,
                      const void* rope_table, int table_len, int H, int Hkv,
                      void* k_layer, void* v_layer, const int32_t* slots,
                      int block_size, uintptr_t stream);
/* (sin, cos) fp32 pairs [max_pos][64] of the RoPE angles pos * theta^(-2i/128),
 * computed with the same device math the kernels use on the fly (so a table
 * lookup is bit-identical); rope_table of swb_gemm_qkv_rope (positions >=
 * table_len fall back to computing). */
int swb_rope_table(float theta, int max_pos, void* table, uintptr_t stream);

/* --------------------------------------------- skinny GEMM / GEMV (decode)
 * Same contract as swb_gemm_bf16 for small M (decode batch, 1..16 rows):
 * weight-streaming kernel, 128-bit coalesced weight loads, fp32 accumulate.
 * Replaces the decode cost lookup PerfModel.token_iter_time (perf.py:125-132)
 * for the linear layers.
 */
int swb_gemv_bf16(const void* x, const void* w, void* out, const void* resid,
                  int M, int N, int K, int epilogue, uintptr_t stream);
int swb_gemv_bf16_bias(const void* x, const void* w, void* out,
                       const void* resid, const void* bias, int M, int N,
                       int K, int epilogue, uintptr_t stream);
/* Pre-norm fused variant: x is the fp32 residual stream [M,K]; the kernel
 * applies RMSNorm with weight norm_w on the fly (bit-identical to
 * swb_rmsnorm followed by swb_gemv_bf16).  out may not alias x. */
int swb_gemv_rmsnorm_bf16(const float* x, const void* norm_w, float eps,
                          const void* w, void* out, const void* resid, int M,
                          int N, int K, int epilogue, uintptr_t stream);

/* ------------------------------------------------------- elementwise ops */
/* x fp32 [rows,d] <- table bf16 [V,d][tokens[r]] */
int swb_embed(const int32_t* tokens, const void* table, float* x, int rows,
              int d, uintptr_t stream);
/* out bf16 [rows,d] = rmsnorm(x fp32 [src_rows,d]) * w; row_index (may be
 * NULL) selects src rows (e.g. the last token of each prompt). */
int swb_rmsnorm(const float* x, const int32_t* row_index, const void* w,
                void* out, int rows, int d, float eps, uintptr_t stream);
/* LayerNorm with bias (BLOOM): out = (x - mean) * rstd * w + b, bf16 out, or
 * fp32 out when out_f32 (may then be x itself: the embedding LayerNorm). */
int swb_layernorm(const float* x, const int32_t* row_index, const void* w,
                  const void* b, void* out, int rows, int d, float eps,
                  int out_f32, uintptr_t stream);
/* Greedy sampling: out[r] = argmax_v logits fp32 [rows,V] (lowest index on
 * ties). */
/* TP prefill: x[src] += addend[src] (bf16, the all-reduced sum of the ranks'
 * bf16 projection partials) over the normalised rows, written back to the
 * fp32 residual stream, then the norm as swb_rmsnorm / swb_layernorm. */
int swb_add_rmsnorm(float* x, const void* addend, const int32_t* row_index, const void* w,
                    void* out, int rows, int d, float eps, uintptr_t stream);
int swb_add_layernorm(float* x, const void* addend, const int32_t* row_index, const void* w,
                      const void* b, void* out, int rows, int d, float eps, uintptr_t stream);
/* Same with the TP ranks' bf16 partials still apart (copy-engine exchange,
 * swb_tp_stage_*): x[src] += (parts[0][src] + ... + parts[n-1][src]) summed
 * in fp32 in the given (rank) order, 1 <= n_parts <= 8. */
int swb_add_parts_rmsnorm(float* x, const void* const* parts, int n_parts,
                          const int32_t* row_index, const void* w, void* out, int rows, int d,
                          float eps, uintptr_t stream);
int swb_add_parts_layernorm(float* x, const void* const* parts, int n_parts,
                            const int32_t* row_index, const void* w, const void* b, void* out,
                            int rows, int d, float eps, uintptr_t stream);
int swb_argmax(const float* logits, int rows, int V, int32_t* out,
               uintptr_t stream);

/* -------------------------------------------- RoPE + KV write into blocks
 * qkv bf16 [rows, row_stride] holds q (H heads), k (Hkv), v (Hkv) at column
 * offsets 0, H*dh, (H+Hkv)*dh.  Rotates q and k in place (NeoX half split,
 * theta) at positions[r], and, when k_layer/v_layer are non-NULL, writes the
 * rotated k and v of row r into paged slot slots[r] of the layer's block
 * pool (layout [block][Hkv][block_size][dh]).  The KV bytes it writes are
 * what PerfModel.kv_cache_bytes (perf.py:134-137) counts.  theta == 0: no
 * rotation (ALiBi models), KV write only.
 */
int swb_rope_kv_write(void* qkv, int rows, int row_stride, const int32_t* positions,
                      int H, int Hkv, int dh, float theta, void* k_layer,
                      void* v_layer, const int32_t* slots, int block_size,
                      uintptr_t stream);

/* ------------------------------------------------ KV pack-and-push (a5)
 * Copies rows' k/v (already rotated, in qkv layout as above) into the paged
 * blocks of a destination pool that may live on a peer GPU (P2P stores over
 * NVLink through an IPC-mapped pointer).  `num_ctas` bounds the SMs the push
 * borrows from concurrent prefill compute (0 = auto).  Replaces
 * transfer.plan_transfer / raw_transfer_time (transfer.py:66-99): the bytes
 * are moved instead of priced.
 */
int swb_kv_push_layer(const void* qkv, int rows, int row_stride, int k_col,
                      int v_col, int Hkv, int dh, void* dst_k_layer,
                      void* dst_v_layer, const int32_t* dst_slots,
                      int block_size, int num_ctas, uintptr_t stream);
/* Serialized transfer mode (reference select_mode / plan_transfer,
 * transfer.py:73-99: prompts below the mode threshold move their KV after
 * the prompt phase instead of layer by layer): one launch pushes `layers`
 * layers; layer l reads qkv + l * qkv_layer_stride elements and writes the
 * destination layer arrays at dst_k/v_layer0 + l * dst_layer_stride_bytes. */
int swb_kv_push_layers(const void* qkv, size_t qkv_layer_stride, int layers,
                       int rows, int row_stride, int k_col, int v_col, int Hkv,
                       int dh, void* dst_k_layer0, void* dst_v_layer0,
                       size_t dst_layer_stride_bytes, const int32_t* dst_slots,
                       int block_size, int num_ctas, uintptr_t stream);
/* Hand-off of a finished prompt batch — the paper's per-request semaphore
 * and the reference's TRANSFER event (engine.py:286-297):
 * after all prior work on `stream` (the KV pushes), request i's record at
 * table + seqs[i] * stride_bytes (int32 [flag, first_token, group_key, n])
 * gets first_tok[rows[i]] (device; rows NULL = i), group_key and n, and then
 * epochs[i] in word 0.  The flag stores are stream memory operations
 * preceded by a full memory barrier, so a consumer that observes
 * flag == epoch also observes the record and every pushed KV page; it admits
 * the n records of one group together.  `table` is device-accessible:
 * host-mapped shared memory (swb_host_register) polled by the token
 * machine's host, or peer memory.  n <= 64; rows/seqs/epochs are host
 * arrays; stride_bytes >= 16. */
int swb_kv_handoff(const int32_t* first_tok, int n, const int32_t* rows,
                   const int32_t* seqs, const uint32_t* epochs, int group_key,
                   void* table, int stride_bytes, uintptr_t stream);
/* Page-lock and map host memory (e.g. a /dev/shm mapping shared with the
 * token machine's process) for device stores; *dev_ptr receives its device
 * address. */
int swb_host_register(void* ptr, size_t bytes, void** dev_ptr);
int swb_host_unregister(void* ptr);

/* ---------------------------------------------------- attention kernels */
/* Causal varlen prefill attention with GQA over qkv rows; sequences are
 * delimited by cu_seqlens[num_seqs+1]; out bf16 [rows, H*dh]. dh == 128. */
int swb_attn_prefill(const void* qkv, int row_stride, const int32_t* cu_seqlens,
                     int num_seqs, int max_seqlen, int H, int Hkv, int dh,
                     float scale, void* out, uintptr_t stream);
/* Same contract on the 5th-gen tensor cores (tcgen05.mma, TMEM S/O
 * accumulators, TMA-fed K/V rings); total_rows = cu_seqlens[num_seqs] bounds
 * the TMA view of qkv.  alibi_slopes (fp32 [H], may be NULL) adds
 * slope_h * (key_pos - query_pos) to the scores (BLOOM).  The default prefill
 * attention of the runner. */
int swb_attn_prefill_tc(const void* qkv, int row_stride, int total_rows,
                        const int32_t* cu_seqlens, int num_seqs, int max_seqlen,
                        int H, int Hkv, int dh, float scale,
                        const float* alibi_slopes, void* out, uintptr_t stream);
/* Paged decode attention for one layer, fused with the current token's
 * RoPE and KV append and with the split-K merge: q/k/v of the current token
 * come from qkv rows [B, row_stride] (q at column 0); when positions/slots are
 * given, q and k are rotated at positions[b] and the token's k/v are written
 * to pool slot slots[b] (both NULL: K/V already in the pool, no rotation).
 * Keys/values are read through block_tables [B, max_blocks] for ctx_lens[b]
 * tokens (including the current one).  The context is split into partitions
 * of `partition` tokens; the last CTA of each (b, kv head) merges them.
 * workspace must hold swb_attn_decode_workspace(B, H, max_ctx, partition, dh)
 * bytes and be ZERO-initialised once (its merge tickets self-reset).
 * alibi_slopes (fp32 [H], may be NULL): ALiBi instead of RoPE (BLOOM) —
 * no rotation, scores + slope_h * (key_pos - query_pos).
 * Replaces the attention share of PerfModel.token_iter_time (perf.py:125-132)
 * and the KV growth of Machine.complete_iteration (machine.py:263-266). */
size_t swb_attn_decode_workspace(int B, int H, int max_ctx, int partition,
                                 int dh);
int swb_attn_decode(const void* qkv, int row_stride, void* k_layer,
                    void* v_layer, const int32_t* block_tables, int max_blocks,
                    const int32_t* ctx_lens, const int32_t* positions,
                    const int32_t* slots, float theta,
                    const float* alibi_slopes, int B, int H, int Hkv, int dh,
                    int block_size, float scale, int max_ctx, int partition,
                    void* workspace, void* out, uintptr_t stream);

/* Decode-graph form of swb_attn_decode: ctx[b] = tokens already cached for
 * sequence b; the current token (q/k/v in qkv row b) is at position ctx[b],
 * rotated there (RoPE; or ALiBi when alibi_slopes is given), appended at the
 * slot block_tables[b][ctx/bs]*bs + ctx%bs, and attends over ctx[b]+1 tokens.
 * ctx, block_tables and the cached pages are read before the kernel's
 * programmatic-dependency wait, so they must be produced by work that
 * completed before the PRECEDING kernel on the stream started (in the decode
 * graph: the previous replay / the host); only qkv may come from the
 * preceding kernel.  Same workspace contract as swb_attn_decode.
 * Replaces the same reference lookups as swb_attn_decode. */
int swb_attn_decode_step(const void* qkv, int row_stride, void* k_layer,
                         void* v_layer, const int32_t* block_tables,
                         int max_blocks, const int32_t* ctx, float theta,
                         const float* alibi_slopes, int B, int H, int Hkv,
                         int dh, int block_size, float scale, int max_ctx,
                         int partition, void* workspace, void* out,
                         uintptr_t stream);

/* Chunked prefill attention: rows [0, C) of qkv are the queries of prompt
 * positions q_start .. q_start+C-1 (already RoPE'd; their K/V already in the
 * pool, e.g. by swb_gemm_qkv_rope with slots), keys are read through
 * table_row for positions <= each query's own (causal).  out bf16 [C, H*128].
 * workspace: swb_attn_chunk_workspace(C, H, max_ctx) bytes, zeroed once.
 * Lets a long prompt be prefilled in chunks (mixed with decode rows per
 * iteration) instead of one batch — the chunked-prefill option of
 * SURVEY §8(f); reference prompt batching machine.py:186-203. */
size_t swb_attn_chunk_workspace(int C, int H, int max_ctx);
int swb_attn_chunk(const void* qkv, int row_stride, int C, int q_start,
                   const void* k_layer, const void* v_layer,
                   const int32_t* table_row, int H, int Hkv, int dh,
                   int block_size, float scale, const float* alibi_slopes,
                   int max_ctx, void* workspace, void* out, uintptr_t stream);

/* Vocab-parallel greedy pick for TP pools (the LM head split by vocabulary
 * rows): swb_argmax_shard writes each row's (max logit, global index =
 * local argmax + offset) into slot `rank` of cand fp32 [rows][tp][2] and
 * zeros into the other slots; after the pool's sum all-reduce of cand,
 * swb_argmax_pick returns the index of the largest candidate (lowest index
 * on ties) — equal to swb_argmax over the full vocabulary. */
int swb_argmax_shard(const float* logits, int rows, int V, int offset, int rank,
                     int tp, float* cand, uintptr_t stream);
int swb_argmax_pick(const float* cand, int rows, int tp, int32_t* out,
                    uintptr_t stream);

/* --------------------------------------------- decode-step bookkeeping
 * Graph-resident per-step state update so the decode loop needs no host
 * round trip (Machine.complete_iteration, machine.py:247-275):
 *  advance: cur_tok[b] = next_tok[b]; out_ring[b*ring + step[b]] = next_tok[b];
 *           step[b] += 1; ctx[b] += 1
 */
int swb_decode_advance(const int32_t* next_tok, int32_t* cur_tok, int32_t* ctx,
                       int32_t* step, int32_t* out_ring, int ring, int B,
                       uintptr_t stream);
/* slots[i] = table_row[(start+i)/bs]*bs + (start+i)%bs for i < n (table_row
 * may be peer memory: the prompt side reads the token side's table). */
int swb_slots_from_table(const int32_t* table_row, int start, int n,
                         int block_size, int32_t* slots, uintptr_t stream);

/* ----------------------------------------------- KV block pool (a3/a4)
 * Device-resident pool: per layer K and V arrays [num_blocks][Hkv][bs][dh]
 * bf16, block tables int32 [max_seqs][max_blocks_per_seq], and a free-block
 * bitmap.  Allocation is lowest-free-first, done by a device kernel that
 * writes the sequence's block-table row; the host keeps only the free count
 * (admission = Machine._memory_fits, machine.py:125-128).  Replaces the
 * byte-count memory model (perf.py:134-141, machine.py:107-128).
 */
typedef struct swb_kv_pool swb_kv_pool;
typedef struct {
  void* k_base;               /* layer l K = k_base + l*layer_stride bytes */
  void* v_base;
  size_t layer_stride_bytes;
  size_t block_bytes;         /* one block of one layer, K or V */
  int32_t* block_tables;      /* [max_seqs][max_blocks_per_seq] */
  uint32_t* bitmap;           /* 1 bit per block, 1 = in use */
  int num_layers, num_blocks, Hkv, block_size, dh, max_seqs,
      max_blocks_per_seq;
  int free_blocks;            /* host mirror */
  int is_peer_view;           /* opened through IPC, not owned */
} swb_kv_pool_info;

int swb_kv_pool_create(int num_layers, int num_blocks, int Hkv, int block_size,
                       int dh, int max_seqs, int max_blocks_per_seq,
                       swb_kv_pool** out);
int swb_kv_pool_destroy(swb_kv_pool* pool);
int swb_kv_pool_get_info(const swb_kv_pool* pool, swb_kv_pool_info* out);
/* Reserve n blocks for sequence slot `seq` (lowest free first), writing its
 * block-table row; SWB_ERR_CAPACITY if fewer than n blocks are free. */
int swb_block_alloc(swb_kv_pool* pool, int seq, int n_blocks, uintptr_t stream);
/* Release the first n blocks of seq's row back to the pool. */
int swb_block_free(swb_kv_pool* pool, int seq, int n_blocks, uintptr_t stream);
/* IPC: SWB_KV_POOL_IPC_BYTES-byte handle of the pool (KV arrays + block
 * tables) for a peer process; the peer opens a non-owning view it can push
 * into and whose block tables it can read. */
#define SWB_KV_POOL_IPC_BYTES 256
int swb_kv_pool_ipc_export(const swb_kv_pool* pool, void* handle_out,
                           size_t handle_bytes);
int swb_kv_pool_ipc_open(const void* handle, size_t handle_bytes,
                         swb_kv_pool** out);
/* Enable direct peer access between the current device and `peer`. */
int swb_enable_peer(int peer_device);

/* ------------------------------------------- tensor-parallel all-reduce
 * The TP pools' "all-reduce twice per layer" (the reference
 * prices it inside PerfModel.prompt_time / token_iter_time, perf.py:119-132)
 * over NVLink peer memory instead of a library collective.  Each rank
 * creates a communicator owning two fp32 slots of slot_bytes (IPC-exported,
 * blob of SWB_TP_IPC_BYTES), exchanges blobs with its group (any host
 * channel), connects, then per reduction: the producing GEMM/GEMV writes
 * its partial sums into swb_tp_comm_slot(comm, s) and
 * swb_tp_allreduce_f32(comm, s, out, n) writes the rank-ordered sum of all
 * ranks' slot s into out (identical bits on every rank).  Alternate the
 * slot between consecutive reductions.  Epochs live on the device, so the
 * call is CUDA-graph capturable.  Messages up to min(slot_bytes, 1 MB) are
 * pushed into per-peer receive buffers (decode sizes); larger ones are
 * pulled (one-shot, or reduce-scatter + all-gather for W > 2); the sum
 * order, and so the result bits, are the same in every form. */
#define SWB_TP_IPC_BYTES 128
typedef struct swb_tp_comm swb_tp_comm;
int swb_tp_comm_create(int rank, int world, size_t slot_bytes, swb_tp_comm** out,
                       void* ipc_out, size_t ipc_bytes);
/* blobs: world entries of blob_stride bytes, indexed by rank (own ignored). */
int swb_tp_comm_connect(swb_tp_comm* comm, const void* blobs, size_t blob_stride);
int swb_tp_comm_destroy(swb_tp_comm* comm);
void* swb_tp_comm_slot(const swb_tp_comm* comm, int slot);
int swb_tp_allreduce_f32(swb_tp_comm* comm, int slot, float* out, size_t n,
                         uintptr_t stream);
/* Fused projection + all-reduce push (decode, one row): the weight-streaming
 * GEMV (epilogue SWB_EPI_F32, or SWB_EPI_RESID_F32 with resid on the rank
 * that folds the residual) writes its fp32 partial into this rank's slot
 * `slot` AND stores it straight into every peer's receive lines for this
 * rank over NVLink from the epilogue, each output as one 8-byte (value,
 * epoch) word, so the data carries its own flag (no release fence); each CTA
 * then counts itself on this rank's own counter (gpu-scope release).
 * swb_tp_allreduce_recv_f32 waits for the own count and every peer word of
 * the current epoch and writes the rank-ordered sum (same bits as
 * swb_tp_allreduce_f32), without waiting for the GEMV grid to exit.  Use the
 * two as a pair on the same slot, alternating slots like
 * swb_tp_allreduce_f32.  N <= 16384 (128 KB of lines per source). */
int swb_gemv_bf16_tp(const void* x, const void* w, const void* resid, const void* bias,
                     int M, int N, int K, int epilogue, swb_tp_comm* comm, int slot,
                     uintptr_t stream);
int swb_tp_allreduce_recv_f32(swb_tp_comm* comm, int slot, float* out, size_t n,
                              uintptr_t stream);

/* Prefill partial exchange over the copy engines (TP > 1; replaces the
 * prefill all-reduces priced in PerfModel.prompt_time, perf.py:119-123 /
 * 297-326).  Each rank owns rx[n_bufs][world] receive buffers of
 * bytes_per_src bytes and flags[n_bufs][SWB_TP_STAGE_MAXCH][world] in
 * IPC-shared device memory (create -> all-gather the blobs -> connect).
 * swb_tp_stage_send enqueues on `stream`: a DMA copy of src[0, bytes) into
 * every peer's rx[buf][this rank] + offset, then a write of `epoch` into
 * every peer's flag[buf][chunk][this rank].  swb_tp_stage_wait makes
 * `stream` wait until flag[buf][chunk][p] >= epoch for every peer p; the
 * received partials are then at swb_tp_stage_rx(buf, p) + offset.  The
 * caller keeps epochs increasing and a buffer's next send behind its last
 * consumer (tp prefill: one send per projection per chunk, epoch = layer
 * counter). */
#define SWB_TP_STAGE_MAXCH 8
#define SWB_TP_STAGE_IPC_BYTES 128
typedef struct swb_tp_stage swb_tp_stage;
int swb_tp_stage_create(int rank, int world, size_t bytes_per_src, int n_bufs,
                        swb_tp_stage** out, void* ipc_blob, size_t ipc_bytes);
int swb_tp_stage_connect(swb_tp_stage* stage, const void* blobs, size_t blob_stride);
int swb_tp_stage_destroy(swb_tp_stage* stage);
void* swb_tp_stage_rx(const swb_tp_stage* stage, int buf, int src);
int swb_tp_stage_send(swb_tp_stage* stage, int buf, int chunk, const void* src, size_t offset,
                      size_t bytes, uint32_t epoch, uintptr_t stream);
int swb_tp_stage_wait(swb_tp_stage* stage, int buf, int chunk, uint32_t epoch,
                      uintptr_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SWB200_H_ */
