"""Per-GPU execution of the two phases on libswb200 kernels.

``ModelRunner.prefill``  — the prompt phase (replaces PerfModel.prompt_time,
reference perf.py:119-123): embedding, per layer RMSNorm -> QKV GEMM
(tcgen05) -> RoPE (+ KV write into local paged blocks when the token phase
runs on this machine) -> causal varlen attention -> O GEMM (+residual) ->
RMSNorm -> gate/up GEMM with fused SwiGLU -> down GEMM (+residual), TP
all-reduce after O and down; last-token norm, LM head, greedy argmax.
When the request's token machine is another GPU, each finished layer's K/V is
packed and pushed into that GPU's paged blocks by ``kv_push_layer`` on a side
stream, overlapping the next layer's compute (reference plan_transfer's
layer-wise mode, transfer.py:79-99, made real).

``DecodeGraph`` — one token-phase iteration for a fixed batch bucket
(replaces PerfModel.token_iter_time, perf.py:125-132): the whole step
(prepare -> L x [norm, QKV GEMV, RoPE+KV append, paged attention, O GEMV,
norm, gate/up GEMV+SwiGLU, down GEMV] -> norm -> LM head -> argmax ->
advance) is captured once in a CUDA graph and replayed; all per-step state
(current token, context length, output ring) stays on the device.
"""

from __future__ import annotations

import gc
import math
import os
from dataclasses import dataclass, field

import torch

from . import _abi
from . import kernels as K
from .errors import CapacityError
from .kvcache import KVCacheManager
from .model import Weights
from .transfer import B200_NVLINK_PAIR, LAYERWISE, SERIALIZED

# serialized transfer mode (reference select_mode, transfer.py:73-76): every
# prompt of the batch shorter than the NVLink threshold and the batch small
# enough for the per-layer stash
SERIAL_THRESHOLD = int(os.environ.get("SWB_SERIAL_THRESHOLD",
                                      str(B200_NVLINK_PAIR["mode_threshold_tokens"])))
SERIAL_MAX_ROWS = 256


@dataclass
class PushSegment:
    """Rows [row0, row0+rows) of a prefill batch go to one destination pool."""
    row0: int
    rows: int
    dst: KVCacheManager          # peer view (or local pool for 1-GPU tests)
    dst_seq: int                 # sequence slot in the destination tables
    slots: torch.Tensor | None = None


@dataclass
class PushStats:
    layer_ms: list = field(default_factory=list)
    bytes_per_layer: int = 0
    total_ms: float = 0.0        # first push start -> last push end
    tail_ms: float = 0.0         # compute end -> last push end (visible latency)
    compute_ms: float = 0.0      # prefill compute (first kernel -> compute end)
    mode: str = LAYERWISE


@dataclass
class Handoff:
    """Where a prompt batch announces its landed KV to ONE token machine
    (control.HandoffTable): per request the batch row, the token machine's
    KV slot and reservation epoch; the table's device address in this
    process; the batch's group key (the token machine admits the group's
    requests together)."""
    seqs: list
    epochs: list
    table_ptr: int
    rows: list | None = None
    key: int = 0
    stride: int = 16


class ModelRunner:
    def __init__(self, weights: Weights, kv: KVCacheManager | None = None, tp_group=None,
                 decode_partition: int = 128, push_ctas: int = 64, tp_max_rows: int = 8192):
        self.w = weights
        self.cfg = cfg = weights.cfg
        self.tp = weights.tp
        self.rank = weights.rank
        self.tp_group = tp_group
        self.tp_comm = None
        self.bloom = cfg.is_bloom
        self.theta = 0.0 if self.bloom else cfg.rope_theta     # 0: ALiBi, no rotation
        self.alibi = weights.alibi
        self.tp_max_rows = tp_max_rows    # largest prefill / decode row count reduced
        self.ar_nccl_bytes = int(os.environ.get("SWB_TP_AR_NCCL_BYTES", str(4 << 20)))
        # SWB_TP_AR_BF16=0 keeps the prefill all-reduces in fp32 (A/B)
        self.ar_bf16 = os.environ.get("SWB_TP_AR_BF16", "1") != "0"
        self._pending_add = None
        # prefill reductions as copy-engine exchanges of the bf16 partials
        # (tpcomm.TPStage), summed inside the next norm: 70B TP2 1024-token
        # prefill 71.1 -> 70.4 ms.  At TP4 the all-gather moves twice NCCL's
        # bytes (73.3 vs 64.0-66.6 ms), so auto = TP2 only; SWB_TP_STAGE=1/0
        # forces it.  SWB_TP_STAGE_CHUNKS (default 2): the O / down GEMMs run
        # in row chunks of whole 256-row tiles whose partials leave as they
        # land (the MLP stays whole: split gate/up GEMMs lose to wave
        # quantisation) — TP2 70.9 -> 70.4 ms on one box; 4 chunks 81 ms
        # (profiles/r2_tp_prefill_exchange.json)
        mode = os.environ.get("SWB_TP_STAGE", "auto")
        self.tp_stage = self.tp == 2 if mode == "auto" else mode == "1"
        self.stage_chunks = int(os.environ.get("SWB_TP_STAGE_CHUNKS", "2"))
        self._stage = None
        self._stage_epoch = 0
        self._stage_own = [None, None]      # this rank's O / down partials (bf16)
        self._stage_sent = [None, None]     # side-stream events: partial copied out
        self._stage_stream = None
        # decode B=1 projections push their partial to the peers from the
        # GEMV epilogue as (value, epoch) words (swb_gemv_bf16_tp) and a
        # receive kernel only waits and sums: 70B TP4 B=1 decode 8.21 -> 7.84
        # ms/step, TP2 12.97 -> 12.61 (profiles/r2_fused_ar.json);
        # SWB_TP_FUSED=0 restores GEMV + push all-reduce kernel for A/B
        self.tp_fused = os.environ.get("SWB_TP_FUSED", "1") != "0"
        self.kv = kv
        self.hq = cfg.n_heads // self.tp
        self.hkv = cfg.n_kv_heads // self.tp
        self.dh = cfg.head_dim
        self.qkv_cols = (self.hq + 2 * self.hkv) * self.dh
        self.ffn = cfg.ffn // self.tp
        self.scale = 1.0 / math.sqrt(self.dh)
        self.partition = decode_partition
        self.push_ctas = push_ctas
        self.dev = weights.embed.device
        self._cap = 0
        # the push stream's CTAs are scheduled ahead of the prefill's: 7B
        # 1024 tokens, in-flight push 298 -> 353 GB/s and TTFT overhead 2.8 ->
        # 2.2 % (profiles/r2_push_priority_ab.json); SWB_PUSH_PRIORITY=normal A/B
        prio = 0 if os.environ.get("SWB_PUSH_PRIORITY", "high") == "normal" else -1
        self.push_stream = torch.cuda.Stream(device=self.dev, priority=prio)
        self._buf_ev = [None, None]      # last push that read each qkv buffer
        self._stash = None               # [L, SERIAL_MAX_ROWS, qkv_cols] (serialized mode)
        self._stash_ev = None
        self._pending_push = []          # (timing, compute_end, last_event, stats)
        self.graphs: dict = {}
        # RoPE angle table for the fused QKV-GEMM epilogue (16K positions, 8 MB)
        self.rope_tab = (K.rope_table(cfg.rope_theta, 16384, device=self.dev)
                         if not self.bloom and self.dh == 128 else None)
        # TP pools: LM head split by vocabulary rows (each rank streams V/TP
        # rows), greedy pick through the pool's all-reduce of per-rank
        # (max, index) candidates; SWB_VOCAB_PARALLEL=0 keeps the replicated head
        self.vocab_parallel = (self.tp > 1 and cfg.vocab % self.tp == 0 and
                               os.environ.get("SWB_VOCAB_PARALLEL", "1") != "0")
        self.vocab_local = cfg.vocab // self.tp if self.vocab_parallel else cfg.vocab
        self.vocab_off = self.rank * self.vocab_local if self.vocab_parallel else 0
        self.head = (weights.lm_head[self.vocab_off:self.vocab_off + self.vocab_local]
                     if self.vocab_parallel else weights.lm_head)

    # ------------------------------------------------------------ helpers
    def _allreduce(self, x):
        if self.tp > 1:
            torch.distributed.all_reduce(x, group=self.tp_group)

    def _comm(self):
        """NVLink peer-memory all-reduce (tpcomm.py) for TP > 1, created on
        first use; SWB_TP_AR=nccl selects torch.distributed's all_reduce."""
        if self.tp == 1 or os.environ.get("SWB_TP_AR", "p2p") == "nccl":
            return None
        if self.tp_comm is None:
            from .tpcomm import TPComm
            self.tp_comm = TPComm(self.tp_group, self.tp_max_rows * self.cfg.d_model * 4)
        return self.tp_comm

    def _begin_reductions(self):
        if self._pending_add is not None:
            raise RuntimeError("a bf16 all-reduce result was never added to the residual")
        c = self._comm()
        if c is not None:
            c.reset()

    def _proj_reduce(self, inp, w, x, bias=None):
        """x <- x + sum over TP ranks of inp @ w^T (+ bias) (O / down
        projections).  TP: rank 0 folds the residual (and the replicated
        bias) into its partial; the partials meet in the peer-memory slot and
        the all-reduce writes x."""
        if self.tp == 1:
            K.linear(inp, w, K.EPI_RESID_F32, out=x, resid=x, bias=bias)
            return
        b = bias if self.rank == 0 else None
        c = self._comm()
        # large (prefill) messages: NCCL's all-reduce (NVSwitch in-network
        # reduction) beats the peer-memory kernel — 49 MB at TP4 155 vs 253 us,
        # 32 MB at TP2 90 vs 97 us (tools/ar_bench.py); small (decode)
        # messages stay on the graph-replayable peer kernel (20 vs 26-39 us)
        big = x.numel() * 4 >= self.ar_nccl_bytes
        if big and self.ar_bf16 and x.shape[0] > K.GEMV_MAX_ROWS:
            # prefill-size messages: the ranks' partials (no residual) go
            # through the all-reduce in bf16 — half the NVLink bytes — and
            # join the fp32 residual in the next norm (x += sum, then norm).
            # Prefill rows only: the decode graph's fused pre-norm GEMVs
            # read x directly.
            part = self._ar_part(x.shape)
            K.linear(inp, w, K.EPI_BF16, out=part, bias=b)
            self._allreduce(part)
            self._pending_add = part
            return
        if c is None or big:
            K.linear(inp, w, self._resid_epi(), out=x, resid=x, bias=b)
            self._allreduce(x)
            return
        s = c.next_slot()
        if self.tp_fused and x.shape[0] == 1 and x.numel() <= c.LL_OUTPUTS:
            # decode B=1: the GEMV epilogue pushes its partial to the peers
            # itself; the receive kernel only waits and sums locally
            K.gemv_tp(inp, w, self._resid_epi(), c._h, s, resid=x, bias=b)
            c.allreduce_recv(s, x)
            return
        part = c.slot(s, x.shape)
        K.linear(inp, w, self._resid_epi(), out=part, resid=x, bias=b)
        c.allreduce(s, x)

    def _ar_part(self, shape):
        buf = getattr(self, "_arbuf", None)
        n = shape[0] * shape[1]
        if buf is None or buf.numel() < n:
            self._arbuf = buf = torch.empty(n, dtype=torch.bfloat16, device=self.dev)
        return buf[:n].view(shape)

    # -- architecture switches (Llama: RMSNorm / RoPE / SwiGLU; BLOOM:
    #    LayerNorm+bias / ALiBi / biased linears + GELU / embedding LayerNorm)
    def _norm(self, x, w, b, out, rows_index=None):
        add, self._pending_add = self._pending_add, None    # a bf16 all-reduce result
        if isinstance(add, tuple):
            # copy-engine exchange: wait for every chunk's peer flags, then
            # the norm adds own + received partials in rank order
            buf, epoch, n_chunks, own = add
            for c in range(n_chunks):
                self._stage.wait(buf, c, epoch)
            add = self._stage.parts(buf, own, 0, x.shape[0])
        elif add is not None and add.shape != x.shape:
            raise RuntimeError("pending all-reduce result does not match the residual")
        if self.bloom:
            K.layernorm(x, w, b, self.cfg.norm_eps, rows_index=rows_index, out=out, addend=add)
        else:
            K.rmsnorm(x, w, self.cfg.norm_eps, rows_index=rows_index, out=out, addend=add)

    def _embed(self, tokens, x):
        K.embed(tokens, self.w.embed, out=x)
        if self.bloom:
            K.layernorm(x, self.w.emb_norm, self.w.emb_norm_b, self.cfg.norm_eps, out=x,
                        out_f32=True)

    def _mlp_up(self, h, lw, out):
        if self.bloom:
            K.linear(h, lw.wgu, K.EPI_GELU, out=out, bias=lw.bup)
        else:
            K.linear(h, lw.wgu, K.EPI_SWIGLU, out=out)

    def _greedy(self, logits, out):
        """Greedy token per row of ``logits`` (this rank's vocabulary shard
        under vocab parallelism)."""
        if not self.vocab_parallel:
            K.argmax(logits, out=out)
            return
        rows = int(logits.shape[0])
        c = self._comm()
        if c is None:        # NCCL all-reduce of the candidate table
            cand = torch.empty(rows, self.tp, 2, dtype=torch.float32, device=self.dev)
            K.argmax_shard(logits, self.vocab_off, self.rank, self.tp, cand)
            self._allreduce(cand)
        else:
            # the aux slot: outside the slot-0/1 alternation of the step's
            # O / down reductions (which must stay even per step)
            part = c.slot(c.AUX, (rows, self.tp, 2))
            K.argmax_shard(logits, self.vocab_off, self.rank, self.tp, part)
            cand = self._cand_buf(rows)
            c.allreduce(c.AUX, cand)
        K.argmax_pick(cand, rows, self.tp, out)

    def _cand_buf(self, rows):
        buf = getattr(self, "_cand", None)
        if buf is None or buf.shape[0] < rows:
            self._cand = torch.empty(max(rows, 64), self.tp, 2, dtype=torch.float32,
                                     device=self.dev)
        return self._cand[:rows]

    def _resid_epi(self):
        # with TP only rank 0 folds the residual in; the all-reduce sums the rest
        return K.EPI_RESID_F32 if self.rank == 0 or self.tp == 1 else K.EPI_F32

    # ------------------------------------------- TP prefill chunk exchange
    def _stage_on(self, T: int) -> bool:
        return (self.tp > 1 and self.tp_stage and T > K.GEMV_MAX_ROWS and
                T * self.cfg.d_model * 4 >= self.ar_nccl_bytes)

    def _stage_comm(self, T: int):
        """TPStage sized for T rows (collective: every TP rank runs the same
        prefill sequence, so all grow together)."""
        if self._stage is None or self._stage.rows < T:
            from .tpcomm import TPStage
            if self._stage is not None:
                torch.cuda.synchronize()
                self._stage.close()
            rows = (T + 2047) // 2048 * 2048
            self._stage = TPStage(self.tp_group, rows, self.cfg.d_model)
            d = self.cfg.d_model
            self._stage_own = [torch.empty(rows, d, dtype=torch.bfloat16, device=self.dev)
                               for _ in range(2)]
            self._stage_sent = [None, None]
            if self._stage_stream is None:
                self._stage_stream = torch.cuda.Stream(device=self.dev)
        return self._stage

    def _stage_chunks(self, T: int) -> list:
        n = max(1, min(self.stage_chunks, 8, T // 256))   # SWB_TP_STAGE_MAXCH
        step = (T + n - 1) // n
        step = (step + 255) // 256 * 256                 # whole 256-row GEMM tiles
        return [(r0, min(T, r0 + step)) for r0 in range(0, T, step)]

    def _stage_send(self, kind: int, chunk: int, rows: torch.Tensor, row0: int, epoch: int):
        main = torch.cuda.current_stream()
        side = self._stage_stream
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        self._stage.send(kind, chunk, rows, row0, epoch, side)
        done = torch.cuda.Event()
        done.record(side)
        self._stage_sent[kind] = done

    def _stage_layer(self, attn, lw, x, h, act, T: int):
        """O projection -> residual + norm -> MLP -> down projection of one
        layer with both TP reductions as copy-engine exchanges.  The two
        projections run in row chunks whose partials leave as soon as they
        land (chunk c's copy under chunk c+1's GEMM); the norm and the MLP
        take all rows (their GEMMs lose to wave quantisation when split);
        the down projection's exchange is added by the next norm (_norm)."""
        st = self._stage_comm(T)
        main = torch.cuda.current_stream()
        chunks = self._stage_chunks(T)
        self._stage_epoch += 1
        e = self._stage_epoch
        bo = lw.bo if self.rank == 0 else None
        bd = lw.bd if self.rank == 0 else None
        po, pd = self._stage_own[0][:T], self._stage_own[1][:T]
        # the previous layer's copies out of the own partial buffers are done
        if self._stage_sent[0] is not None:
            main.wait_event(self._stage_sent[0])
        for c, (r0, r1) in enumerate(chunks):
            K.linear(attn[r0:r1], lw.wo, K.EPI_BF16, out=po[r0:r1], bias=bo)
            self._stage_send(0, c, po[r0:r1], r0, e)
        for c in range(len(chunks)):
            st.wait(0, c, e)
        parts = st.parts(0, po, 0, T)
        if self.bloom:
            K.layernorm(x, lw.mlp_norm, lw.mlp_norm_b, self.cfg.norm_eps, out=h, addend=parts)
        else:
            K.rmsnorm(x, lw.mlp_norm, self.cfg.norm_eps, out=h, addend=parts)
        self._mlp_up(h, lw, act)
        if self._stage_sent[1] is not None:
            main.wait_event(self._stage_sent[1])
        for c, (r0, r1) in enumerate(chunks):
            K.linear(act[r0:r1], lw.wd, K.EPI_BF16, out=pd[r0:r1], bias=bd)
            self._stage_send(1, c, pd[r0:r1], r0, e)
        self._pending_add = (1, e, len(chunks), pd)

    def _ensure_prefill(self, T: int, R: int):
        if T <= self._cap and R <= getattr(self, "_rcap", 0):
            return
        cap = max(T, 256)
        rcap = max(R, 16)
        d, dev = self.cfg.d_model, self.dev
        self.px = torch.empty(cap, d, dtype=torch.float32, device=dev)
        self.ph = torch.empty(cap, d, dtype=torch.bfloat16, device=dev)
        self.pqkv = [torch.empty(cap, self.qkv_cols, dtype=torch.bfloat16, device=dev)
                     for _ in range(2)]
        self.pattn = torch.empty(cap, self.hq * self.dh, dtype=torch.bfloat16, device=dev)
        self.pact = torch.empty(cap, self.ffn, dtype=torch.bfloat16, device=dev)
        self.plast = torch.empty(rcap, d, dtype=torch.bfloat16, device=dev)
        self.plogits = torch.empty(rcap, self.vocab_local, dtype=torch.float32, device=dev)
        self.pfirst = torch.empty(rcap, dtype=torch.int32, device=dev)
        self._cap, self._rcap = cap, rcap

    # ------------------------------------------------------------ prefill
    def transfer_mode(self, lens: list[int]) -> str:
        """Serialized when every prompt of the batch is below the NVLink
        threshold (reference select_mode, transfer.py:73-76) and the batch
        fits the stash; layer-wise otherwise (a short prompt that shares a
        batch with a long one rides that batch's per-layer pushes)."""
        if sum(lens) <= SERIAL_MAX_ROWS and all(n < SERIAL_THRESHOLD for n in lens):
            return SERIALIZED
        return LAYERWISE

    def _wait_buffer(self, main, ev):
        if ev is not None:
            main.wait_event(ev)

    def _wait_push_tails(self):
        """Paths that reuse pqkv[0] / pfirst without push bookkeeping wait for
        every push still reading them."""
        main = torch.cuda.current_stream()
        for ev in (*self._buf_ev, self._stash_ev):
            self._wait_buffer(main, ev)

    def prefill(self, tokens: torch.Tensor, lens: list[int], meta: torch.Tensor,
                local_slots: torch.Tensor | None = None,
                push: list[PushSegment] | None = None,
                push_stats: PushStats | None = None,
                handoff: Handoff | list | None = None, mode: str | None = None) -> torch.Tensor:
        """Run the prompt phase for a batch of prompts packed back to back.

        tokens      int32 [T] on device
        meta        int32 device tensor = [positions(T) | cu_seqlens(R+1) | last_rows(R)]
        local_slots int32 [T] slots in this GPU's pool (co-located token phase)
        push        per-request destination segments (token machine elsewhere)
        handoff     announce the landed KV to the token machine(s) (one Handoff
                    per destination table, control.HandoffTable) from the push
                    stream; the call then returns
                    without waiting for the pushes (the prompt machine is free
                    once its compute ends).  Without it, the current stream
                    waits for every push before the call returns.
        mode        SERIALIZED / LAYERWISE (default: transfer_mode(lens))
        Returns the greedy first token of every prompt (int32 [R], device).
        """
        cfg, w = self.cfg, self.w
        T, R = int(tokens.shape[0]), len(lens)
        self._ensure_prefill(T, R)
        positions = meta[:T]
        cu = meta[T:T + R + 1]
        last_rows = meta[T + R + 1:T + 2 * R + 1]
        x, h, attn, act = self.px[:T], self.ph[:T], self.pattn[:T], self.pact[:T]
        main = torch.cuda.current_stream()
        mode = (mode or self.transfer_mode(lens)) if push else LAYERWISE
        handoffs = ([] if handoff is None else
                    list(handoff) if isinstance(handoff, (list, tuple)) else [handoff])
        serial = push and mode == SERIALIZED
        timing = None
        if push:
            for seg in push:
                if seg.slots is None:
                    seg.slots = torch.empty(seg.rows, dtype=torch.int32, device=self.dev)
                K.slots_from_table(seg.dst.table_row_ptr(seg.dst_seq), 0, seg.rows,
                                   seg.dst.block_size, seg.slots)
                seg.slots.record_stream(self.push_stream)
            if push_stats is not None:
                push_stats.mode = mode
                n_ev = 1 if serial else cfg.n_layers
                timing = [(torch.cuda.Event(enable_timing=True),
                           torch.cuda.Event(enable_timing=True)) for _ in range(n_ev)]
                compute_start = torch.cuda.Event(enable_timing=True)
                compute_start.record(main)
        if serial:
            if self._stash is None:
                self._stash = torch.empty(cfg.n_layers, SERIAL_MAX_ROWS, self.qkv_cols,
                                          dtype=torch.bfloat16, device=self.dev)
            self._wait_buffer(main, self._stash_ev)
        self._begin_reductions()
        self._embed(tokens, x)
        for li, lw in enumerate(w.layers):
            if serial:
                qkv = self._stash[li, :T]
            else:
                qkv = self.pqkv[li & 1][:T]
                self._wait_buffer(main, self._buf_ev[li & 1])    # qkv buffer reuse
            self._norm(x, lw.attn_norm, lw.attn_norm_b, out=h)
            local = local_slots is not None and self.kv is not None
            if T > K.GEMV_MAX_ROWS and self.dh == 128:
                # RoPE (+ KV write into this GPU's pages) fused into the GEMM epilogue
                K.gemm_qkv_rope(h, lw.wqkv, qkv, positions, self.hq, self.hkv, self.theta,
                                bias=lw.bqkv,
                                k_layer=self.kv.k_layer_ptr(li) if local else None,
                                v_layer=self.kv.v_layer_ptr(li) if local else None,
                                slots=local_slots if local else None,
                                block_size=self.kv.block_size if local else 16,
                                rope_table=self.rope_tab)
            else:
                K.linear(h, lw.wqkv, K.EPI_BF16, out=qkv, bias=lw.bqkv)
                if local:
                    K.rope_kv_write(qkv, positions, self.hq, self.hkv, self.dh, self.theta,
                                    self.kv.k_layer_ptr(li), self.kv.v_layer_ptr(li),
                                    local_slots, self.kv.block_size)
                elif not self.bloom:
                    K.rope_kv_write(qkv, positions, self.hq, self.hkv, self.dh, self.theta)
            if push and not serial:
                ev = torch.cuda.Event()
                ev.record(main)
                self.push_stream.wait_event(ev)
                with torch.cuda.stream(self.push_stream):
                    if timing:
                        timing[li][0].record(self.push_stream)
                    for seg in push:
                        K.kv_push_layer(qkv[seg.row0:seg.row0 + seg.rows], seg.rows, self.hq,
                                        self.hkv, self.dh, seg.dst.k_layer_ptr(li),
                                        seg.dst.v_layer_ptr(li), seg.slots,
                                        seg.dst.block_size, self.push_ctas,
                                        stream=self.push_stream.cuda_stream)
                    if timing:
                        timing[li][1].record(self.push_stream)
                    done = torch.cuda.Event()
                    done.record(self.push_stream)
                self._buf_ev[li & 1] = done
            K.attn_prefill(qkv, cu, R, max(lens), self.hq, self.hkv, self.dh, self.scale,
                           out=attn, alibi=self.alibi)
            if self._stage_on(T):
                self._stage_layer(attn, lw, x, h, act, T)
            else:
                self._proj_reduce(attn, lw.wo, x, lw.bo)
                self._norm(x, lw.mlp_norm, lw.mlp_norm_b, out=h)
                self._mlp_up(h, lw, act)
                self._proj_reduce(act, lw.wd, x, lw.bd)
        last = self.plast[:R]
        self._norm(x, w.final_norm, w.final_norm_b, out=last, rows_index=last_rows)
        logits = self.plogits[:R]
        K.linear(last, self.head, K.EPI_F32, out=logits)
        first = self.pfirst[:R]
        self._greedy(logits, first)
        if push:
            compute_end = torch.cuda.Event(enable_timing=True)
            compute_end.record(main)
            self.push_stream.wait_event(compute_end)
            with torch.cuda.stream(self.push_stream):
                if serial:
                    # serialized mode: every layer of the finished prompts in one launch
                    if timing:
                        timing[0][0].record(self.push_stream)
                    for seg in push:
                        K.kv_push_layers(self._stash, seg.rows, self.hq, self.hkv, self.dh,
                                         seg.dst.k_layer_ptr(0), seg.dst.v_layer_ptr(0),
                                         seg.dst.info.layer_stride_bytes, seg.slots,
                                         seg.dst.block_size, self.push_ctas, row0=seg.row0,
                                         stream=self.push_stream.cuda_stream)
                    if timing:
                        timing[0][1].record(self.push_stream)
                for hnd in handoffs:
                    K.kv_handoff(first, hnd.seqs, hnd.epochs, hnd.table_ptr, hnd.stride,
                                 rows=hnd.rows, group_key=hnd.key,
                                 stream=self.push_stream.cuda_stream)
                tail = torch.cuda.Event()
                tail.record(self.push_stream)
            # the next batch reuses the buffers (and pfirst) only after this tail
            if serial:
                self._stash_ev = tail
            else:
                self._buf_ev[(cfg.n_layers - 1) & 1] = tail
            if not handoffs:
                main.wait_event(tail)       # KV fully landed before we report done
            if push_stats is not None:
                self._pending_push.append((timing, compute_start, compute_end, tail, push_stats))
        return first
    def mixed(self, tokens: torch.Tensor, lens: list[int], meta: torch.Tensor,
              local_slots: torch.Tensor, dec_tables: torch.Tensor, dec_tok: torch.Tensor,
              dec_ctx: torch.Tensor, dec_max_ctx: int) -> torch.Tensor:
        """One mixed iteration (reference machine.py:181-243 mixed batches): the
        prompt rows of a prefill batch and one decode token for each of Bd
        running sequences go through every weight GEMM together, so the
        iteration streams the weights once; attention splits by row kind —
        causal prefill attention (+ RoPE/KV write) for the prompt rows, paged
        decode attention (RoPE + KV append at position dec_ctx) for the
        decode rows.  Prompt KV goes to this machine's pool (local_slots).

        tokens      int32 [T] prompt tokens; meta as for ``prefill``
        dec_tables  int32 [Bd, max_blocks] table rows of the decoding sequences
        dec_tok     int32 [Bd] their current tokens; dec_ctx int32 [Bd] cached
                    lengths (advanced by one here)
        Returns int32 [R + Bd]: first tokens of the prompts, then the decode rows'
        next tokens."""
        cfg, w, kv = self.cfg, self.w, self.kv
        T, R, Bd = int(tokens.shape[0]), len(lens), int(dec_tok.shape[0])
        rows = T + Bd
        self._ensure_prefill(rows, R + Bd)
        positions = meta[:T]
        cu = meta[T:T + R + 1]
        last_rows = meta[T + R + 1:T + 2 * R + 1]
        x, h, attn, act = self.px[:rows], self.ph[:rows], self.pattn[:rows], self.pact[:rows]
        key = ("mixed_ws", Bd, dec_max_ctx)
        ws = self.graphs.get(key)
        if ws is None:
            ws = torch.zeros(K.attn_decode_workspace_bytes(Bd, self.hq, dec_max_ctx,
                                                           self.partition, self.dh),
                             dtype=torch.uint8, device=self.dev)
            self.graphs[key] = ws
        self._wait_push_tails()
        self._begin_reductions()
        self._embed(torch.cat([tokens, dec_tok]), x)
        for li, lw in enumerate(w.layers):
            qkv = self.pqkv[0][:rows]
            self._norm(x, lw.attn_norm, lw.attn_norm_b, out=h)
            K.linear(h, lw.wqkv, K.EPI_BF16, out=qkv, bias=lw.bqkv)
            K.rope_kv_write(qkv[:T], positions, self.hq, self.hkv, self.dh, self.theta,
                            kv.k_layer_ptr(li), kv.v_layer_ptr(li), local_slots, kv.block_size)
            K.attn_prefill(qkv[:T], cu, R, max(lens), self.hq, self.hkv, self.dh, self.scale,
                           out=attn[:T], alibi=self.alibi)
            K.attn_decode_step(qkv[T:], kv.k_layer_ptr(li), kv.v_layer_ptr(li), dec_tables,
                               dec_ctx, Bd, self.hq, self.hkv, self.dh, kv.block_size,
                               self.scale, dec_max_ctx, self.partition, ws, out=attn[T:],
                               theta=cfg.rope_theta, alibi=self.alibi)
            self._proj_reduce(attn, lw.wo, x, lw.bo)
            self._norm(x, lw.mlp_norm, lw.mlp_norm_b, out=h)
            self._mlp_up(h, lw, act)
            self._proj_reduce(act, lw.wd, x, lw.bd)
        idx = torch.cat([last_rows, torch.arange(T, rows, dtype=torch.int32, device=self.dev)])
        last = self.plast[:R + Bd]
        self._norm(x, w.final_norm, w.final_norm_b, out=last, rows_index=idx)
        logits = self.plogits[:R + Bd]
        K.linear(last, self.head, K.EPI_F32, out=logits)
        nxt = self.pfirst[:R + Bd]
        self._greedy(logits, nxt)
        dec_ctx += 1
        return nxt

    def mixed_chunk(self, tokens: torch.Tensor, seq: int, start: int,
                    dec_tables: torch.Tensor | None = None, dec_tok: torch.Tensor | None = None,
                    dec_ctx: torch.Tensor | None = None, dec_max_ctx: int = 0) -> torch.Tensor:
        """One chunked-prefill iteration (workers.Machine with
        prefill_chunk_tokens): rows [0, n) are prompt positions start..start+n
        of sequence ``seq`` of this machine's pool (RoPE'd, K/V written to
        their pages, causal attention over every page up to their own
        position — swb_attn_chunk), rows [n, n+Bd) one decode token of each
        running sequence (paged decode attention + KV append, as in
        ``mixed``); every weight GEMM runs once over all rows.  Returns int32
        [1 + Bd]: the greedy token after the chunk's last row (the prompt's
        first token when the chunk is its last) and the decode rows' next
        tokens; dec_ctx advances by one."""
        cfg, w, kv = self.cfg, self.w, self.kv
        n = int(tokens.shape[0])
        Bd = 0 if dec_tok is None else int(dec_tok.shape[0])
        rows = n + Bd
        self._ensure_prefill(rows, 1 + Bd)
        x, h, attn, act = self.px[:rows], self.ph[:rows], self.pattn[:rows], self.pact[:rows]
        positions = torch.arange(start, start + n, dtype=torch.int32, device=self.dev)
        slots = torch.empty(n, dtype=torch.int32, device=self.dev)
        K.slots_from_table(kv.table_row_ptr(seq), start, n, kv.block_size, slots)
        max_ctx = kv.max_blocks_per_seq * kv.block_size
        ws = self.graphs.get(("chunk_ws", n, max_ctx))
        if ws is None:
            ws = torch.zeros(K.attn_chunk_workspace_bytes(n, self.hq, max_ctx),
                             dtype=torch.uint8, device=self.dev)
            self.graphs[("chunk_ws", n, max_ctx)] = ws
        if Bd:
            dws = self.graphs.get(("mixed_ws", Bd, dec_max_ctx))
            if dws is None:
                dws = torch.zeros(K.attn_decode_workspace_bytes(Bd, self.hq, dec_max_ctx,
                                                                self.partition, self.dh),
                                  dtype=torch.uint8, device=self.dev)
                self.graphs[("mixed_ws", Bd, dec_max_ctx)] = dws
        self._wait_push_tails()
        self._begin_reductions()
        self._embed(tokens if not Bd else torch.cat([tokens, dec_tok]), x)
        for li, lw in enumerate(w.layers):
            qkv = self.pqkv[0][:rows]
            self._norm(x, lw.attn_norm, lw.attn_norm_b, out=h)
            K.linear(h, lw.wqkv, K.EPI_BF16, out=qkv, bias=lw.bqkv)
            K.rope_kv_write(qkv[:n], positions, self.hq, self.hkv, self.dh, self.theta,
                            kv.k_layer_ptr(li), kv.v_layer_ptr(li), slots, kv.block_size)
            K.attn_chunk(qkv[:n], n, start, kv.k_layer_ptr(li), kv.v_layer_ptr(li),
                         kv.table_row_ptr(seq), self.hq, self.hkv, self.dh, kv.block_size,
                         self.scale, max_ctx, ws, attn[:n], alibi=self.alibi)
            if Bd:
                K.attn_decode_step(qkv[n:], kv.k_layer_ptr(li), kv.v_layer_ptr(li), dec_tables,
                                   dec_ctx, Bd, self.hq, self.hkv, self.dh, kv.block_size,
                                   self.scale, dec_max_ctx, self.partition, dws, out=attn[n:],
                                   theta=cfg.rope_theta, alibi=self.alibi)
            self._proj_reduce(attn, lw.wo, x, lw.bo)
            self._norm(x, lw.mlp_norm, lw.mlp_norm_b, out=h)
            self._mlp_up(h, lw, act)
            self._proj_reduce(act, lw.wd, x, lw.bd)
        idx = torch.arange(n - 1, rows, dtype=torch.int32, device=self.dev)
        last = self.plast[:1 + Bd]
        self._norm(x, w.final_norm, w.final_norm_b, out=last, rows_index=idx)
        logits = self.plogits[:1 + Bd]
        K.linear(last, self.head, K.EPI_F32, out=logits)
        nxt = self.pfirst[:1 + Bd]
        self._greedy(logits, nxt)
        if Bd:
            dec_ctx += 1
        return nxt

    def prefill_chunked(self, tokens: torch.Tensor, seq: int, chunk: int = 512) -> torch.Tensor:
        """Prompt phase of ONE prompt in chunks of ``chunk`` tokens against this
        GPU's pool (sequence slot ``seq``): every chunk's QKV GEMM rotates and
        writes its K/V into the pages (fused epilogue), then the chunk's
        queries attend over all pages up to their own position
        (swb_attn_chunk).  Same result as ``prefill`` with local slots (within
        bf16 rounding); bounds the rows per iteration so a long prompt can
        share iterations with decode rows.  Returns the first token (int32 [1])."""
        cfg, w, kv = self.cfg, self.w, self.kv
        P = int(tokens.shape[0])
        self._ensure_prefill(min(P, chunk), 1)
        slots = torch.empty(P, dtype=torch.int32, device=self.dev)
        K.slots_from_table(kv.table_row_ptr(seq), 0, P, kv.block_size, slots)
        max_ctx = kv.max_blocks_per_seq * kv.block_size
        key = ("chunk_ws", chunk, max_ctx)
        ws = self.graphs.get(key)
        if ws is None:
            ws = torch.zeros(K.attn_chunk_workspace_bytes(chunk, self.hq, max_ctx),
                             dtype=torch.uint8, device=self.dev)
            self.graphs[key] = ws
        self._wait_push_tails()
        self._begin_reductions()
        for c0 in range(0, P, chunk):
            n = min(chunk, P - c0)
            x, h, attn, act = self.px[:n], self.ph[:n], self.pattn[:n], self.pact[:n]
            qkv = self.pqkv[0][:n]
            positions = torch.arange(c0, c0 + n, dtype=torch.int32, device=self.dev)
            self._embed(tokens[c0:c0 + n], x)
            for li, lw in enumerate(w.layers):
                self._norm(x, lw.attn_norm, lw.attn_norm_b, out=h)
                K.gemm_qkv_rope(h, lw.wqkv, qkv, positions, self.hq, self.hkv, self.theta,
                                bias=lw.bqkv, k_layer=kv.k_layer_ptr(li),
                                v_layer=kv.v_layer_ptr(li), slots=slots[c0:c0 + n],
                                block_size=kv.block_size, rope_table=self.rope_tab)
                K.attn_chunk(qkv, n, c0, kv.k_layer_ptr(li), kv.v_layer_ptr(li),
                             kv.table_row_ptr(seq), self.hq, self.hkv, self.dh, kv.block_size,
                             self.scale, max_ctx, ws, attn, alibi=self.alibi)
                self._proj_reduce(attn, lw.wo, x, lw.bo)
                self._norm(x, lw.mlp_norm, lw.mlp_norm_b, out=h)
                self._mlp_up(h, lw, act)
                self._proj_reduce(act, lw.wd, x, lw.bd)
        last = self.plast[:1]
        idx = torch.tensor([n - 1], dtype=torch.int32, device=self.dev)
        self._norm(x, w.final_norm, w.final_norm_b, out=last, rows_index=idx)
        logits = self.plogits[:1]
        K.linear(last, self.head, K.EPI_F32, out=logits)
        first = self.pfirst[:1]
        self._greedy(logits, first)
        return first

    def finish_push_stats(self, block: bool = True):
        """Resolve the push timings of finished prefills (all of them when
        ``block``); returns the latest resolved PushStats or None."""
        last = None
        while self._pending_push:
            timing, c0, c1, tail, st = self._pending_push[0]
            if block:
                tail.synchronize()
            elif not tail.query():
                break
            self._pending_push.pop(0)
            st.layer_ms = [a.elapsed_time(b) for a, b in timing]
            st.total_ms = timing[0][0].elapsed_time(timing[-1][1])
            st.tail_ms = max(0.0, c1.elapsed_time(timing[-1][1]))
            st.compute_ms = c0.elapsed_time(c1)
            last = st
        return last

    @staticmethod
    def pack_meta(lens: list[int]) -> torch.Tensor:
        """Host int32 [positions | cu_seqlens | last_rows] for ``prefill``."""
        pos, cu, last = [], [0], []
        for n in lens:
            pos.extend(range(n))
            cu.append(cu[-1] + n)
            last.append(cu[-1] - 1)
        return torch.tensor(pos + cu + last, dtype=torch.int32)

    # ------------------------------------------------------------- decode
    def decode_partition(self, B: int, max_ctx: int) -> int:
        """Context partition of decode attention.  GQA groups (tensor-core
        kernel) and short grids: 128 tokens — smaller partitions only add
        split-K merge work (7B B=1 10.0 vs 10.7 us per layer at 64; 70B TP4
        B=1 step 10.9 vs 12.7 ms at 32).  MHA with >= 4 CTAs per SM at 128:
        64 tokens (half the staged pages per CTA, twice the CTAs resident):
        7B B=8 44.8 vs 48.9 us, B=32 142 vs 165 us per layer.
        SWB_DECODE_PART overrides; ``decode_partition=`` pins it."""
        env = os.environ.get("SWB_DECODE_PART")
        if env:
            return int(env)
        if self.partition != 128:
            return self.partition
        mha = self.hq // self.hkv < 4
        if mha and B * self.hkv * ((max_ctx + 127) // 128) >= 4 * 148:
            return 64
        return 128

    def decode_graph(self, B: int, max_ctx: int, ring: int) -> "DecodeGraph":
        part = self.decode_partition(B, max_ctx)
        np_ = (max_ctx + part - 1) // part
        key = (B, np_ * part, part, ring)
        g = self.graphs.get(key)
        if g is None:
            g = DecodeGraph(self, B, np_ * part, ring, part)
            self.graphs[key] = g
        return g


class DecodeGraph:
    """Static buffers + captured CUDA graph of one decode iteration at batch B."""

    def __init__(self, runner: ModelRunner, B: int, max_ctx: int, ring: int, part: int = 128):
        self.r = runner
        self.part = part
        self.B = B
        self.max_ctx = max_ctx
        self.ring = ring
        cfg, dev = runner.cfg, runner.dev
        kv = runner.kv
        i32 = dict(dtype=torch.int32, device=dev)
        self.cur_tok = torch.zeros(B, **i32)
        self.ctx = torch.zeros(B, **i32)
        self.step = torch.zeros(B, **i32)
        self.out_ring = torch.zeros(B, ring, **i32)
        self.tables = torch.zeros(B, kv.max_blocks_per_seq, **i32)
        self.pos = torch.zeros(B, **i32)
        self.slots = torch.zeros(B, **i32)
        self.attn_len = torch.zeros(B, **i32)
        self.next_tok = torch.zeros(B, **i32)
        d = cfg.d_model
        self.x = torch.zeros(B, d, dtype=torch.float32, device=dev)
        self.h = torch.zeros(B, d, dtype=torch.bfloat16, device=dev)
        self.qkv = torch.zeros(B, runner.qkv_cols, dtype=torch.bfloat16, device=dev)
        self.attn = torch.zeros(B, runner.hq * runner.dh, dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros(B, runner.ffn, dtype=torch.bfloat16, device=dev)
        self.logits = torch.zeros(B, runner.vocab_local, dtype=torch.float32, device=dev)
        wsb = K.attn_decode_workspace_bytes(B, runner.hq, max_ctx, part, runner.dh)
        self.ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
        self.graph = None

    def _step_body(self):
        r, cfg, w, kv = self.r, self.r.cfg, self.r.w, self.r.kv
        B = self.B
        r._begin_reductions()
        r._embed(self.cur_tok, self.x)
        # pre-norm folded into the weight-streaming GEMV: h = rmsnorm(x) is
        # normalised once into shared memory per CTA (B=1: CUDA-core kernel;
        # B=2..8 with h <= 32 KB: mma.sync kernel, rstd reduced in
        # swb_rmsnorm's order, bit-identical to the two-kernel path) while the
        # weight ring fills; SWB_FUSED_NORM=0/1 forces it off/on (Llama).  Auto
        # = B=1, and B=2 for d <= 4096: 7B B=2 3.253 vs 3.285 ms/step with the
        # separate norm, but B=4 3.85 vs 3.79 and 70B TP2 B=2 15.41 vs 15.35
        # (the staged variant's 4-stage ring costs more than the launch it
        # saves once h grows)
        mode = os.environ.get("SWB_FUSED_NORM", "auto")
        fused = ((B == 1 and cfg.d_model * 2 <= 16384) or (B == 2 and cfg.d_model <= 4096)
                 if mode == "auto" else mode == "1")
        fused = fused and not r.bloom
        for li, lw in enumerate(w.layers):
            if fused:
                K.gemv_rmsnorm(self.x, lw.attn_norm, cfg.norm_eps, lw.wqkv, K.EPI_BF16,
                               out=self.qkv)
            else:
                r._norm(self.x, lw.attn_norm, lw.attn_norm_b, out=self.h)
                K.linear(self.h, lw.wqkv, K.EPI_BF16, out=self.qkv, bias=lw.bqkv)
            # RoPE (or ALiBi) + KV append of the current token at position
            # ctx + attention + split-K merge; the cached pages are gathered
            # before the PDL wait (ctx / tables come from the previous replay)
            K.attn_decode_step(self.qkv, kv.k_layer_ptr(li), kv.v_layer_ptr(li), self.tables,
                               self.ctx, B, r.hq, r.hkv, r.dh, kv.block_size, r.scale,
                               self.max_ctx, self.part, self.ws, out=self.attn,
                               theta=cfg.rope_theta, alibi=r.alibi)
            r._proj_reduce(self.attn, lw.wo, self.x, lw.bo)
            if fused:
                K.gemv_rmsnorm(self.x, lw.mlp_norm, cfg.norm_eps, lw.wgu, K.EPI_SWIGLU,
                               out=self.act)
            else:
                r._norm(self.x, lw.mlp_norm, lw.mlp_norm_b, out=self.h)
                r._mlp_up(self.h, lw, self.act)
            r._proj_reduce(self.act, lw.wd, self.x, lw.bd)
        if fused:
            K.gemv_rmsnorm(self.x, w.final_norm, cfg.norm_eps, r.head, K.EPI_F32,
                           out=self.logits)
        else:
            r._norm(self.x, w.final_norm, w.final_norm_b, out=self.h)
            K.linear(self.h, r.head, K.EPI_F32, out=self.logits)
        r._greedy(self.logits, self.next_tok)
        K.decode_advance(self.next_tok, self.cur_tok, self.ctx, self.step, self.out_ring, B)

    def load(self, seqs: list[int], cur_tok, ctx, steps=None):
        """Bind batch rows to KV sequence slots and their state (host lists
        or device tensors).  Called when the batch composition changes."""
        kv = self.r.kv
        # host mirror of the largest context: a replay past the bucket would
        # append K/V outside every attention partition (silently dropped)
        self._ctx_max = (None if isinstance(ctx, torch.Tensor) and ctx.is_cuda
                         else int(max(torch.as_tensor(ctx).tolist(), default=0)))
        if self._ctx_max is not None and self._ctx_max >= self.max_ctx:
            raise CapacityError(f"context {self._ctx_max} >= decode bucket {self.max_ctx}")
        idx = torch.tensor(seqs, dtype=torch.long, device=self.r.dev)
        torch.index_select(kv.tables(), 0, idx, out=self.tables)
        self.cur_tok.copy_(torch.as_tensor(cur_tok, dtype=torch.int32), non_blocking=True)
        self.ctx.copy_(torch.as_tensor(ctx, dtype=torch.int32), non_blocking=True)
        if steps is None:
            self.step.zero_()
        else:
            self.step.copy_(torch.as_tensor(steps, dtype=torch.int32), non_blocking=True)

    def capture(self):
        s = torch.cuda.Stream(device=self.r.dev)
        s.wait_stream(torch.cuda.current_stream())
        # snapshot state: a warm-up step mutates ctx/step/cur_tok/out_ring/KV
        saved = [t.clone() for t in (self.cur_tok, self.ctx, self.step)]
        with torch.cuda.stream(s):
            self._step_body()  # warm-up (lazy attrs, workspace) outside capture
        torch.cuda.current_stream().wait_stream(s)
        for t, v in zip((self.cur_tok, self.ctx, self.step), saved):
            t.copy_(v)
        g = torch.cuda.CUDAGraph()
        n0 = _abi.launch_count()
        # a garbage-collected KV pool / TP communicator frees device memory
        # (cudaFree), which is illegal while a stream captures and would
        # invalidate the capture: collect now, and not during the capture
        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()
        # explicit capture stream on this runner's device: torch.cuda.graph's
        # default capture stream is created once, on whichever device was
        # current then, and would bind a second GPU's graph to the first GPU
        try:
            with torch.cuda.graph(g, stream=torch.cuda.Stream(device=self.r.dev)):
                self._step_body()
        finally:
            if gc_was:
                gc.enable()
        if self.r.tp_comm is not None:
            self.r.tp_comm.assert_even()
        self.launches_per_step = _abi.launch_count() - n0
        _abi.add_launches(-self.launches_per_step)  # capture launches nothing
        self.graph = g

    def replay(self):
        if getattr(self, "_ctx_max", None) is not None:
            if self._ctx_max >= self.max_ctx:
                raise CapacityError(f"decode step at context {self._ctx_max} overruns the "
                                    f"{self.max_ctx}-token bucket")
            self._ctx_max += 1
        if self.graph is None:
            self._step_body()
        else:
            self.graph.replay()
            _abi.add_launches(self.launches_per_step)
