"""Tensor-level wrappers over the C-ABI kernels (device memory comes from
PyTorch; all arithmetic runs in libswb200.so).  Each wrapper validates dtype,
device and contiguity, then launches on the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _abi
from ._abi import EPI_BF16, EPI_F32, EPI_GELU, EPI_RESID_F32, EPI_SWIGLU, call
from .errors import ValidationError

__all__ = ["gemm", "gemv", "gemv_rmsnorm", "linear", "embed", "rmsnorm", "layernorm", "argmax",
           "rope_kv_write",
           "kv_push_layer", "kv_push_layers", "kv_handoff", "attn_prefill", "attn_decode",
           "attn_decode_step", "decode_advance", "slots_from_table",
           "gemv_tp", "EPI_BF16", "EPI_F32", "EPI_RESID_F32", "EPI_SWIGLU", "EPI_GELU",
           "GEMV_MAX_ROWS"]

# rows handled by the weight-streaming GEMVs (the tcgen05 GEMV takes up to 32)
GEMV_MAX_ROWS = 16 if os.environ.get("SWB_GEMV_TC", "1") == "0" else 32


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _req(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValidationError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValidationError(f"{name} must be contiguous")


def _out_shape(M, N, epi):
    return (M, N // 2) if epi == EPI_SWIGLU else (M, N)


def _alloc_out(a, M, N, epi):
    dt = torch.bfloat16 if epi in (EPI_BF16, EPI_SWIGLU, EPI_GELU) else torch.float32
    return torch.empty(_out_shape(M, N, epi), dtype=dt, device=a.device)


def _ptr(t):
    return t.data_ptr() if t is not None else None


def gemm(a, w, epi=EPI_BF16, out=None, resid=None, bias=None):
    """tcgen05 GEMM: out = epi(a[M,K] @ w[N,K]^T + bias)."""
    _req(a, torch.bfloat16, "a")
    _req(w, torch.bfloat16, "w")
    M, K = a.shape
    N = w.shape[0]
    if w.shape[1] != K:
        raise ValidationError(f"K mismatch {a.shape} vs {w.shape}")
    if out is None:
        out = _alloc_out(a, M, N, epi)
    call("swb_gemm_bf16_bias", a.data_ptr(), w.data_ptr(), out.data_ptr(), _ptr(resid),
         _ptr(bias), M, N, K, epi, _stream())
    return out


def gemv(x, w, epi=EPI_BF16, out=None, resid=None, bias=None):
    """Weight-streaming skinny GEMM for M <= 16 rows."""
    _req(x, torch.bfloat16, "x")
    _req(w, torch.bfloat16, "w")
    M, K = x.shape
    N = w.shape[0]
    if out is None:
        out = _alloc_out(x, M, N, epi)
    call("swb_gemv_bf16_bias", x.data_ptr(), w.data_ptr(), out.data_ptr(), _ptr(resid),
         _ptr(bias), M, N, K, epi, _stream())
    return out


def gemm_qkv_rope(a, w, qkv, positions, H, Hkv, theta, bias=None, k_layer=None, v_layer=None,
                  slots=None, block_size=16, rope_table=None):
    """Prefill QKV projection with RoPE (+ KV write into the paged pool) fused
    into the tcgen05 GEMM epilogue; bit-identical to gemm + rope_kv_write.
    rope_table: fp32 [max_pos, 64, 2] from ``rope_table`` (optional)."""
    _req(a, torch.bfloat16, "a")
    M, Kd = a.shape
    call("swb_gemm_qkv_rope", a.data_ptr(), w.data_ptr(), qkv.data_ptr(), _ptr(bias), M,
         w.shape[0], Kd, positions.data_ptr(), float(theta), _ptr(rope_table),
         0 if rope_table is None else rope_table.shape[0], H, Hkv, k_layer, v_layer,
         _ptr(slots), block_size, _stream())
    return qkv


def rope_table(theta, max_pos, device=None):
    """(sin, cos) of every RoPE angle for positions < max_pos, head_dim 128."""
    t = torch.empty(max_pos, 64, 2, dtype=torch.float32, device=device or "cuda")
    call("swb_rope_table", float(theta), max_pos, t.data_ptr(), _stream())
    return t


def gemv_rmsnorm(x, norm_w, eps, w, epi=EPI_BF16, out=None, resid=None):
    """Decode pre-norm linear: out = epi(rmsnorm(x fp32) @ w^T), one kernel."""
    _req(x, torch.float32, "x")
    _req(w, torch.bfloat16, "w")
    _req(norm_w, torch.bfloat16, "norm_w")
    M, K = x.shape
    N = w.shape[0]
    if out is None:
        out = _alloc_out(x, M, N, epi)
    call("swb_gemv_rmsnorm_bf16", x.data_ptr(), norm_w.data_ptr(), float(eps), w.data_ptr(),
         out.data_ptr(), resid.data_ptr() if resid is not None else None, M, N, K, epi,
         _stream())
    return out


def linear(x, w, epi=EPI_BF16, out=None, resid=None, bias=None):
    """Dispatch on row count: <= 16 rows streams weights (decode), more rows
    go to the tcgen05 GEMM (prefill).  Both are native kernels."""
    if x.shape[0] <= GEMV_MAX_ROWS:
        return gemv(x, w, epi, out, resid, bias)
    return gemm(x, w, epi, out, resid, bias)


def gemv_tp(x, w, epi, comm_handle, slot, resid=None, bias=None):
    """Fused projection + all-reduce push (one decode row): the fp32 partial
    lands in this rank's TP slot ``slot`` and, from the epilogue, in every
    peer's receive buffer; finish with TPComm.allreduce_recv(slot, out)."""
    _req(x, torch.bfloat16, "x")
    _req(w, torch.bfloat16, "w")
    if x.shape[0] != 1 or w.shape[1] != x.shape[1]:
        raise ValidationError(f"gemv_tp: one row with K = {w.shape[1]}, got {tuple(x.shape)}")
    call("swb_gemv_bf16_tp", x.data_ptr(), w.data_ptr(), _ptr(resid), _ptr(bias), 1,
         w.shape[0], w.shape[1], epi, comm_handle, slot, _stream())


def embed(tokens, table, out=None):
    _req(tokens, torch.int32, "tokens")
    _req(table, torch.bfloat16, "table")
    rows, d = tokens.shape[0], table.shape[1]
    if out is None:
        out = torch.empty(rows, d, dtype=torch.float32, device=table.device)
    call("swb_embed", tokens.data_ptr(), table.data_ptr(), out.data_ptr(), rows, d, _stream())
    return out


def _parts(parts, x, fn):
    """Pointer array of the TP ranks' bf16 partials (each x's shape)."""
    if not 1 <= len(parts) <= 8:
        raise ValidationError(f"{fn}: 1..8 partials, got {len(parts)}")
    for p in parts:
        _req(p, torch.bfloat16, "addend")
        if p.shape != x.shape:
            raise ValidationError(f"{fn}: every partial must match x")
    return (ctypes.c_void_p * len(parts))(*[p.data_ptr() for p in parts])


def rmsnorm(x, w, eps, rows_index=None, out=None, addend=None):
    """RMSNorm of fp32 rows; with ``addend`` (bf16, x's shape) the rows first
    get x += addend (written back); a list of bf16 partials (the TP ranks',
    rank order) is summed in fp32 first."""
    _req(x, torch.float32, "x")
    _req(w, torch.bfloat16, "w")
    rows = x.shape[0] if rows_index is None else rows_index.shape[0]
    d = x.shape[1]
    if out is None:
        out = torch.empty(rows, d, dtype=torch.bfloat16, device=x.device)
    if isinstance(addend, (list, tuple)):
        arr = _parts(addend, x, "rmsnorm")
        call("swb_add_parts_rmsnorm", x.data_ptr(), arr, len(addend), _ptr(rows_index),
             w.data_ptr(), out.data_ptr(), rows, d, float(eps), _stream())
        return out
    if addend is not None:
        _req(addend, torch.bfloat16, "addend")
        if addend.shape != x.shape:
            raise ValidationError("rmsnorm: addend must match x")
        call("swb_add_rmsnorm", x.data_ptr(), addend.data_ptr(), _ptr(rows_index), w.data_ptr(),
             out.data_ptr(), rows, d, float(eps), _stream())
        return out
    call("swb_rmsnorm", x.data_ptr(), rows_index.data_ptr() if rows_index is not None else None,
         w.data_ptr(), out.data_ptr(), rows, d, float(eps), _stream())
    return out


def layernorm(x, w, b, eps, rows_index=None, out=None, out_f32=False, addend=None):
    """LayerNorm with bias (BLOOM); fp32 out (may be x) when out_f32; with
    ``addend`` (bf16) the rows first get x += addend (written back); a list of
    bf16 partials (rank order) is summed in fp32 first."""
    _req(x, torch.float32, "x")
    _req(w, torch.bfloat16, "w")
    _req(b, torch.bfloat16, "b")
    rows = x.shape[0] if rows_index is None else rows_index.shape[0]
    d = x.shape[1]
    if out is None:
        out = torch.empty(rows, d, dtype=torch.float32 if out_f32 else torch.bfloat16,
                          device=x.device)
    if isinstance(addend, (list, tuple)):
        if out_f32:
            raise ValidationError("layernorm: partials need the bf16 output")
        arr = _parts(addend, x, "layernorm")
        call("swb_add_parts_layernorm", x.data_ptr(), arr, len(addend), _ptr(rows_index),
             w.data_ptr(), b.data_ptr(), out.data_ptr(), rows, d, float(eps), _stream())
        return out
    if addend is not None:
        _req(addend, torch.bfloat16, "addend")
        if addend.shape != x.shape or out_f32:
            raise ValidationError("layernorm: addend must match x (bf16 output only)")
        call("swb_add_layernorm", x.data_ptr(), addend.data_ptr(), _ptr(rows_index),
             w.data_ptr(), b.data_ptr(), out.data_ptr(), rows, d, float(eps), _stream())
        return out
    call("swb_layernorm", x.data_ptr(), _ptr(rows_index), w.data_ptr(), b.data_ptr(),
         out.data_ptr(), rows, d, float(eps), int(bool(out_f32)), _stream())
    return out


def argmax(logits, out=None):
    _req(logits, torch.float32, "logits")
    rows, V = logits.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.int32, device=logits.device)
    call("swb_argmax", logits.data_ptr(), rows, V, out.data_ptr(), _stream())
    return out


def argmax_shard(logits, offset, rank, tp, cand):
    rows, V = logits.shape
    call("swb_argmax_shard", logits.data_ptr(), rows, V, offset, rank, tp, cand.data_ptr(),
         _stream())
    return cand


def argmax_pick(cand, rows, tp, out):
    call("swb_argmax_pick", cand.data_ptr(), rows, tp, out.data_ptr(), _stream())
    return out


def rope_kv_write(qkv, positions, H, Hkv, dh, theta, k_layer=None, v_layer=None,
                  slots=None, block_size=16, rows=None):
    _req(qkv, torch.bfloat16, "qkv")
    _req(positions, torch.int32, "positions")
    rows = qkv.shape[0] if rows is None else rows
    call("swb_rope_kv_write", qkv.data_ptr(), rows, qkv.shape[1], positions.data_ptr(), H, Hkv,
         dh, float(theta), k_layer, v_layer,
         slots.data_ptr() if slots is not None else None, block_size, _stream())


def kv_push_layer(qkv, rows, H, Hkv, dh, dst_k, dst_v, dst_slots, block_size, num_ctas=0,
                  stream=None):
    """Pack-and-push one layer's k/v rows into (possibly peer) paged blocks."""
    call("swb_kv_push_layer", qkv.data_ptr(), rows, qkv.shape[1], H * dh, (H + Hkv) * dh, Hkv,
         dh, dst_k, dst_v, dst_slots.data_ptr(), block_size, num_ctas,
         stream if stream is not None else _stream())


def kv_push_layers(qkv_stack, rows, H, Hkv, dh, dst_k0, dst_v0, dst_layer_stride, dst_slots,
                   block_size, num_ctas=0, row0=0, stream=None):
    """Serialized mode: push rows [row0, row0+rows) of every layer of
    qkv_stack [L, T, qkv_cols] into the destination pool in ONE launch."""
    _req(qkv_stack, torch.bfloat16, "qkv_stack")
    L, T, cols = qkv_stack.shape
    if row0 < 0 or row0 + rows > T:
        raise ValidationError("kv_push_layers: rows outside the stash")
    call("swb_kv_push_layers", qkv_stack.data_ptr() + 2 * row0 * cols, T * cols, L, rows, cols,
         H * dh,
         (H + Hkv) * dh, Hkv, dh, dst_k0, dst_v0, dst_layer_stride, dst_slots.data_ptr(),
         block_size, num_ctas, stream if stream is not None else _stream())


def attn_prefill(qkv, cu_seqlens, num_seqs, max_seqlen, H, Hkv, dh, scale, out=None,
                 impl=None, alibi=None):
    """Causal varlen prefill attention.  impl "tc" = tcgen05/TMEM kernel (the
    default; SWB_ATTN_TC=0 selects the mma.sync FlashAttention-2 kernel).
    ``alibi``: fp32 [H] slopes (BLOOM), tcgen05 kernel only."""
    _req(qkv, torch.bfloat16, "qkv")
    _req(cu_seqlens, torch.int32, "cu_seqlens")
    if out is None:
        out = torch.empty(qkv.shape[0], H * dh, dtype=torch.bfloat16, device=qkv.device)
    if impl is None:
        impl = "fa2" if os.environ.get("SWB_ATTN_TC", "1") == "0" else "tc"
    if alibi is not None:
        _req(alibi, torch.float32, "alibi")
        if impl != "tc":
            raise ValidationError("ALiBi prefill attention is implemented by the tcgen05 kernel")
    if impl == "tc":
        call("swb_attn_prefill_tc", qkv.data_ptr(), qkv.shape[1], qkv.shape[0],
             cu_seqlens.data_ptr(), num_seqs, max_seqlen, H, Hkv, dh, float(scale),
             _ptr(alibi), out.data_ptr(), _stream())
    else:
        call("swb_attn_prefill", qkv.data_ptr(), qkv.shape[1], cu_seqlens.data_ptr(), num_seqs,
             max_seqlen, H, Hkv, dh, float(scale), out.data_ptr(), _stream())
    return out


def attn_decode_workspace_bytes(B, H, max_ctx, partition, dh):
    return int(_abi.lib.swb_attn_decode_workspace(B, H, max_ctx, partition, dh))


def attn_decode(qkv, k_layer, v_layer, block_tables, ctx_lens, B, H, Hkv, dh, block_size,
                scale, max_ctx, partition, workspace, out=None, positions=None, slots=None,
                theta=10000.0, alibi=None):
    """Paged decode attention; with positions/slots it also applies RoPE to the
    current token and appends its K/V to the pool (one kernel per layer).
    ``workspace`` must be zero-initialised once (merge tickets)."""
    if out is None:
        out = torch.empty(B, H * dh, dtype=torch.bfloat16, device=qkv.device)
    call("swb_attn_decode", qkv.data_ptr(), qkv.shape[1], k_layer, v_layer,
         block_tables.data_ptr(), block_tables.shape[1], ctx_lens.data_ptr(),
         positions.data_ptr() if positions is not None else None,
         slots.data_ptr() if slots is not None else None, float(theta), _ptr(alibi), B, H,
         Hkv, dh,
         block_size, float(scale), max_ctx, partition, workspace.data_ptr(), out.data_ptr(),
         _stream())
    return out


def attn_decode_step(qkv, k_layer, v_layer, block_tables, ctx, B, H, Hkv, dh, block_size,
                     scale, max_ctx, partition, workspace, out, theta=10000.0, alibi=None):
    """Decode-graph attention: the current token sits at position ctx[b] (RoPE
    there, KV appended at the table's slot) and attends over ctx[b]+1 tokens;
    the cached pages are gathered before the PDL wait (see swb200.h)."""
    call("swb_attn_decode_step", qkv.data_ptr(), qkv.shape[1], k_layer, v_layer,
         block_tables.data_ptr(), block_tables.shape[1], ctx.data_ptr(), float(theta),
         _ptr(alibi), B, H, Hkv, dh, block_size, float(scale), max_ctx, partition,
         workspace.data_ptr(), out.data_ptr(), _stream())
    return out


def attn_chunk_workspace_bytes(C, H, max_ctx):
    return int(_abi.lib.swb_attn_chunk_workspace(C, H, max_ctx))


def attn_chunk(qkv, C, q_start, k_layer, v_layer, table_row_ptr, H, Hkv, dh, block_size, scale,
               max_ctx, workspace, out, alibi=None):
    """Causal attention of a prompt chunk (positions q_start..) over the paged pool."""
    call("swb_attn_chunk", qkv.data_ptr(), qkv.shape[1], C, q_start, k_layer, v_layer,
         table_row_ptr, H, Hkv, dh, block_size, float(scale), _ptr(alibi), max_ctx,
         workspace.data_ptr(), out.data_ptr(), _stream())
    return out


def decode_advance(next_tok, cur_tok, ctx, step, ring, B):
    call("swb_decode_advance", next_tok.data_ptr(), cur_tok.data_ptr(), ctx.data_ptr(),
         step.data_ptr(), ring.data_ptr(), ring.shape[1], B, _stream())


def slots_from_table(table_row_ptr, start, n, block_size, slots, stream=None):
    call("swb_slots_from_table", table_row_ptr, start, n, block_size, slots.data_ptr(),
         stream if stream is not None else _stream())


def kv_handoff(first_tok, seqs, epochs, table_dev_ptr, stride_bytes, rows=None, group_key=0,
               stream=None):
    """Publish a finished prompt batch to a token machine's hand-off table:
    per request its first token (first_tok[rows[i]]), the group key and
    size, then its flag = epoch — after all prior work on the stream (the
    KV pushes)."""
    _req(first_tok, torch.int32, "first_tok")
    n = len(seqs)
    if n == 0:
        return
    rows = list(range(n)) if rows is None else list(rows)
    if n != len(epochs) or n != len(rows) or max(rows) >= first_tok.numel():
        raise ValidationError("kv_handoff: seqs / epochs / rows / first_tok lengths differ")
    r = (ctypes.c_int32 * n)(*rows)
    s = (ctypes.c_int32 * n)(*seqs)
    e = (ctypes.c_uint32 * n)(*epochs)
    call("swb_kv_handoff", first_tok.data_ptr(), n, r, s, e, int(group_key), table_dev_ptr,
         stride_bytes, stream if stream is not None else _stream())
