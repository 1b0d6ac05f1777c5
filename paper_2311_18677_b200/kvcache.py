"""KV-cache manager: the host handle on a device-resident paged KV pool.

Reference semantics (what this replaces):
  * KV is a byte count, ``tokens * kv_bytes_per_token`` (perf.py:134-137);
  * a machine's memory = weights + KV of every resident context
    (perf.py:139-141, machine.py:118-123);
  * admission reserves a token task's *final* context
    (``_resident_projected``, machine.py:107-110, :216-223) and checks it
    against capacity (``_memory_fits``, machine.py:125-128).

Here the KV bytes are real: libswb200 owns per-layer K/V block arrays
``[num_blocks][Hkv][block_size][dh]`` (bf16) plus int32 block tables, and a
device kernel hands out the lowest free block ids.  The host mirrors only the
free-block count, so admission stays a pure host decision exactly like the
reference's, and a reservation is ``ceil((prompt + outputs) / block_size)``
blocks written into the sequence's table row.
"""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _abi
from .errors import CapacityError, ValidationError


class _CudaView:
    """Zero-copy torch view of device memory owned by libswb200."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None,
        }


def device_view(ptr: int, shape, dtype: torch.dtype) -> torch.Tensor:
    typestr = {torch.int32: "<i4", torch.uint32: "<u4", torch.bfloat16: "<V2",
               torch.float32: "<f4", torch.uint8: "|u1"}[dtype]
    if dtype == torch.bfloat16:
        t = torch.as_tensor(_CudaView(ptr, shape, "<i2"), device="cuda")
        return t.view(torch.bfloat16)
    if dtype == torch.uint32:
        return torch.as_tensor(_CudaView(ptr, shape, "<i4"), device="cuda")
    return torch.as_tensor(_CudaView(ptr, shape, typestr), device="cuda")


def blocks_for(tokens: int, block_size: int) -> int:
    return (tokens + block_size - 1) // block_size


class KVCacheManager:
    """Device block pool + block tables of one machine (one TP rank)."""

    def __init__(self, num_layers: int, num_blocks: int, n_kv_heads: int, head_dim: int,
                 block_size: int = 16, max_seqs: int = 256, max_blocks_per_seq: int = 1024):
        if min(num_layers, num_blocks, n_kv_heads, head_dim, block_size, max_seqs,
               max_blocks_per_seq) <= 0:
            raise ValidationError("KV pool sizes must be positive")
        h = C.c_void_p()
        _abi.call("swb_kv_pool_create", num_layers, num_blocks, n_kv_heads, block_size,
                  head_dim, max_seqs, max_blocks_per_seq, C.byref(h))
        self._h = h
        self._owned = True
        self._refresh()
        self._free_slots = list(range(max_seqs))
        self.seq_blocks: dict[int, int] = {}

    @classmethod
    def open_peer(cls, handle: bytes) -> "KVCacheManager":
        """Non-owning view of a peer process's pool (prompt side pushes into
        it and reads its block tables)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        buf = C.create_string_buffer(handle, len(handle))
        _abi.call("swb_kv_pool_ipc_open", buf, len(handle), C.byref(h))
        self._h = h
        self._owned = False
        self._refresh()
        self._free_slots = []
        self.seq_blocks = {}
        return self

    def _refresh(self):
        info = _abi.KVPoolInfo()
        _abi.call("swb_kv_pool_get_info", self._h, C.byref(info))
        self.info = info
        self.num_layers = info.num_layers
        self.num_blocks = info.num_blocks
        self.block_size = info.block_size
        self.n_kv_heads = info.Hkv
        self.head_dim = info.dh
        self.max_seqs = info.max_seqs
        self.max_blocks_per_seq = info.max_blocks_per_seq

    # -- geometry ----------------------------------------------------------
    @property
    def block_bytes(self) -> int:
        return int(self.info.block_bytes)

    def k_layer_ptr(self, layer: int) -> int:
        return self.info.k_base + layer * self.info.layer_stride_bytes

    def v_layer_ptr(self, layer: int) -> int:
        return self.info.v_base + layer * self.info.layer_stride_bytes

    def table_row_ptr(self, seq: int) -> int:
        return self.info.block_tables + seq * self.max_blocks_per_seq * 4

    def tables(self) -> torch.Tensor:
        """Zero-copy int32 view [max_seqs, max_blocks_per_seq] (owned pools)."""
        return device_view(self.info.block_tables, (self.max_seqs, self.max_blocks_per_seq),
                           torch.int32)

    def k_view(self, layer: int) -> torch.Tensor:
        return device_view(self.k_layer_ptr(layer),
                           (self.num_blocks, self.n_kv_heads, self.block_size, self.head_dim),
                           torch.bfloat16)

    def v_view(self, layer: int) -> torch.Tensor:
        return device_view(self.v_layer_ptr(layer),
                           (self.num_blocks, self.n_kv_heads, self.block_size, self.head_dim),
                           torch.bfloat16)

    # -- accounting (host mirror) -------------------------------------------
    @property
    def free_blocks(self) -> int:
        self._refresh()
        return int(self.info.free_blocks)

    def fits(self, tokens: int) -> bool:
        """Admission test in blocks (Machine._memory_fits, machine.py:125-128)."""
        return blocks_for(tokens, self.block_size) <= self.free_blocks

    # -- allocation -----------------------------------------------------------
    def allocate(self, tokens: int, stream: int | None = None) -> int:
        """Reserve blocks for ``tokens`` (prompt + all outputs) and return the
        sequence slot whose table row the device allocator filled."""
        if not self._owned:
            raise ValidationError("peer views cannot allocate")
        n = blocks_for(tokens, self.block_size)
        if n > self.max_blocks_per_seq:
            raise CapacityError(f"{tokens} tokens need {n} blocks > {self.max_blocks_per_seq}")
        if not self._free_slots:
            raise CapacityError("no free sequence slot")
        seq = self._free_slots.pop(0)
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        try:
            _abi.call("swb_block_alloc", self._h, seq, n, s)
        except CapacityError:
            self._free_slots.insert(0, seq)
            raise
        self.seq_blocks[seq] = n
        return seq

    def release(self, seq: int, stream: int | None = None) -> None:
        n = self.seq_blocks.pop(seq)
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        _abi.call("swb_block_free", self._h, seq, n, s)
        self._free_slots.append(seq)
        self._free_slots.sort()

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(_abi.KV_POOL_IPC_BYTES)
        _abi.call("swb_kv_pool_ipc_export", self._h, buf, _abi.KV_POOL_IPC_BYTES)
        return buf.raw

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _abi.call("swb_kv_pool_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kv_bytes(tokens: int, num_layers: int, n_kv_heads: int, head_dim: int) -> int:
    """K+V bytes of ``tokens`` tokens (bf16) — the reference's
    kv_cache_bytes (perf.py:134-137) with a GQA-aware bytes/token."""
    return tokens * 2 * num_layers * n_kv_heads * head_dim * 2


__all__ = ["KVCacheManager", "device_view", "blocks_for", "kv_bytes"]
_ = math
