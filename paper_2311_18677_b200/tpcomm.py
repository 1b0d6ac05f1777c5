"""Tensor-parallel all-reduce over NVLink peer memory (libswb200's
``swb_tp_comm_*`` / ``swb_tp_allreduce_f32``).

One ``TPComm`` per TP rank.  The producing GEMM/GEMV writes its fp32 partial
sums into ``slot(s)`` (a view of IPC-shared device memory), then
``allreduce(s, out)`` writes the rank-ordered sum of every rank's slot ``s``
into ``out``.  Slots 0 and 1 must strictly alternate between consecutive
reductions (``next_slot``); ``reset()`` at the start of every prefill / decode
step keeps the sequence graph-replayable, so every step must perform an even
number of them (``assert_even``).  Slot 2 (``AUX``, <= 1 MB) carries the one
reduction per step outside that alternation: the vocab-parallel greedy
candidates.
Replaces the NCCL ``all_reduce`` of ``ModelRunner._allreduce``
("all-reduce twice per layer").
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _abi
from .kvcache import device_view


class TPComm:
    def __init__(self, group, slot_bytes: int):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.slot_bytes = (int(slot_bytes) + 255) // 256 * 256
        h = C.c_void_p()
        blob = C.create_string_buffer(_abi.TP_IPC_BYTES)
        _abi.call("swb_tp_comm_create", self.rank, self.world, self.slot_bytes, C.byref(h),
                  blob, _abi.TP_IPC_BYTES)
        self._h = h
        blobs = [None] * self.world
        dist.all_gather_object(blobs, bytes(blob.raw), group=group)
        allb = C.create_string_buffer(b"".join(blobs), _abi.TP_IPC_BYTES * self.world)
        _abi.call("swb_tp_comm_connect", self._h, allb, _abi.TP_IPC_BYTES)
        self._slots = [int(_abi.lib.swb_tp_comm_slot(self._h, s)) for s in (0, 1, 2)]
        self._next = 0

    AUX = 2
    AUX_BYTES = 1 << 20
    LL_OUTPUTS = 16384      # fused projection push: outputs per source (TP_LL_BYTES / 8)

    def assert_even(self) -> None:
        """A step must end on the slot it started with (even count of 0/1
        reductions), or the next replay would reuse a slot back to back."""
        if self._next != 0:
            raise RuntimeError("odd number of slot-0/1 all-reduces in one step")

    def reset(self) -> None:
        self._next = 0

    def next_slot(self) -> int:
        s = self._next
        self._next ^= 1
        return s

    def slot(self, s: int, shape) -> torch.Tensor:
        n = 1
        for v in shape:
            n *= int(v)
        if 4 * n > (self.slot_bytes if s < 2 else min(self.slot_bytes, self.AUX_BYTES)):
            raise ValueError(f"TP slot of {self.slot_bytes} bytes cannot hold {tuple(shape)} fp32")
        return device_view(self._slots[s], tuple(shape), torch.float32)

    def allreduce(self, s: int, out: torch.Tensor) -> None:
        _abi.call("swb_tp_allreduce_f32", self._h, s, out.data_ptr(), out.numel(),
                  torch.cuda.current_stream().cuda_stream)

    def allreduce_recv(self, s: int, out: torch.Tensor) -> None:
        """Second half of the fused form: the peers' projection GEMVs
        (kernels.gemv_tp on slot s) already pushed their partials."""
        _abi.call("swb_tp_allreduce_recv_f32", self._h, s, out.data_ptr(), out.numel(),
                  torch.cuda.current_stream().cuda_stream)

    def close(self) -> None:
        if self._h:
            _abi.call("swb_tp_comm_destroy", self._h)
            self._h = None
