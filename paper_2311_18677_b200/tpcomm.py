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


class TPStage:
    """Prefill partial exchange over the copy engines (libswb200's
    ``swb_tp_stage_*``): ``send(buf, chunk, part, row0, epoch)`` DMA-copies
    this rank's bf16 rows into every peer's receive buffer ``buf`` (on the
    caller's side stream) and raises the peers' flag ``(buf, chunk)`` to
    ``epoch``; ``wait(buf, chunk, epoch)`` makes the current stream wait for
    every peer's flag; ``parts(buf, own, row0, rows)`` lists the rank-ordered
    partials of those rows (own rows + received views) for the norm that
    adds them (kernels.rmsnorm / layernorm with a list addend)."""

    def __init__(self, group, rows: int, d: int, n_bufs: int = 2):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.rows, self.d, self.n_bufs = int(rows), int(d), int(n_bufs)
        per_src = (self.rows * self.d * 2 + 255) // 256 * 256
        h = C.c_void_p()
        blob = C.create_string_buffer(_abi.TP_STAGE_IPC_BYTES)
        _abi.call("swb_tp_stage_create", self.rank, self.world, per_src, self.n_bufs,
                  C.byref(h), blob, _abi.TP_STAGE_IPC_BYTES)
        self._h = h
        blobs = [None] * self.world
        dist.all_gather_object(blobs, bytes(blob.raw), group=group)
        allb = C.create_string_buffer(b"".join(blobs), _abi.TP_STAGE_IPC_BYTES * self.world)
        _abi.call("swb_tp_stage_connect", self._h, allb, _abi.TP_STAGE_IPC_BYTES)
        self._rx = [[device_view(int(_abi.lib.swb_tp_stage_rx(self._h, b, p)),
                                 (self.rows, self.d), torch.bfloat16)
                     for p in range(self.world)] for b in range(self.n_bufs)]

    MAXCH = _abi.TP_STAGE_MAXCH

    def send(self, buf: int, chunk: int, part: torch.Tensor, row0: int, epoch: int,
             stream: torch.cuda.Stream) -> None:
        if part.dtype != torch.bfloat16 or not part.is_contiguous() or part.shape[1] != self.d:
            raise ValueError("TPStage.send: contiguous bf16 rows of width d")
        if row0 + part.shape[0] > self.rows:
            raise ValueError(f"TPStage.send: rows {row0}+{part.shape[0]} exceed {self.rows}")
        _abi.call("swb_tp_stage_send", self._h, buf, chunk, part.data_ptr(),
                  row0 * self.d * 2, part.numel() * 2, epoch & 0xFFFFFFFF, stream.cuda_stream)

    def wait(self, buf: int, chunk: int, epoch: int) -> None:
        _abi.call("swb_tp_stage_wait", self._h, buf, chunk, epoch & 0xFFFFFFFF,
                  torch.cuda.current_stream().cuda_stream)

    def parts(self, buf: int, own: torch.Tensor, row0: int, rows: int) -> list:
        out = []
        for p in range(self.world):
            if p == self.rank:
                out.append(own[row0:row0 + rows])
            else:
                out.append(self._rx[buf][p][row0:row0 + rows])
        return out

    def close(self) -> None:
        if self._h:
            _abi.call("swb_tp_stage_destroy", self._h)
            self._h = None
