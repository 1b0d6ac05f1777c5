"""ctypes binding of libswb200.so — the thin layer between the Python host
(workers / KV-cache manager / scheduler) and the sm_100a kernels.

No logic lives here: every entry point of include/swb200.h is declared with
its C signature and wrapped so a non-zero status raises the exception type
the reference would raise (errors.py:4-31).  There is deliberately no
fallback: if the library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import CapacityError, ConfigurationError, NativeError, ValidationError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libswb200.so")

SWB_OK, SWB_ERR_INVALID, SWB_ERR_CAPACITY, SWB_ERR_CUDA, SWB_ERR_CONFIG = 0, 1, 2, 3, 4
EPI_BF16, EPI_F32, EPI_RESID_F32, EPI_SWIGLU, EPI_GELU = 0, 1, 2, 3, 4
KV_POOL_IPC_BYTES = 256
TP_IPC_BYTES = 128
TP_STAGE_IPC_BYTES = 128   # SWB_TP_STAGE_IPC_BYTES
TP_STAGE_MAXCH = 8         # SWB_TP_STAGE_MAXCH

_P = C.c_void_p
_I = C.c_int
_F = C.c_float
_U = C.c_uint32
_S = C.c_size_t
_ST = C.c_size_t  # uintptr_t stream


class KVPoolInfo(C.Structure):
    _fields_ = [
        ("k_base", _P), ("v_base", _P), ("layer_stride_bytes", _S), ("block_bytes", _S),
        ("block_tables", _P), ("bitmap", _P),
        ("num_layers", _I), ("num_blocks", _I), ("Hkv", _I), ("block_size", _I), ("dh", _I),
        ("max_seqs", _I), ("max_blocks_per_seq", _I), ("free_blocks", _I),
        ("is_peer_view", _I),
    ]


# name -> argtypes (all return int status unless listed in _RESTYPE)
SIGNATURES = {
    "swb_abi_version": [],
    "swb_last_error": [],
    "swb_sync_stream": [_ST],
    "swb_gemm_bf16": [_P, _P, _P, _P, _I, _I, _I, _I, _ST],
    "swb_gemv_bf16": [_P, _P, _P, _P, _I, _I, _I, _I, _ST],
    "swb_gemm_bf16_bias": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _ST],
    "swb_gemv_bf16_bias": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _ST],
    "swb_gemm_qkv_rope": [_P, _P, _P, _P, _I, _I, _I, _P, _F, _P, _I, _I, _I, _P, _P, _P, _I,
                          _ST],
    "swb_rope_table": [_F, _I, _P, _ST],
    "swb_gemv_rmsnorm_bf16": [_P, _P, _F, _P, _P, _P, _I, _I, _I, _I, _ST],
    "swb_embed": [_P, _P, _P, _I, _I, _ST],
    "swb_rmsnorm": [_P, _P, _P, _P, _I, _I, _F, _ST],
    "swb_layernorm": [_P, _P, _P, _P, _P, _I, _I, _F, _I, _ST],
    "swb_add_rmsnorm": [_P, _P, _P, _P, _P, _I, _I, _F, _ST],
    "swb_add_layernorm": [_P, _P, _P, _P, _P, _P, _I, _I, _F, _ST],
    "swb_argmax": [_P, _I, _I, _P, _ST],
    "swb_argmax_shard": [_P, _I, _I, _I, _I, _I, _P, _ST],
    "swb_argmax_pick": [_P, _I, _I, _P, _ST],
    "swb_rope_kv_write": [_P, _I, _I, _P, _I, _I, _I, _F, _P, _P, _P, _I, _ST],
    "swb_kv_push_layer": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _I, _ST],
    "swb_kv_push_layers": [_P, _S, _I, _I, _I, _I, _I, _I, _I, _P, _P, _S, _P, _I, _I, _ST],
    "swb_kv_handoff": [_P, _I, _P, _P, _P, _I, _P, _I, _ST],
    "swb_host_register": [_P, _S, C.POINTER(_P)],
    "swb_host_unregister": [_P],
    "swb_attn_prefill": [_P, _I, _P, _I, _I, _I, _I, _I, _F, _P, _ST],
    "swb_attn_prefill_tc": [_P, _I, _I, _P, _I, _I, _I, _I, _I, _F, _P, _P, _ST],
    "swb_attn_decode_workspace": [_I, _I, _I, _I, _I],
    "swb_attn_chunk_workspace": [_I, _I, _I],
    "swb_attn_chunk": [_P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _I, _F, _P, _I, _P, _P, _ST],
    "swb_attn_decode": [_P, _I, _P, _P, _P, _I, _P, _P, _P, _F, _P, _I, _I, _I, _I, _I, _F,
                        _I, _I, _P, _P, _ST],
    "swb_attn_decode_step": [_P, _I, _P, _P, _P, _I, _P, _F, _P, _I, _I, _I, _I, _I, _F, _I,
                             _I, _P, _P, _ST],
    "swb_decode_advance": [_P, _P, _P, _P, _P, _I, _I, _ST],
    "swb_slots_from_table": [_P, _I, _I, _I, _P, _ST],
    "swb_kv_pool_create": [_I, _I, _I, _I, _I, _I, _I, C.POINTER(_P)],
    "swb_kv_pool_destroy": [_P],
    "swb_kv_pool_get_info": [_P, C.POINTER(KVPoolInfo)],
    "swb_block_alloc": [_P, _I, _I, _ST],
    "swb_block_free": [_P, _I, _I, _ST],
    "swb_kv_pool_ipc_export": [_P, _P, _S],
    "swb_kv_pool_ipc_open": [_P, _S, C.POINTER(_P)],
    "swb_enable_peer": [_I],
    "swb_tp_comm_create": [_I, _I, _S, C.POINTER(_P), _P, _S],
    "swb_tp_comm_connect": [_P, _P, _S],
    "swb_tp_comm_destroy": [_P],
    "swb_tp_comm_slot": [_P, _I],
    "swb_tp_allreduce_f32": [_P, _I, _P, _S, _ST],
    "swb_tp_allreduce_recv_f32": [_P, _I, _P, _S, _ST],
    "swb_gemv_bf16_tp": [_P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _ST],
    "swb_add_parts_rmsnorm": [_P, _P, _I, _P, _P, _P, _I, _I, _F, _ST],
    "swb_add_parts_layernorm": [_P, _P, _I, _P, _P, _P, _P, _I, _I, _F, _ST],
    "swb_tp_stage_create": [_I, _I, _S, _I, C.POINTER(_P), _P, _S],
    "swb_tp_stage_connect": [_P, _P, _S],
    "swb_tp_stage_destroy": [_P],
    "swb_tp_stage_rx": [_P, _I, _I],
    "swb_tp_stage_send": [_P, _I, _I, _P, _S, _S, C.c_uint32, _ST],
    "swb_tp_stage_wait": [_P, _I, _I, C.c_uint32, _ST],
}
_RESTYPE = {"swb_last_error": C.c_char_p, "swb_attn_decode_workspace": _S,
            "swb_attn_chunk_workspace": _S,
            "swb_tp_comm_slot": _P, "swb_tp_stage_rx": _P}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); "
            "the hot path has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    return lib


lib = _load()


def last_error() -> str:
    return lib.swb_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == SWB_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == SWB_ERR_INVALID:
        raise ValidationError(msg)
    if status == SWB_ERR_CAPACITY:
        raise CapacityError(msg)
    if status == SWB_ERR_CONFIG:
        raise ConfigurationError(msg)
    raise NativeError(msg)


# kernels launched per successful call (for the bench's gpu_launches claim)
LAUNCH_MULT = {
    "swb_gemm_bf16": 1, "swb_gemv_bf16": 1, "swb_gemm_bf16_bias": 1, "swb_gemv_bf16_bias": 1,
    "swb_gemm_qkv_rope": 1, "swb_rope_table": 1,
    "swb_layernorm": 1, "swb_add_rmsnorm": 1, "swb_add_layernorm": 1, "swb_gemv_rmsnorm_bf16": 1, "swb_embed": 1, "swb_rmsnorm": 1,
    "swb_argmax": 1, "swb_argmax_shard": 1, "swb_argmax_pick": 1, "swb_rope_kv_write": 1, "swb_kv_push_layer": 1, "swb_kv_push_layers": 1,
    "swb_kv_handoff": 1,
    "swb_attn_prefill": 1, "swb_attn_prefill_tc": 1, "swb_attn_decode": 1, "swb_attn_decode_step": 1, "swb_attn_chunk": 1,
    "swb_decode_advance": 1, "swb_slots_from_table": 1, "swb_block_alloc": 1,
    "swb_block_free": 1, "swb_tp_allreduce_f32": 1, "swb_tp_allreduce_recv_f32": 1,
    "swb_gemv_bf16_tp": 1, "swb_add_parts_rmsnorm": 1, "swb_add_parts_layernorm": 1,
}
_launches = [0]


def launch_count() -> int:
    return _launches[0]


def add_launches(n: int) -> None:
    _launches[0] += n


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)
    _launches[0] += LAUNCH_MULT.get(name, 0)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
