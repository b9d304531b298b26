"""ctypes binding of libmpcg.so (the C ABI declared in include/mpcg.h).

The shared library is built in-tree (paper_2209_13643_b200/lib/libmpcg.so) by
`__graft_entry__.build()` / `make -C paper_2209_13643_b200/csrc`. There is no CPU
fallback: importing the ops without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPCG_LIB selects another build of the same ABI (e.g. lib/libmpcg_nodealer.so, the online-only
# timing build of tools/dealer_split.py); there is no CPU fallback either way.
LIB_PATH = os.environ.get("MPCG_LIB") or os.path.join(_HERE, "lib", "libmpcg.so")


class Error(RuntimeError):
    """Base error (mpcpipe::Error, H/errors.hpp:8-45)."""


class RangeError(Error): pass
class ShapeError(Error): pass
class ConfigError(Error): pass
class ProtocolError(Error): pass
class TransportError(Error): pass
class BudgetError(Error): pass
class UsageError(Error): pass
class CudaError(Error): pass
class NcclError(Error): pass


_CODES = {1: RangeError, 2: ShapeError, 3: ConfigError, 4: ProtocolError, 5: TransportError,
          6: BudgetError, 7: UsageError, 8: CudaError, 9: NcclError, 10: Error}

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
U64 = C.c_uint64
U64P = C.POINTER(C.c_uint64)
I32 = C.c_int
STR = C.c_char_p
DBL = C.c_double

# name -> argtypes (all return int status unless listed in _RET)
SIGNATURES = {
    "mpcg_last_error": [],
    "mpcg_version": [],
    "mpcg_device_count": [C.POINTER(I32)],
    "mpcg_session_create": [I32, I32, I32, U64, U64, I32, PP],
    "mpcg_session_destroy": [P],
    "mpcg_session_set_pipeline": [P, I32, U64, I32],
    "mpcg_session_set_link": [P, DBL, DBL, DBL],
    "mpcg_session_set_shard": [P, U64, U64, U64],
    "mpcg_nccl_unique_id": [C.c_char_p],
    "mpcg_session_connect_nccl": [P, C.c_char_p, I32],
    "mpcg_session_connect_socket": [P, C.c_char_p, I32, DBL],
    "mpcg_session_connect_p2p": [P, P],
    "mpcg_triple_queue_create": [PP],
    "mpcg_triple_queue_destroy": [P],
    "mpcg_triple_queue_size": [P, U64P, U64P],
    "mpcg_triple_queue_rewind": [P],
    "mpcg_triple_queue_save": [P, STR],
    "mpcg_triple_queue_load": [P, STR],
    "mpcg_session_record_triples": [P, P],
    "mpcg_session_use_triple_queue": [P, P],
    "mpcg_dealer_fetch": [P, I32, I32, I32, I32, I32, U64P, I32, U64P, STR, PP, PP, PP],
    "mpcg_session_sync": [P],
    "mpcg_session_set_persistent": [P, I32],
    "mpcg_session_stats": [P, I32, U64P],
    "mpcg_session_n_local": [P, C.POINTER(I32)],
    "mpcg_session_trace": [P, I32],
    "mpcg_session_trace_count": [P, U64P],
    "mpcg_session_trace_get": [P, U64, C.POINTER(C.c_uint32), C.POINTER(I32), U64P, C.POINTER(DBL), C.c_char_p, I32],
    "mpcg_session_clear_trace": [P],
    "mpcg_session_now": [P, C.POINTER(DBL)],
    "mpcg_session_add_delay": [P, DBL],
    "mpcg_tensor_create": [P, I32, U64P, I32, U64P, PP],
    "mpcg_tensor_download": [P, U64P],
    "mpcg_tensor_shape": [P, C.POINTER(I32), U64P, C.POINTER(I32)],
    "mpcg_tensor_destroy": [P],
    "mpcg_deal_input": [P, C.POINTER(DBL), I32, U64P, U64, U64, U64, PP],
    "mpcg_open": [P, P, I32, STR, PP],
    "mpcg_beaver_mul": [P, P, P, STR, I32, PP],
    "mpcg_beaver_square": [P, P, STR, I32, PP],
    "mpcg_beaver_and": [P, P, P, STR, I32, PP],
    "mpcg_beaver_matmul": [P, P, P, I32, STR, I32, PP],
    "mpcg_binary_add": [P, P, P, I32, I32, I32, STR, PP],
    "mpcg_a2b": [P, P, I32, STR, PP],
    "mpcg_msb": [P, P, I32, STR, PP],
    "mpcg_b2a_bit": [P, P, STR, I32, PP],
    "mpcg_less_than": [P, P, P, I32, STR, PP],
    "mpcg_truncate": [P, P, I32, PP],
    "mpcg_relu": [P, P, STR, PP],
    "mpcg_max_last_dim": [P, P, U64, STR, PP],
    "mpcg_exp": [P, P, STR, PP],
    "mpcg_reciprocal": [P, P, STR, PP],
    "mpcg_softmax": [P, P, U64, STR, PP],
    "mpcg_maxpool2d": [P, P, U64, U64, U64, U64, U64, U64, STR, PP],
    "mpcg_model_create": [STR, I32, I32, U64P, PP],
    "mpcg_model_add_layer": [P, STR, I32, U64, U64, U64, U64, U64, I32],
    "mpcg_model_add_layer_ex": [P, STR, I32, U64, U64, U64, U64, U64, I32, STR, STR],
    "mpcg_sigmoid": [P, P, STR, PP],
    "mpcg_gelu": [P, P, STR, PP],
    "mpcg_inv_sqrt": [P, P, STR, I32, PP],
    "mpcg_layernorm": [P, P, U64, P, P, I32, STR, PP],
    "mpcg_global_avg_pool": [P, P, U64, U64, U64, PP],
    "mpcg_model_destroy": [P],
    "mpcg_executor_create": [P, P, I32, I32, I32, U64, I32, PP],
    "mpcg_executor_deal_weights": [P, I32, C.POINTER(C.c_char_p), C.POINTER(C.POINTER(DBL)), C.POINTER(U64), U64],
    "mpcg_executor_release_graph": [P],
    "mpcg_executor_set_linear_chunks": [P, I32],
    "mpcg_set_pair_eval": [I32],
    "mpcg_executor_run": [P, P, PP],
    "mpcg_executor_capture": [P, P],
    "mpcg_executor_replay": [P, PP],
    "mpcg_executor_time_layers": [P, I32],
    "mpcg_executor_layer_times": [P, I32, C.POINTER(C.c_float), C.POINTER(I32)],
    "mpcg_executor_destroy": [P],
    "mpcg_set_gemm_mode": [I32],
    "mpcg_set_gemv": [I32],
    "mpcg_debug_tc2_trace": [U64P, I32],
    "mpcg_debug_tc3_trace": [U64P, I32],
    "mpcg_debug_draw_peak": [I32, C.POINTER(C.c_double)],
    "mpcg_session_connect_loopback": [P, P],
    "mpcg_launch_count": [],
    "mpcg_probe_start": [I32],
    "mpcg_probe_stop": [C.POINTER(DBL), U64P, C.POINTER(DBL)],
    "mpcg_pinned_alloc": [U64, PP],
    "mpcg_pinned_free": [P],
    "mpcg_tensor_copy_from_host": [P, U64P],
    "mpcg_session_flush_l2": [P],
    "mpcg_session_timer": [P, I32, C.POINTER(DBL)],
    "mpcg_fnv1a_words": [U64P, U64],
}
_RET = {"mpcg_last_error": C.c_char_p, "mpcg_fnv1a_words": U64, "mpcg_launch_count": U64}

_lib = None


def lib():
    """Load libmpcg.so once; raise if it was not built (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libmpcg.so not built at {LIB_PATH}; run __graft_entry__.build()")
        l = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = _RET.get(name, I32)
        _lib = l
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().mpcg_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))
