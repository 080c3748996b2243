"""ctypes binding of the C-ABI in include/devplace_b200.h.

The product path has no fallback: if the sm_100a library is missing or no CUDA
device is visible, every entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .build import LIB

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
F64 = ctypes.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "dp_last_error": (ctypes.c_char_p, []),
    "dp_launch_count": (I64, []),
    "dp_fp64_fma_probe": (I32, [I32, I32, I32, P, P]),
    "dp_graph_create": (I32, [I32, I32, P, P, P, P, P, P, P, P, P, P, P]),
    "dp_graph_destroy": (None, [P]),
    "dp_simulate_batch": (I32, [P, I32, P, I32, P, P, P, P, P, P, P, P]),
    "dp_policy_create": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, I32, P]),
    "dp_policy_destroy": (None, [P]),
    "dp_policy_num_params": (I64, [P]),
    "dp_policy_encode": (I32, [P, P, P]),
    "dp_policy_read_inputs": (I32, [P, P, P]),
    "dp_debug_phase_clocks": (I32, [I32, P]),
    "dp_debug_warp_clocks": (I32, [P]),
    "dp_debug_decoder_variant": (I32, [I32]),
    "dp_debug_encoder_variant": (I32, [I32]),
    "dp_debug_decoder_plan": (I32, [P, I32, P]),
    "dp_margin_accumulate": (I32, [I32, P, ctypes.c_double, P, P, P]),
    "dp_debug_policy_drop_stores": (I32, [P, I32]),
    "dp_debug_tensor_core": (I32, [I32]),
    "dp_group_features": (I32, [I32, I32, P, P, I32, P, P, I32, P, P, P, I32, I32, P, P, P, P, P, P, P, P]),
    "dp_debug_fastmath_error": (I32, [I64, P]),
    "dp_debug_att_clocks": (I32, [I32, P]),
    "dp_debug_sim_variant": (I32, [I32]),
    "dp_debug_lstm_clocks": (I32, [I32, P]),
    "dp_policy_decode": (I32, [P, P, I32, I64, P, U64, P, I64, P, P, P, P, P, P]),
    "dp_policy_backward": (I32, [P, P, I32, P, P, P]),
    "dp_policy_backward_rows": (I32, [P, P, I32, P]),
    "dp_policy_backward_grads": (I32, [P, P, I32, P, P, P]),
    "dp_reinforce_epilogue": (I32, [I32, I32, P, P, P, I32, F64, F64, I64, I64, I32, P, P, P, P, I64, I32, P]),
    "dp_adam_apply": (I32, [I64, P, P, P, P, P, I64, F64, F64, F64, F64, P, P, P, P, I64, P]),
    "dp_apply_measurement_noise": (I32, [I32, I64, I32, P, P, P, I64, I32, P, P]),
    "dp_exchange_record_bytes": (I64, [I32, I32]),
    "dp_exchange_pack": (I32, [I32, I32, P, P, P, P, P]),
    "dp_exchange_unpack": (I32, [I32, I32, I32, P, P, P, P, P]),
    "dp_comm_version": (I32, [P]),
    "dp_comm_unique_id": (I32, [P]),
    "dp_comm_init_rank": (I32, [I32, P, I32, P]),
    "dp_comm_init_all": (I32, [I32, P, P]),
    "dp_comm_destroy": (None, [P]),
    "dp_comm_group_start": (I32, []),
    "dp_comm_group_end": (I32, []),
    "dp_comm_all_gather": (I32, [P, P, P, I64, P]),
    "dp_comm_all_reduce_f64": (I32, [P, P, I64, I32, P]),
    "dp_enumerate_placements": (I32, [I32, I32, ctypes.c_uint64, I32, P, P]),
    "dp_argmin_feasible": (I32, [I32, P, P, I64, P, P, P]),
}

# struct dp_train_state (include/devplace_b200.h): 3 doubles then 9 int64
TRAIN_STATE_FIELDS = ("baseline", "baseline_prev", "best_r", "update", "adam_t", "version", "rejected",
                      "n_used", "n_feasible", "best_update", "best_k", "error")
TRAIN_STATE_WORDS = len(TRAIN_STATE_FIELDS)


class NativeUnavailable(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not torch.cuda.is_available():
            raise NativeUnavailable("devplace_b200 needs a CUDA device (sm_100a); none is visible")
        if not os.path.exists(LIB):
            raise NativeUnavailable(f"CUDA library not built: {LIB} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def load_only():
    """Load the library and bind every declared symbol without touching CUDA
    (used by CPU tests to check the exported ABI)."""
    L = ctypes.CDLL(LIB)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def check(rc: int, what: str):
    if rc == 0:
        return
    msg = lib().dp_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
