"""ctypes binding of libpsg.so (include/psg.h).

The library is built in-tree (``paper_1511_06051_b200/libpsg.so``).  There is no CPU
fallback: if the library is missing or a CUDA call fails, the error surfaces as an
exception mapped from the C status code, exactly like the reference's exception types
(SURVEY §8(b)):  PSG_EINVAL -> ValueError (std::invalid_argument),
PSG_ERUNTIME -> RuntimeError (std::runtime_error), PSG_ECUDA -> CudaError,
PSG_ELOGIC -> LogicError (std::logic_error).
"""
from __future__ import annotations

import ctypes
import os
import threading

from .netspec import CLayerDesc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpsg.so")

OK, EINVAL, ERUNTIME, ECUDA, ELOGIC = range(5)
PRECISION_FP32, PRECISION_TF32 = 0, 1
AVERAGE_FAST, AVERAGE_ORDERED = 0, 1
TC_PAIR = {"auto": 0, "never": 1, "always": 2}


class CudaError(RuntimeError):
    """CUDA / NCCL failure (PSG_ECUDA)."""


class LogicError(RuntimeError):
    """std::logic_error (PSG_ELOGIC)."""


_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U64 = ctypes.POINTER(ctypes.c_uint64)
_I64 = ctypes.POINTER(ctypes.c_int64)
_VP = ctypes.c_void_p
_SZ = ctypes.c_size_t
_PP = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); every symbol declared in include/psg.h
SIGNATURES = {
    "psg_layer_desc_init": (None, [ctypes.POINTER(CLayerDesc), ctypes.c_int, ctypes.c_char_p]),
    "psg_last_error": (ctypes.c_char_p, []),
    "psg_abi_version": (ctypes.c_int, []),
    "psg_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "psg_splitmix64": (ctypes.c_uint64, [ctypes.c_uint64]),
    "psg_derive_seed": (ctypes.c_uint64, [ctypes.c_uint64, _U64, ctypes.c_int]),
    "psg_shard": (ctypes.c_int, [_SZ, ctypes.c_int, ctypes.c_uint64, _U64, _U64]),
    "psg_worker_stream_seed": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_int]),
    "psg_epoch_order": (ctypes.c_int, [_U64, _SZ, ctypes.c_uint64, ctypes.c_uint64, _U64]),
    "psg_generate_synthetic": (ctypes.c_int, [ctypes.c_int, _SZ, _SZ, _SZ, _SZ, ctypes.c_double,
                                              ctypes.c_uint64, ctypes.c_uint64, _D, _I32]),
    "psg_ctx_create": (ctypes.c_int, [ctypes.c_int, _PP]),
    "psg_ctx_destroy": (ctypes.c_int, [_VP]),
    "psg_ctx_sync": (ctypes.c_int, [_VP]),
    "psg_dataset_upload_f64": (ctypes.c_int, [_VP, _D, _I32, _SZ, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, _PP]),
    "psg_dataset_upload_f32": (ctypes.c_int, [_VP, _F, _I32, _SZ, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, _PP]),
    "psg_dataset_synthetic_device": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int,
                                                    ctypes.c_int, ctypes.c_int, _SZ,
                                                    ctypes.c_double, ctypes.c_uint64,
                                                    ctypes.c_uint64, _PP]),
    "psg_dataset_read_f32": (ctypes.c_int, [_VP, _SZ, _SZ, _F, _I32]),
    "psg_read_idx": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(_SZ),
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int), _F, _I32]),
    "psg_read_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.POINTER(_SZ), _F, _I32]),
    "psg_dataset_load_idx": (ctypes.c_int, [_VP, ctypes.c_char_p, ctypes.c_char_p, _PP]),
    "psg_dataset_load_csv": (ctypes.c_int, [_VP, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, _PP]),
    "psg_dataset_synthetic": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, _SZ, ctypes.c_double, ctypes.c_uint64,
                                             ctypes.c_uint64, _PP]),
    "psg_dataset_size": (ctypes.c_int, [_VP, ctypes.POINTER(_SZ)]),
    "psg_dataset_destroy": (ctypes.c_int, [_VP]),
    "psg_net_create": (ctypes.c_int, [_VP, ctypes.POINTER(CLayerDesc), ctypes.c_int,
                                      ctypes.c_uint64, _PP]),
    "psg_net_destroy": (ctypes.c_int, [_VP]),
    "psg_net_num_classes": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int)]),
    "psg_net_param_count": (ctypes.c_int, [_VP, ctypes.POINTER(_SZ)]),
    "psg_net_num_tensors": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int)]),
    "psg_net_tensor_info": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int), _I64,
                                           ctypes.POINTER(_SZ)]),
    "psg_net_set_precision": (ctypes.c_int, [_VP, ctypes.c_int]),
    "psg_net_set_sgd": (ctypes.c_int, [_VP, ctypes.c_double, ctypes.c_double, ctypes.c_double]),
    "psg_net_get_weights_f64": (ctypes.c_int, [_VP, _D, _SZ]),
    "psg_net_set_weights_f64": (ctypes.c_int, [_VP, _D, _SZ]),
    "psg_net_get_velocity_f64": (ctypes.c_int, [_VP, _D, _SZ]),
    "psg_net_reset_velocity": (ctypes.c_int, [_VP]),
    "psg_net_forward": (ctypes.c_int, [_VP, _D, _I32, _SZ, _D, _D]),
    "psg_net_backward": (ctypes.c_int, [_VP, _D, _I32, _SZ, _D, _D]),
    "psg_net_apply_update": (ctypes.c_int, [_VP, _D, _SZ]),
    "psg_net_layer_shape": (ctypes.c_int, [_VP, ctypes.c_int, _I64]),
    "psg_net_layer_output": (ctypes.c_int, [_VP, ctypes.c_int, _D, _SZ]),
    "psg_net_layer_grad": (ctypes.c_int, [_VP, ctypes.c_int, _D, _SZ]),
    "psg_net_attach_shard": (ctypes.c_int, [_VP, _VP, _U64, _SZ, _SZ, ctypes.c_uint64]),
    "psg_net_get_stream_position": (ctypes.c_int, [_VP, _U64, _U64]),
    "psg_net_set_stream_position": (ctypes.c_int, [_VP, ctypes.c_uint64, ctypes.c_uint64]),
    "psg_net_train": (ctypes.c_int, [_VP, ctypes.c_long]),
    "psg_net_sync": (ctypes.c_int, [_VP]),
    "psg_net_last_train_ms": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_float)]),
    "psg_net_last_loss": (ctypes.c_int, [_VP, _D]),
    "psg_net_attach_validation": (ctypes.c_int, [_VP, _VP, _SZ]),
    "psg_net_test": (ctypes.c_int, [_VP, ctypes.c_long, _D]),
    "psg_net_test_begin": (ctypes.c_int, [_VP, ctypes.c_long, ctypes.c_long, ctypes.c_long]),
    "psg_net_test_end": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_ulonglong),
                                        ctypes.POINTER(ctypes.c_ulonglong)]),
    "psg_net_attach_shard_part": (ctypes.c_int, [_VP, _VP, _U64, _SZ, _SZ, ctypes.c_uint64,
                                                 ctypes.c_int, ctypes.c_int]),
    "psg_net_grad_step": (ctypes.c_int, [_VP]),
    "psg_net_set_tc_options": (ctypes.c_int, [_VP, ctypes.c_int]),
    "psg_debug_guard_violations": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_char_p, _SZ]),
    "psg_debug_tc_prof": (ctypes.c_int, [ctypes.c_char_p, _SZ, ctypes.c_int]),
    "psg_net_train_round": (ctypes.c_int, [_VP, ctypes.c_long, _VP]),
    "psg_net_train_host_rows": (ctypes.c_int, [_VP, _F, _I32, _SZ, _U64, ctypes.c_long, _D, ctypes.c_int]),
    "psg_net_set_fusion": (ctypes.c_int, [_VP, ctypes.c_int]),
    "psg_net_apply_grads": (ctypes.c_int, [_VP]),
    "psg_average_grads_local": (ctypes.c_int, [_PP, ctypes.c_int]),
    "psg_comm_average_grads": (ctypes.c_int, [_PP, _PP, ctypes.c_int, ctypes.c_int]),
    "psg_net_kernels_per_step": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int)]),
    "psg_net_profile_step": (ctypes.c_int, [_VP, ctypes.c_int, _VP, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_int)]),
    "psg_net_train_host": (ctypes.c_int, [_VP, _F, _I32, ctypes.c_long, _D]),
    "psg_host_alloc": (ctypes.c_int, [_SZ, _PP]),
    "psg_host_free": (ctypes.c_int, [_VP]),
    "psg_net_event_record": (ctypes.c_int, [_VP, ctypes.c_int]),
    "psg_net_event_elapsed": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_float)]),
    "psg_average_local": (ctypes.c_int, [_PP, ctypes.c_int]),
    "psg_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "psg_comm_create": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _PP]),
    "psg_comm_create_all": (ctypes.c_int, [_PP, ctypes.c_int, _PP]),
    "psg_comm_destroy": (ctypes.c_int, [_VP]),
    "psg_comm_average": (ctypes.c_int, [_PP, _PP, ctypes.c_int, ctypes.c_int]),
    "psg_comm_broadcast": (ctypes.c_int, [_PP, _PP, ctypes.c_int, ctypes.c_int]),
    "psg_buffer_create": (ctypes.c_int, [_VP, _SZ, _PP]),
    "psg_buffer_fill_uniform": (ctypes.c_int, [_VP, ctypes.c_uint64, ctypes.c_double,
                                               ctypes.c_double]),
    "psg_buffer_read": (ctypes.c_int, [_VP, _F, _SZ]),
    "psg_buffer_write": (ctypes.c_int, [_VP, _F, _SZ]),
    "psg_buffer_destroy": (ctypes.c_int, [_VP]),
    "psg_buffer_average_local": (ctypes.c_int, [_PP, ctypes.c_int]),
    "psg_comm_average_buffer": (ctypes.c_int, [_PP, _PP, ctypes.c_int, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_float)]),
}

class OpTime(ctypes.Structure):
    """psg_op_time (include/psg.h)."""
    _fields_ = [("name", ctypes.c_char * 64), ("layer", ctypes.c_int), ("phase", ctypes.c_int),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double), ("ms", ctypes.c_float),
                ("launches", ctypes.c_int)]


PHASES = ["gather", "forward", "loss", "wgrad", "dgrad", "backward", "update"]


class PinnedArray:
    """numpy view over page-locked host memory (psg_host_alloc)."""

    def __init__(self, shape, dtype):
        import numpy as np
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * self.dtype.itemsize
        p = ctypes.c_void_p()
        call("psg_host_alloc", nbytes, ctypes.byref(p))
        self._ptr = p
        buf = (ctypes.c_char * nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype).reshape(shape)

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p:
            try:
                lib().psg_host_free(p)
            except Exception:
                pass
            self._ptr = None


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libpsg.so (once).  Raises loudly when the native library is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libpsg.so not found at {LIB_PATH}: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().psg_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ECUDA:
        raise CudaError(msg)
    if rc == ELOGIC:
        raise LogicError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
