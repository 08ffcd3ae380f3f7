"""ctypes binding of libpartime_b200.so (the C ABI in include/partime_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a). No
CPU fallback exists: if the shared object is missing, loading raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PT_LIBNAME selects a build variant (libpartime_b200_jitter.so: the PT_JITTER race detector)
LIB_PATH = os.path.join(_HERE, os.environ.get("PT_LIBNAME", "libpartime_b200.so"))

PT_OK = 0
PT_EINVAL = -1
PT_EUNSUPPORTED = -2
PT_ECUDA = -3
PT_EBUSY = -4
PT_ENONFINITE = -5
PT_ETIMEOUT = -6
PT_ESTATE = -7

PT_HOST = 0
PT_DEVICE = 1

PT_ACT = {"none": 0, "relu": 1, "tanh": 2}
PT_LOSS = {"mse": 0, "softmax_ce": 1}
PT_OPT = {"sgd": 0, "adam": 1}

# every symbol include/partime_b200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "pt_create", "pt_set_params", "pt_get_params", "pt_step", "pt_run", "pt_sync",
    "pt_set_stream", "pt_get_stream", "pt_last_kernel_ms", "pt_tick", "pt_set_trace", "pt_get_trace",
    "pt_ipc_export", "pt_ipc_import", "pt_kernel_path", "pt_stage_device",
    "pt_destroy", "pt_last_error", "pt_abi_version",
)


class PTConfig(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int32),
        ("dims", ctypes.POINTER(ctypes.c_int32)),
        ("act", ctypes.POINTER(ctypes.c_int32)),
        ("loss", ctypes.c_int32),
        ("optimizer", ctypes.c_int32),
        ("lr", ctypes.c_float),
        ("n_stages", ctypes.c_int32),
        ("stage_first_layer", ctypes.POINTER(ctypes.c_int32)),
        ("batch", ctypes.c_int32),
        ("learn", ctypes.c_int32),
        ("act_delay", ctypes.c_int32),
        ("local_stage_first", ctypes.c_int32),
        ("local_stage_count", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("timeout_ms", ctypes.c_int32),
        ("device_of_stage", ctypes.POINTER(ctypes.c_int32)),
    ]


class PipelineError(RuntimeError):
    """Error raised by the B200 engine; `.code` is the PT_E* value."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ContractViolation(PipelineError):
    """Concurrent use of one pipeline."""


class NonFiniteLoss(PipelineError, FloatingPointError):
    """Non-finite loss; the message names the first bad step."""


_lib = None


def load():
    """Load the shared library (once). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 engine has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    f32p = ctypes.POINTER(ctypes.c_float)
    lib.pt_create.argtypes = [ctypes.POINTER(PTConfig), ctypes.POINTER(P)]
    lib.pt_create.restype = ctypes.c_int
    lib.pt_set_params.argtypes = [P, ctypes.c_int32, P, P, ctypes.c_int32]
    lib.pt_get_params.argtypes = [P, ctypes.c_int32, P, P, ctypes.c_int32]
    lib.pt_step.argtypes = [P, P, P, P, P, P, ctypes.c_int32]
    lib.pt_run.argtypes = [P, P, P, ctypes.c_int64, P, P, P, ctypes.c_int32]
    lib.pt_sync.argtypes = [P]
    lib.pt_set_stream.argtypes = [P, P]
    lib.pt_get_stream.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
    lib.pt_last_kernel_ms.argtypes = [P, f32p]
    lib.pt_tick.argtypes = [P]
    lib.pt_tick.restype = ctypes.c_int64
    lib.pt_kernel_path.argtypes = [P]
    lib.pt_kernel_path.restype = ctypes.c_int32
    lib.pt_stage_device.argtypes = [P, ctypes.c_int32]
    lib.pt_stage_device.restype = ctypes.c_int32
    lib.pt_ipc_export.argtypes = [P, ctypes.c_int32, P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    lib.pt_ipc_import.argtypes = [P, P, ctypes.c_size_t]
    lib.pt_set_trace.argtypes = [P, ctypes.c_int32, ctypes.c_int32]
    lib.pt_get_trace.argtypes = [P, P, ctypes.c_int32]
    lib.pt_destroy.argtypes = [P]
    lib.pt_destroy.restype = None
    lib.pt_last_error.restype = ctypes.c_char_p
    lib.pt_abi_version.restype = ctypes.c_int32
    for name in ("pt_set_params", "pt_get_params", "pt_step", "pt_run", "pt_sync", "pt_set_stream", "pt_get_stream",
                 "pt_last_kernel_ms", "pt_ipc_export", "pt_ipc_import", "pt_set_trace", "pt_get_trace"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(rc, what=""):
    if rc == PT_OK:
        return
    msg = load().pt_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == PT_EBUSY:
        raise ContractViolation(rc, text)
    if rc == PT_ENONFINITE:
        raise NonFiniteLoss(rc, text)
    if rc in (PT_EINVAL,):
        raise ValueError(text)
    if rc == PT_EUNSUPPORTED:
        raise NotImplementedError(text)
    raise PipelineError(rc, text)
