"""The C-ABI library loads on a CPU-only host and exports every symbol include/partime_b200.h
declares; argument validation happens before any CUDA call; without a GPU the engine fails
loudly instead of falling back to the CPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2210_09147_b200 import _lib, model as mdl

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "partime_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pt_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = _lib.load()
    syms = header_symbols()
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.pt_abi_version() == 2


def _cfg(dims, D_first, act=None, batch=1, **kw):
    L = len(dims) - 1
    D_i = (ctypes.c_int32 * len(dims))(*dims)
    A_i = (ctypes.c_int32 * L)(*(act or [1] * L))
    S_i = (ctypes.c_int32 * len(D_first))(*D_first)
    base = dict(n_layers=L, dims=D_i, act=A_i, loss=0, optimizer=0, lr=1e-3, n_stages=len(D_first) - 1,
                stage_first_layer=S_i, batch=batch, learn=1, act_delay=1, local_stage_first=0,
                local_stage_count=0, grid=0, timeout_ms=0)
    base.update(kw)
    return _lib.PTConfig(**base), (D_i, A_i, S_i)


@pytest.mark.parametrize("dims,sfl,kw,msg", [
    ([4, 4], [0, 1, 1], {}, "D=2 > L=1"),
    ([4, 4, 4, 4], [0, 2, 1, 3], {}, "empty or out of order"),
    ([4, 4, 4], [0, 2], {"batch": 65}, "batch"),
    ([4, 9000], [0, 1], {}, "8192"),
    ([4, 4], [1, 1], {}, "start at layer 0"),
    ([4, 4], [0, 1], {"act_delay": 2}, "act_delay"),
])
def test_create_validation(dims, sfl, kw, msg):
    lib = _lib.load()
    cfg, keep = _cfg(dims, sfl, **kw)
    h = ctypes.c_void_p()
    rc = lib.pt_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == _lib.PT_EINVAL and msg in lib.pt_last_error().decode()


def test_adam_and_softmax_ce_pass_validation():
    """Adam and softmax cross-entropy are implemented: the config validates (without a GPU
    pt_create then fails with PT_ECUDA, never PT_EINVAL / PT_EUNSUPPORTED)."""
    lib = _lib.load()
    for kw in (dict(loss=1), dict(optimizer=1), dict(loss=1, optimizer=1, batch=4)):
        cfg, keep = _cfg([4, 4], [0, 1], **kw)
        h = ctypes.c_void_p()
        rc = lib.pt_create(ctypes.byref(cfg), ctypes.byref(h))
        assert rc not in (_lib.PT_EINVAL, _lib.PT_EUNSUPPORTED), lib.pt_last_error()
        if rc == _lib.PT_OK:
            lib.pt_destroy(h)


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    from paper_2210_09147_b200 import engine
    m = mdl.mlp([8, 8, 4], seed=0)
    with pytest.raises(_lib.PipelineError):
        engine.Pipeline(m, [3], "sgd", 0.1, np.zeros(8, np.float32), np.zeros(4, np.float32))


def test_engine_rejects_bad_shapes_before_the_library():
    from paper_2210_09147_b200 import engine
    m = mdl.mlp([8, 8, 4], seed=0)
    with pytest.raises(ValueError, match="stage-1 input"):
        engine.Pipeline(m, [3], "sgd", 0.1, np.zeros(7, np.float32), np.zeros(4, np.float32))
    with pytest.raises(ValueError, match="splits dense layer"):
        engine.Pipeline(m, [1, 2], "sgd", 0.1, np.zeros(8, np.float32), np.zeros(4, np.float32))
