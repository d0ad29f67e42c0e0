"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, and validates arguments (ShapeError mapping) before any
device work."""

import ctypes as C
import os
import re

import pytest

from paper_2506_15976_b200 import _lib
from paper_2506_15976_b200.errors import ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "lbscan_b200.h")).read()
    return sorted(set(re.findall(r"\b(lbs_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_symbols()
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTS)


def test_abi_version_and_tile_rule():
    L = _lib.lib()
    assert L.lbs_abi_version() == 2
    # engine.py:54-62 / test_engine.py:11-19
    for Ln, M in ((1024, 16), (257, 16), (256, 8), (200, 8), (129, 8), (128, 4), (64, 4), (1, 4)):
        assert L.lbs_select_tile_len(Ln) == M
    assert L.lbs_select_tile_len(0) == -1


def _args(**kw):
    a = _lib.ScanFwdArgs()
    a.batch, a.seqlen, a.dim, a.dstate, a.window = 2, 8, 4, 4, 4
    a.io_dtype = a.bc_dtype = _lib.LBS_F32
    a.flags = _lib.FLAG_LB | _lib.FLAG_SOFTPLUS
    fake = C.c_void_p(0x1000)
    for f in ("u", "delta", "A", "B", "C", "out"):
        setattr(a, f, fake)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("kw,msg", [
    (dict(seqlen=0), "dimensions"),
    (dict(window=0), "tile length"),
    (dict(io_dtype=9), "dtype"),
    (dict(u=None), "non-null"),
])
def test_invalid_arguments_raise_shape_error(kw, msg):
    L = _lib.lib()
    rc = L.lbs_scan_fwd(C.byref(_args(**kw)), None, 0, None)
    assert rc == _lib.LBS_ERR_INVALID
    assert msg in L.lbs_last_error().decode()
    with pytest.raises(ShapeError):
        _lib.check(rc, "lbm_selective_scan")


def test_prediscretized_rejects_bad_window():
    L = _lib.lib()
    a = _lib.PrediscretizedArgs()
    a.batch, a.seqlen, a.dim, a.dstate, a.window = 1, 4, 2, 2, 0
    a.dtype = _lib.LBS_F32
    assert L.lbs_prediscretized_fwd(C.byref(a), None) == _lib.LBS_ERR_INVALID


def test_python_api_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2506_15976_b200.scan import lbm_selective_scan
    x = torch.zeros(1, 4, 2)
    with pytest.raises(ShapeError):
        lbm_selective_scan(x, x, torch.zeros(2, 3), torch.zeros(1, 4, 3), torch.zeros(1, 4, 3))


def test_long_window_and_many_states_take_the_generic_path():
    """min(window, L) > 16 or N > 16 has no register tile: the state-outer generic
    kernels run instead (any M >= 1, any N, engine.py:65-85).  They need an fp32
    workspace of B*L*E floats (fwd), take no training checkpoints, and the argument
    checks still run before any launch."""
    L = _lib.lib()
    for kw in (dict(seqlen=40, window=32), dict(seqlen=40, window=64), dict(dstate=17), dict(dstate=64, window=40)):
        a = _args(**kw)
        need = L.lbs_scan_fwd_workspace_bytes(C.byref(a))
        assert need == 4 * a.batch * a.seqlen * a.dim, kw
        assert L.lbs_scan_ckpt_bytes(C.byref(a)) == 0, kw
        rc = L.lbs_scan_fwd(C.byref(a), None, 0, None)  # no workspace: rejected, nothing launched
        assert rc == _lib.LBS_ERR_INVALID, kw
        with pytest.raises(ShapeError):
            _lib.check(rc, "lbm_selective_scan")
    assert L.lbs_scan_fwd(C.byref(_args(dstate=5000)), None, 0, None) == _lib.LBS_ERR_UNSUPPORTED


def test_checkpoint_plan():
    L = _lib.lib()
    # backward chunk = whole tiles in an 8-step (M <= 8) or 16-step register window
    for M, K in ((1, 8), (3, 6), (4, 8), (5, 5), (8, 8), (9, 9), (16, 16)):
        assert L.lbs_scan_ckpt_len(1000, M) == K
    assert L.lbs_scan_ckpt_len(5, 16) == 5   # window clamps to L = 5
    assert L.lbs_scan_ckpt_len(40, 32) == -1
    a = _args(batch=2, seqlen=197, dim=384, dstate=16, window=8)
    assert L.lbs_scan_ckpt_bytes(C.byref(a)) == 2 * 25 * 384 * 16 * 4
    # a wrong ckpt_len is an argument error
    a.checkpoints, a.ckpt_len = C.c_void_p(0x2000), 4
    assert L.lbs_scan_fwd(C.byref(a), None, 0, None) == _lib.LBS_ERR_INVALID


def _bwd_args(**kw):
    a = _lib.ScanBwdArgs()
    a.fwd = _args()
    fake = C.c_void_p(0x3000)
    for f in ("dout", "du", "ddelta", "dA", "dB", "dC"):
        setattr(a, f, fake)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_bwd_argument_validation():
    L = _lib.lib()
    assert L.lbs_scan_bwd_workspace_bytes(C.byref(_bwd_args())) > 0
    for kw, msg in ((dict(dout=None), "non-null"), (dict(dz=C.c_void_p(0x10)), "dz"),
                    (dict(dD=C.c_void_p(0x10)), "dD")):
        rc = L.lbs_scan_bwd(C.byref(_bwd_args(**kw)), None, 0, None)
        assert rc == _lib.LBS_ERR_INVALID, kw
        assert msg in L.lbs_last_error().decode()
    # workspace is checked before any launch
    assert L.lbs_scan_bwd(C.byref(_bwd_args()), None, 0, None) == _lib.LBS_ERR_INVALID
    assert "workspace" in L.lbs_last_error().decode()
