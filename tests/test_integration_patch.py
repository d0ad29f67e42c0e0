"""INTEGRATION.md §2a, executed against the unmodified reference (CPU container).

The reference-side patch a maintainer adds to ``lbscan/block.py:_run_scan``
(block.py:132-138) is taken verbatim from INTEGRATION.md and installed into the
reference's own ``block`` module; the reference's block and model forward then
run with ``scan_impl="cuda"``.  There is no GPU here, so
``paper_2506_15976_b200.engine`` is replaced by a stub whose entry points have
the *same signatures* as the real module (checked with ``inspect``) and compute
with the CPU oracle — what is pinned is the call shape (numpy in / numpy out,
``TilePlan.for_length``, ``workers=``, ``.y``), so API drift on either side fails
here.  The arithmetic of the real engine is covered by the -m gpu tests.
Skipped where /root/reference is absent (the GPU box)."""

import inspect
import os
import re
import sys
import types

import numpy as np
import pytest

REF = os.environ.get("LBSCAN_REFERENCE", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if not os.path.isdir(os.path.join(REF, "lbscan")):
    pytest.skip("the reference is not present (GPU box)", allow_module_level=True)

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lbscan")
sys.dont_write_bytecode = True
if REF not in sys.path:
    sys.path.insert(0, REF)

ref_block = pytest.importorskip("lbscan.block")
from lbscan import model as ref_model  # noqa: E402
from lbscan.core import seeded_rng  # noqa: E402

import paper_2506_15976_b200  # noqa: E402
from oracle import lbscan_oracle as O  # noqa: E402
from paper_2506_15976_b200 import engine as real_engine  # noqa: E402
from paper_2506_15976_b200.tiling import TilePlan  # noqa: E402


def _patch_source():
    """The ``_run_scan`` code block of INTEGRATION.md §2a, with the elided
    reference branches restored from block.py:132-138."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text.split("### 2a.", 1)[1].split("### 2b.", 1)[0]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    orig = inspect.getsource(ref_block._run_scan).splitlines()
    par = "\n".join(orig[1:4])   # the "par" branch body (block.py:133-135)
    seq = "\n".join(orig[4:6])   # the "seq" branch (block.py:136-137)
    code = code.replace('    if scan_impl == "par":\n        ...', par, 1)
    code = code.replace('    if scan_impl == "seq":\n        ...', seq, 1)
    assert "..." not in code, code
    return code


class _StubEngine(types.ModuleType):
    """CPU stand-in for paper_2506_15976_b200.engine with its exact signatures."""

    TilePlan = TilePlan

    @staticmethod
    def lbm_scan_par(abar, bx, c, dx, plan: TilePlan, workers: int = 1):
        plan.check(np.asarray(abar).shape[1])
        y, hf = O.lbm_scan(abar, bx, c, dx, plan.tile_len)
        return real_engine.ScanOutput(y=y, h_final=hf)


def test_stub_mirrors_the_real_engine_signatures():
    def shape(f):  # parameter names, kinds and defaults (annotations aside)
        return [(p.name, p.kind, p.default) for p in inspect.signature(f).parameters.values()]
    assert shape(_StubEngine.lbm_scan_par) == shape(real_engine.lbm_scan_par)
    assert shape(real_engine.lbm_scan_par)[:5] == [(n, inspect.Parameter.POSITIONAL_OR_KEYWORD, inspect.Parameter.empty)
                                                   for n in ("abar", "bx", "c", "dx", "plan")]
    assert real_engine.TilePlan is TilePlan
    assert TilePlan.for_length(197, None).tile_len == 8  # engine.py:54-62


@pytest.fixture
def patched(monkeypatch):
    stub = _StubEngine("paper_2506_15976_b200.engine")
    monkeypatch.setattr(paper_2506_15976_b200, "engine", stub)
    monkeypatch.setitem(sys.modules, "paper_2506_15976_b200.engine", stub)
    ns = dict(vars(ref_block))
    exec(compile(_patch_source(), "INTEGRATION.md#2a", "exec"), ns)
    monkeypatch.setattr(ref_block, "_run_scan", ns["_run_scan"])
    return ns["_run_scan"]


def test_patched_run_scan_matches_par(patched):
    rng = seeded_rng(3)
    B, L, E, N, M = 2, 37, 5, 4, 4
    abar = rng.uniform(0.3, 0.95, (B, L, E, N))
    bx = rng.standard_normal((B, L, E, N))
    c = rng.standard_normal((B, L, N))
    dx = rng.standard_normal((B, L, E))
    got = patched(abar, bx, c, dx, M, "cuda", 1)
    ref = patched(abar, bx, c, dx, M, "par", 1)
    assert isinstance(got, np.ndarray) and got.shape == (B, L, E)
    assert O.max_rel_err(got, ref) <= 1e-6
    with pytest.raises(ref_block.ShapeError):
        patched(abar, bx, c, dx, M, "nope", 1)


def test_reference_model_forward_through_the_patch(patched):
    cfg = ref_model.ModelConfig(image_size=32, patch_size=8, in_channels=3, embed_dim=16, inner_dim=32,
                                state_dim=4, depth=2, num_classes=5)
    params = ref_model.init_model_weights(cfg, seed=0)
    imgs = seeded_rng(1).standard_normal((2, 32, 32, 3))
    got = ref_model.model_forward(imgs, cfg, params, scan_impl="cuda")
    ref = ref_model.model_forward(imgs, cfg, params, scan_impl="par")
    assert O.max_rel_err(got, ref) <= 1e-6
