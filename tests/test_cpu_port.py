"""The CPU port used as bench.py's CPU baseline is pinned to the reference:
its engine is bitwise the reference's numba engine (golden engine32 outputs)
and its fused op / model agree with the reference's outputs."""

import os

import numpy as np
import pytest

from oracle import cpu_port as P
from oracle import lbscan_oracle as O
from helpers import op_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _build():
    P.build()


def test_engine_port_is_bitwise_the_reference_engine():
    g = np.load(os.path.join(GOLD, "scan_grid.npz"))
    for L in (1, 5, 31, 128, 129, 197, 256, 257):
        p = [g[f"L{L}_{k}"].astype(np.float32) for k in ("abar", "bx", "c", "dx")]
        for M in (1, 3, 4, 8, 16):
            y, h = P.scan_par(*p, M, True, False, threads=2)
            np.testing.assert_array_equal(y, g[f"L{L}_M{M}_engine32_y"])
            np.testing.assert_array_equal(h, g[f"L{L}_M{M}_engine32_h"])


def test_reverse_and_forward_variants():
    p = O.random_scan_params(O.seeded_rng(4), 2, 77, 3, 4)
    for M in (3, 8):
        y, h = P.scan_par(*p, M, True, True)
        ry, rh = O.lbm_scan(*[a[:, ::-1] for a in p], M)
        assert O.max_rel_err(y, ry[:, ::-1]) <= 1e-5
        assert O.max_rel_err(h, rh) <= 1e-5
    y, _ = P.scan_par(*p, 4, False, False)
    assert O.max_rel_err(y, O.forward_scan(*p)[0]) <= 1e-5


def test_fused_op_port():
    inp = {k: np.asarray(v, np.float32) for k, v in op_inputs(5, 2, 97, 12, 16).items()}
    for rev in (False, True):
        got = P.fused_op(**inp, M=8, reverse=rev)
        ref = O.lbm_selective_scan(**inp, window=8, reverse=rev)
        assert O.max_rel_err(got, ref) <= 1e-5


@pytest.mark.parametrize("i", [0, 1])
def test_model_port_matches_reference_golden(i):
    g = np.load(os.path.join(GOLD, "model.npz"))
    pre = f"m{i}_"
    cfg = {k[len(pre) + 4:]: g[k].item() for k in g.files if k.startswith(pre + "cfg_")}
    cfg["tile_len"] = None if cfg["tile_len"] in (None, "auto") else int(cfg["tile_len"])
    params = {k[len(pre) + 2:]: g[k].astype(np.float32) for k in g.files if k.startswith(pre + "p_")}
    logits = P.model_forward(g[pre + "images"].astype(np.float32), cfg, params)
    assert O.max_rel_err(logits, g[pre + "logits"]) <= 1e-4
