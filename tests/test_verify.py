"""The ``verify`` front end (cli/__init__.py:75-139,396-420): its sequential
definition is pinned to the golden-vector-pinned oracle (CPU), its flag
validation returns the reference's exit codes (CPU), and the full default grid
passes on the B200 (GPU)."""

import numpy as np
import pytest

from oracle import lbscan_oracle as O
from paper_2506_15976_b200 import verify as V


@pytest.mark.parametrize("L,M", [(1, 1), (7, 3), (33, 8), (40, 16)])
def test_sequential_definition_equals_oracle(L, M):
    prm = O.random_scan_params(O.seeded_rng(L), 2, L, 3, 4)
    y, h = V.seq_scan("forward", *prm)
    ry, rh = O.forward_scan(*prm)
    assert O.max_rel_err(y, ry) <= 1e-14 and O.max_rel_err(h, rh) <= 1e-14
    y, h = V.seq_scan("lbm", *prm, M)
    ry, rh = O.lbm_scan(*prm, M)
    assert O.max_rel_err(y, ry) <= 1e-14 and O.max_rel_err(h, rh) <= 1e-14
    y, h = V.seq_scan("global_bidir", *prm)
    ry, rh = O.global_bidir_scan(prm, prm)
    assert O.max_rel_err(y, ry) <= 1e-14 and O.max_rel_err(h, rh) <= 1e-14


@pytest.mark.parametrize("reverse", [False, True])
def test_sequential_fused_equals_oracle(reverse):
    from helpers import op_inputs
    x = op_inputs(3, 2, 29, 5, 4)
    got = V.seq_fused(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], 4, reverse)
    ref = O.lbm_selective_scan(**x, window=4, reverse=reverse)
    assert O.max_rel_err(got, ref) <= 1e-12


@pytest.mark.parametrize("argv", [["verify", "--m", "0"], ["verify", "--l", "0"], ["verify", "--variants", "x"],
                                  ["verify", "--precision", "half"]])
def test_bad_flags_exit_2(argv):
    from paper_2506_15976_b200 import cli
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == 2


@pytest.mark.gpu
def test_verify_default_grid_on_gpu(capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_15976_b200 import cli
    assert cli.main(["verify"]) == 0
    out = capsys.readouterr().out
    assert out.strip().endswith("ok")
    assert cli.main(["verify", "--l", "1,31,257,1024", "--m", "1,4,8,16", "--fused",
                     "--variants", "lbm", "--precision", "single"]) == 0


@pytest.mark.gpu
def test_verify_reports_failure(monkeypatch):
    """A wrong engine result is reported as FAIL with exit code 1."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_15976_b200 import cli, engine
    orig = engine.lbm_scan_par

    def broken(*a, **k):
        r = orig(*a, **k)
        r.y = np.asarray(r.y) * 1.001
        return r

    monkeypatch.setattr(engine, "lbm_scan_par", broken)
    assert cli.main(["verify", "--l", "31", "--m", "4", "--variants", "lbm"]) == 1
