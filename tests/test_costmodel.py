"""Cost counters vs the reference's (tests/golden/costs.npz from oracle/gen_golden.py):
count_scan_cost / count_model_cost / reports_to_csv / format_table must match the
reference exactly (test_costmodel.py, test_acceptance.py:56-75 in the reference)."""

import ast
import os

import numpy as np
import pytest

from paper_2506_15976_b200 import costmodel
from paper_2506_15976_b200.errors import ShapeError
from paper_2506_15976_b200.model import ModelConfig

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "costs.npz"))


def _vec(r):
    return [r.flops, r.hbm_reads, r.hbm_writes, r.tile_exchanges, r.register_ops]


def test_scan_cost_matches_reference():
    for dims, variant, want in zip(G["scan_dims"], G["scan_variants"], G["scan_counters"]):
        got = costmodel.count_scan_cost(str(variant), *map(int, dims))
        assert _vec(got) == list(map(int, want)), (variant, dims)


def test_engine_tallies_equal_closed_form():
    # the reference's engine tallies (engine.py:290) equal the closed form for B=2, L=37, E=3, N=4, M=8
    for variant, want in zip(("forward", "lbm"), G["engine_counters"]):
        assert _vec(costmodel.count_scan_cost(variant, 2, 37, 3, 4, 8)) == list(map(int, want))


def test_model_cost_matches_reference():
    for cfg, want in zip(G["model_cfgs"], G["model_counters"]):
        got = costmodel.count_model_cost(ModelConfig(**ast.literal_eval(str(cfg))))
        assert _vec(got) == list(map(int, want)), cfg


def test_csv_and_table_match_reference():
    reps = [costmodel.count_scan_cost(v, 2, 300, 4, 8, 8) for v in costmodel.VARIANTS]
    assert costmodel.reports_to_csv(reps) == str(G["csv"])
    assert costmodel.format_table(reps) == str(G["table"])


def test_structure():
    fwd = costmodel.count_scan_cost("forward", 2, 300, 4, 8, 8)
    lbm = costmodel.count_scan_cost("lbm", 2, 300, 4, 8, 8)
    bid = costmodel.count_scan_cost("global_bidir", 2, 300, 4, 8, 8)
    # LB adds only register work: identical traffic and exchanges (costmodel.py:5-8)
    assert (lbm.hbm_reads, lbm.hbm_writes, lbm.tile_exchanges) == (fwd.hbm_reads, fwd.hbm_writes, fwd.tile_exchanges)
    assert bid.counters() == {k: 2 * v for k, v in fwd.counters().items()}
    assert costmodel.count_scan_cost("lbm", 1, 100, 3, 4, 1).flops == costmodel.count_scan_cost("forward", 1, 100, 3, 4, 1).flops
    s = fwd + lbm
    assert s.variant == "forward+lbm" and s.flops == fwd.flops + lbm.flops
    with pytest.raises(ShapeError):
        costmodel.count_scan_cost("lbm", 1, 0, 1, 1, 1)
    with pytest.raises(ValueError):
        costmodel.count_scan_cost("nope", 1, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        costmodel.CostReport("x", flops=-1)


def test_fused_bytes_formula():
    # LBVim-Ti layer scan, bf16 = 158.18 MB
    assert costmodel.fused_scan_bytes(256, 197, 384, 16, 2, 2) == 158182400


def test_cli_flops(capsys, tmp_path):
    from paper_2506_15976_b200 import cli

    cfg = tmp_path / "cfg.txt"
    cfg.write_text("# LBVim-Ti\nimage_size=224\npatch_size=16\nin_channels=3\nembed_dim=192\ninner_dim=384\n"
                   "depth=24\nclass_token=middle\ntile_len=auto\nnum_classes=1000\nreverse_between_blocks=1\n")
    out = tmp_path / "o.csv"
    assert cli.main(["flops", "--config", str(cfg), "--out", str(out)]) == 0
    text = capsys.readouterr().out
    want = list(map(int, G["model_counters"][3]))  # the same config in the golden grid
    assert str(want[0]) in text and "global_bidir" in text
    rows = out.read_text().splitlines()
    assert rows[0] == "variant,flops,hbm_reads,hbm_writes,tile_exchanges,register_ops" and len(rows) == 5
    bad = tmp_path / "bad.txt"
    bad.write_text("nope=1\n")
    assert cli.main(["flops", "--config", str(bad)]) == 1


@pytest.mark.gpu
def test_cli_bench_gpu(capsys):
    from paper_2506_15976_b200 import cli

    assert cli.main(["bench", "--l", "100", "--m", "8", "--reps", "2", "--ben", "512", "--fused"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "variant,L,M,workers,median_ns,flops,hbm_elems,tile_exchanges"
    names = [ln.split(",")[0] for ln in lines[1:] if not ln.startswith("#")]
    assert names == ["forward", "lbm", "global_bidir", "fused_forward", "fused_lbm", "fused_global_bidir"]
    assert any(ln.startswith("# lbm/forward time ratio") for ln in lines)
