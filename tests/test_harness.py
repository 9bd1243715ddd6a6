"""Harness outputs: records
CSV, active-tree manifest round trip on real oracle trees (2D and separable
3D models), compare_runs.  CPU only: the trees come from the oracle, whose
tree layout the device matches bit-exactly (tests/test_gpu_parity*.py)."""
import io

import numpy as np
import pytest

from paper_1508_04458_b200 import harness as H
from wam_testutil import problem_inputs


def _oracle_tree(orc, name, haar):
    cfg, p, _, I0, d = problem_inputs(name, orc, None, mirror=True)
    if cfg["nz"] > 1:
        p.set_haar_dim(haar)
    p.wam_init(d, I0, cfg["L"])
    done = 0
    for ev in cfg["schedule"][:2]:
        p.wam_iterate(ev - done)
        done = ev
        p.wam_expand(0.1)
    return cfg, p.wam_tree()


@pytest.mark.parametrize("name,haar", [("tiny", 2), ("tiny3d", 2), ("tiny3d16", 3)])
def test_manifest_round_trip(orc, name, haar):
    cfg, tree = _oracle_tree(orc, name, haar)
    assert tree.any()
    args = (cfg["nx"], cfg["ny"], cfg["nz"], cfg["L"], haar)
    text = H.tree_manifest(tree, *args)
    back = H.parse_manifest(text, *args)
    assert np.array_equal(back, tree)
    # one line per active coefficient
    nact = int(tree.sum()) * (7 if haar == 3 else 3 * cfg["nz"])
    napx = (cfg["nx"] >> cfg["L"]) * (cfg["ny"] >> cfg["L"]) * ((cfg["nz"] >> cfg["L"]) if haar == 3 else cfg["nz"])
    assert len(text.splitlines()) == nact + napx


def test_manifest_rejects_broken_trees(orc):
    cfg, tree = _oracle_tree(orc, "tiny", 2)
    args = (cfg["nx"], cfg["ny"], cfg["nz"], cfg["L"], 2)
    lines = [l for l in H.tree_manifest(tree, *args).splitlines() if " a " not in l]
    with pytest.raises(ValueError):                      # a subband missing
        H.parse_manifest("\n".join(lines[1:]), *args)
    fine = [l for l in lines if l.split()[1] == "1"]
    if fine:
        with pytest.raises(ValueError):                  # level-1 blocks without parents
            H.parse_manifest("\n".join(fine), *args)
    with pytest.raises(ValueError):
        H.parse_manifest("0 9 h 0 0", *args)


def test_records_csv_round_trip_and_determinism():
    recs = [{"iter": i, "objective": 1e6 / i + 0.1 * i, "elapsed_s": 0.01 * i, "active_set": 64 + i,
             "cum_updates": 64 * i} for i in range(1, 8)]
    f = io.StringIO()
    H.write_records_csv(f, recs)
    f.seek(0)
    back = H.read_records_csv(f)
    assert back == recs
    a, b = io.StringIO(), io.StringIO()
    H.write_records_csv(a, recs, with_time=False)
    H.write_records_csv(b, [dict(r, elapsed_s=9.0) for r in recs], with_time=False)
    assert a.getvalue() == b.getvalue() and "elapsed_s" not in a.getvalue()
    with pytest.raises(ValueError):
        H.write_records_csv(io.StringIO(), recs[::-1])


def test_compare_runs():
    rng = np.random.default_rng(3)
    img = rng.random(64)
    log = [{"iter": i, "objective": 100.0 / i, "elapsed_s": 0.1 * i} for i in range(1, 11)]
    rep = H.compare_runs(log, log, img, img, truth=img)
    assert rep["a"] == rep["b"] == {"iter": 10, "elapsed_s": 1.0}
    assert not rep["difference"].any() and rep["rmse_a"] == 0.0
    fast = [{"iter": i, "objective": 50.0 / i, "elapsed_s": 0.2 * i} for i in range(1, 11)]
    rep = H.compare_runs(log, fast, img, img + 1.0)
    assert rep["target_objective"] == 5.0 and rep["b"]["iter"] == 10 and rep["a"] is None
    assert np.allclose(rep["difference"], 1.0)
    with pytest.raises(ValueError):
        H.compare_runs(log, log, img, img[:10])
