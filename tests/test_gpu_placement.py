"""Phi^- batch placement at expansions (wamgpu.cu phi_append): the default
counting placement (k_key_hist + scan + k_key_place, warp-aggregated atomics:
the ray order inside a column is arbitrary) and the radix-sort placement
(WAMGPU_PHI_SORT=1, read once per process, hence the subprocess) must give the
same column bounds, and because the split sums each column in exact fixed
point (pin P8), bit-identical b-, beta, trees and objectives.
Run twice, the counting placement must also be run-to-run bit-identical."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
import paper_1508_04458_b200 as W
from oracle import oracle as O
from wam_testutil import problem_inputs
from paper_1508_04458_b200 import configs
O.lib(); W.load()
cfg, _, _, I0, d = problem_inputs(sys.argv[2], O, W)
c = W.Context(0)
c.set_geometry(configs.geometry(cfg, W.Geometry))
c.set_data(d, I0)
c.wam_init(cfg["L"])
rec = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
_, bp, bm = c.stats()
print(json.dumps({"obj": [r["objective"] for r in rec], "act": [r["active_set"] for r in rec],
                  "tree": h(c.tree()), "beta": h(c.beta()), "bm": h(bm), "bp": h(bp), "mu": h(c.image())}))
"""


def _run(name, sort):
    env = dict(os.environ)
    env.pop("WAMGPU_PHI_SORT", None)
    if sort:
        env["WAMGPU_PHI_SORT"] = "1"
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, name], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["small_lug", "cfg1"])
def test_counting_placement_matches_radix_sort(name):
    a, b, a2 = _run(name, False), _run(name, True), _run(name, False)
    assert a == b
    assert a == a2


def test_reinit_reuses_cached_z_approx(wam, orc):
    """zA (the per-ray approximation part of Z) is computed once per (matrix,
    L, Haar model) and reused by later wam_init calls (wamgpu.cu compute_z0):
    a second run, and one after an AM init in between (L = 0 row sums), must
    repeat the first bit for bit."""
    from paper_1508_04458_b200 import configs
    from wam_testutil import problem_inputs
    cfg, _, _, I0, d = problem_inputs("small_lug", orc, wam)
    c = wam.Context(0)
    c.set_geometry(configs.geometry(cfg, wam.Geometry))
    c.set_data(d, I0)
    runs = []
    for am_between in (False, False, True):
        if am_between:
            c.am_init()
            c.am_iterate(2)
        c.wam_init(cfg["L"])
        rec = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        runs.append(([r["objective"] for r in rec], c.tree().tobytes(), c.z_rows().tobytes(), c.scalars()["Z0"]))
    assert runs[0] == runs[1] == runs[2]
    c.close()
