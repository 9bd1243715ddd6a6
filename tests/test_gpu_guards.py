"""Guard-band run of the small parity workloads (the library's own stand-in for
compute-sanitizer memcheck / initcheck, which is closed on the GPU pool:
profiles/r06/sanitizer_memcheck_closed.log).  A subprocess with WAMGPU_GUARD=1
(every device allocation: 256-byte 0xA5 bands on both sides, body filled with
0xFF = NaN) runs the 2D and 3D wavelet-AM / AM paths, the sharded 3D rank
groups' single-rank path, the banded and the on-the-fly TMA forward, compares
each with an unguarded run's objective bits (an uninitialised read would
poison them), and checks that no band was overwritten."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %(root)r)
import numpy as np
import paper_1508_04458_b200 as W
from paper_1508_04458_b200 import configs

out = {}
tot = [0, 0, ""]
def run(name, haar=None, algo=None, projector=0):
    print("start", name, haar, algo, projector, file=sys.stderr, flush=True)
    cfg = configs.get(name)
    g = configs.geometry(cfg, W.Geometry)
    mu = W.rasterize(g, configs.phantom(cfg))
    I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
    d = W.simulate_device(g, mu, I0, cfg["seed"])
    c = W.Context(0)
    c.set_geometry(g)
    c.set_projector(projector)
    if haar:
        c.set_haar_dim(haar)
    c.set_data(d, I0)
    if (algo or cfg["algo"]) == "wam":
        c.wam_init(cfg["L"])
        r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
    else:
        c.am_init()
        r = c.am_iterate(cfg["J"])
    l = c.forward_project(mu)
    b = c.back_project(np.ones(l.size))
    key = f"{name}/{haar}/{algo}/{projector}"
    print("running", key, file=sys.stderr, flush=True)
    out[key] = [float(r[-1]["objective"]).hex(), float(np.abs(c.image()).sum()).hex(),
                float(l.sum()).hex(), float(b.sum()).hex()]
    assert np.isfinite(c.image()).all() and np.isfinite(l).all() and np.isfinite(b).all(), key
    n, b, m = W.debug_guards()   # while the context's buffers are live
    tot[0] += n; tot[1] += b; tot[2] = tot[2] or m
    c.close()

run("tiny"); run("tiny", algo="am"); run("small_lug")
run("tiny3d"); run("tiny3d", algo="am"); run("tiny3d16", haar=3); run("small3d", haar=3)
run("tiny3d24", haar=3, projector=1); run("small3d", algo="am", projector=1)
out["guards"] = tot
print("RESULT " + json.dumps(out))
"""


def _run(guard, extra=None):
    env = dict(os.environ)
    env.pop("WAMGPU_GUARD", None)
    if guard:
        env["WAMGPU_GUARD"] = "1"
    env.update(extra or {})
    p = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], capture_output=True, text=True, env=env,
                       timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")][-1]
    return json.loads(line[7:])


def test_guard_bands_clean_and_results_unchanged():
    plain, guarded = _run(False), _run(True)
    assert plain.pop("guards")[:2] == [0, 0]
    checked, bad, msg = guarded.pop("guards")
    assert checked > 20 and bad == 0, msg
    assert guarded == plain   # bit-identical objectives / sums: nothing read before it was written


def test_guard_bands_banded_forward():
    """the banded 3D forward (cfg4 path) forced on the small stacks"""
    g = _run(True, {"WAMGPU_FWD_BAND_MB": "0.004"})
    checked, bad, msg = g.pop("guards")
    assert checked > 20 and bad == 0, msg
