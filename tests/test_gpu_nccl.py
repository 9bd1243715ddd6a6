"""The NCCL collective path of libwamgpu.so on one GPU: a 1-rank communicator
(wamgpu_set_comm with an ncclUniqueId) routes every all-reduce of the view-
sharded 2D path (partial back projections || b-, objective, Z0 / criterion
maxima) through ncclAllReduce.  Results must be bit-identical to the
communicator-free run (a 1-rank all-reduce is an exact copy)."""
import numpy as np
import pytest

from wam_testutil import problem_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["am", "wam"])
def test_one_rank_nccl_matches_no_comm(wam, orc, algo):
    from paper_1508_04458_b200 import configs
    cfg, p, _, I0, d = problem_inputs("small", orc, wam)
    out = []
    for use_comm in (False, True):
        c = wam.Context(0)
        if use_comm:
            c.set_comm(wam.nccl_unique_id(), 0, 1)
        c.set_geometry(configs.geometry(cfg, wam.Geometry))
        c.set_data(d, I0)
        if algo == "am":
            c.am_init()
            rec = c.am_iterate(cfg["J"])
        else:
            c.wam_init(cfg["L"])
            rec = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        t = c.timing()
        out.append(([r["objective"] for r in rec], c.image(), c.tree() if algo == "wam" else None, t))
        c.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    if algo == "wam":
        assert np.array_equal(out[0][2], out[1][2])
