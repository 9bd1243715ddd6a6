"""Fused back projection + all-reduce over NVLink peer memory (multi-GPU 2D
view sharding; kernels_ar.cuh).

Only one GPU is available, so the R ranks are EMULATED as one cooperative grid
on one GPU (B200_PROFILING.md: "emulate the ranks as one kernel over all ranks'
data"): the same kernel, protocol and peer-pointer tables as production, with
the R ranks' buffers all on this device.  Checked bit-exactly:
  * the protocol: every rank's result equals the rank-order sum of the
    partials, for R = 1..8, ragged tile counts and several epochs;
  * the production producer: R contexts each holding one view shard of the
    matrix (context k plays rank k); the fused result equals the rank-order sum
    of the shards' own back projections (k_back<0,12,1>, same seg_dot) with the
    split partials riding along as the second half.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rank_order_sum(parts):
    s = np.zeros_like(parts[0])
    for p in parts:
        s = s + p
    return s


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 255, 256, 257, 4103, 2 * 262144])
def test_fused_allreduce_protocol(wam, R, n):
    rng = np.random.default_rng(1000 * R + n)
    parts = rng.standard_normal((R, n)) * rng.uniform(1e-3, 1e3, size=(R, 1))
    out = wam.selftest_fused_allreduce(parts, epochs=3)
    want = _rank_order_sum(parts)
    for k in range(R):
        assert np.array_equal(out[k], want), f"rank {k}"


@pytest.mark.parametrize("R", [2, 3, 4])
def test_fused_back_producer_shards(wam, R):
    from paper_1508_04458_b200 import configs
    cfg = configs.get("small")
    full = wam.Context(0)
    full.set_geometry(configs.geometry(cfg, wam.Geometry))
    rp, ci, v = full.matrix_csr()
    M, N = full.M, full.N
    V, D = cfg["views"], cfg["detectors"]
    rng = np.random.default_rng(7 + R)
    ctxs, ws, extras, want = [], [], [], []
    for k in range(R):
        v0, v1 = V * k // R, V * (k + 1) // R              # view shards, as partition()
        r0, r1 = v0 * D, v1 * D
        lo, hi = int(rp[r0]), int(rp[r1])
        c = wam.Context(0)
        c.set_grid(cfg["nx"], cfg["ny"], 1)
        c.set_matrix_csr(rp[r0:r1 + 1] - rp[r0], ci[lo:hi], v[lo:hi].astype(np.float64), N)
        w = rng.uniform(0.0, 2.0, size=r1 - r0).astype(np.float32).astype(np.float64)
        e = rng.standard_normal(N)
        ctxs.append(c); ws.append(w); extras.append(e)
        want.append(np.concatenate([c.back_project(w), e]))
    out = wam.selftest_fused_back(ctxs, ws, extras)
    ref = _rank_order_sum(want)
    for k in range(R):
        assert np.array_equal(out[k], ref), f"rank {k}"
    # and the sharded sum is the full back projection up to summation order
    wfull = np.concatenate(ws)
    g = full.back_project(wfull)
    assert np.allclose(out[0][:N], g, rtol=1e-12, atol=1e-12 * np.abs(g).max())
    for c in ctxs:
        c.close()
    full.close()
