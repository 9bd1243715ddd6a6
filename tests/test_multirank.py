"""World-size-2 gloo tests of the view-sharded 2D algebra, on
CPU: each rank owns a contiguous block of views (CSR rows), computes partial
back projections / signed splits over its rows, and an all-reduce SUM makes the
replicated coefficient update identical to the single-rank result.  The
partition rule is the one libwamgpu.so uses (wamgpu.cu set_geometry)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _geom(name):
    import paper_1508_04458_b200 as W
    from paper_1508_04458_b200 import configs
    return W, configs.get(name), configs.geometry(configs.get(name), W.Geometry)


def lib_plan(name, rank, nranks, view_groups=0, algo="wam", levels=0, haar=3):
    """The rank's share as libwamgpu.so computes it (wamgpu_plan_partition:
    the arithmetic set_geometry applies; host-only, no GPU)."""
    W, cfg, g = _geom(name)
    return W.plan_partition(g, rank, nranks, view_groups, algo, haar, levels)


def view_range(V, rank, nranks):
    """The documented rule: v0 = V*rank/P, v1 = V*(rank+1)/P."""
    return V * rank // nranks, V * (rank + 1) // nranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    from wam_testutil import problem_inputs
    cfg, p, mu_true, I0, d = problem_inputs("tiny", O, None)
    rp, ci, v = p.csr()
    pl = lib_plan("tiny", rank, world)                    # the library's own row shard
    r0, r1 = pl["row_begin"], pl["row_end"]
    # one AM iteration, sharded: partial H^T q and H^T d over own rows, all-reduce
    q = I0 * np.exp(-p.forward_project(np.zeros(p.N)))
    def partial_back(w):
        g = np.zeros(p.N)
        for y in range(r0, r1):
            sl = slice(int(rp[y]), int(rp[y + 1]))
            np.add.at(g, ci[sl].astype(np.int64), v[sl] * w[y])
        return g
    gq = torch.from_numpy(partial_back(q))
    gd = torch.from_numpy(partial_back(d))
    dist.all_reduce(gq)
    dist.all_reduce(gd)
    # objective partial over own rows, all-reduced
    obj = torch.tensor([float(np.sum(q[r0:r1] - d[r0:r1] + d[r0:r1] * np.log(np.where(d[r0:r1] > 0, d[r0:r1] / q[r0:r1], 1.0))))],
                       dtype=torch.float64)
    dist.all_reduce(obj)
    # Z0 partial max over own rows, all-reduced MAX
    rs = np.array([v[int(rp[y]):int(rp[y + 1])].sum() for y in range(r0, r1)] or [0.0])
    z0 = torch.tensor([rs.max()], dtype=torch.float64)
    dist.all_reduce(z0, op=dist.ReduceOp.MAX)
    out[rank] = (gq.numpy().copy(), gd.numpy().copy(), float(obj.item()), float(z0.item()), (r0, r1))
    dist.destroy_process_group()


def test_view_partition_covers_rows_once():
    for V in (180, 720, 7):
        for P in (1, 2, 3, 4, 8):
            rng = [view_range(V, r, P) for r in range(P)]
            assert rng[0][0] == 0 and rng[-1][1] == V
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


@pytest.mark.parametrize("name", ["tiny", "cfg1", "cfg2"])
@pytest.mark.parametrize("R", [1, 2, 3, 8])
def test_library_plan_2d_is_view_sharding(name, R):
    W, cfg, g = _geom(name)
    D = cfg["detectors"]
    rows = []
    for r in range(R):
        pl = lib_plan(name, r, R)
        assert (pl["view_groups"], pl["z_groups"], pl["view_group"]) == (R, 1, r)
        v0, v1 = view_range(cfg["views"], r, R)
        assert (pl["row_begin"], pl["row_end"]) == (v0 * D, v1 * D)
        assert pl["slab_slices"] == 1 and pl["split_update"] == 0
        rows.append((pl["row_begin"], pl["row_end"]))
    assert rows[0][0] == 0 and rows[-1][1] == cfg["views"] * D
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    with pytest.raises(W.ConfigError):          # 2D shards views over ALL ranks
        W.plan_partition(g, 0, R + 1, view_groups=1)


@pytest.mark.parametrize("name,R,Rv", [("cfg3", 8, 8), ("cfg3", 8, 1), ("cfg3", 8, 2), ("cfg4", 8, 8),
                                       ("cfg4", 4, 2), ("tiny3d16", 4, 2), ("cfg5", 8, 8)])
def test_library_plan_3d_grid(name, R, Rv):
    """Every (ray, slice) once; slab strides; the split update's owned tile rows
    tile the image (view groups x z-slabs, rank = zg*Rv + vg)."""
    W, cfg, g = _geom(name)
    algo = "am" if cfg["algo"] == "am" else "wam"
    L = cfg["L"]
    seen = np.zeros((cfg["views"], cfg["nz"]), np.int32)
    own = {}
    for r in range(R):
        pl = lib_plan(name, r, R, Rv, algo, L)
        vg, zg, (v0, v1), (s0, s1) = grid_of(r, R, Rv, cfg["views"], cfg["nz"])
        assert (pl["view_group"], pl["z_group"]) == (vg, zg)
        D = cfg["detectors"]
        assert (pl["row_begin"], pl["row_end"]) == (v0 * D, v1 * D)
        assert (pl["slab_begin"], pl["slab_begin"] + pl["slab_slices"]) == (s0, s1)
        P = pl["slab_stride"]
        assert P >= pl["slab_slices"] and P in (8, 16, 32, 64, 128)
        seen[v0:v1, s0:s1] += 1
        if Rv > 1:
            assert pl["split_update"] == 1
            own.setdefault(zg, []).append((pl["own_row_begin"], pl["own_rows"]))
    assert (seen == 1).all()
    unit = cfg["ny"] if algo == "am" else cfg["ny"] >> L
    for zg, lst in own.items():
        lst.sort()
        assert lst[0][0] == 0 and sum(n for _, n in lst) == unit
        assert all(a[0] + a[1] == b[0] for a, b in zip(lst, lst[1:]))


def test_two_rank_sharded_am_step_matches_single_rank():
    from oracle import oracle as O
    from wam_testutil import problem_inputs
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="fork")
    cfg, p, mu_true, I0, d = problem_inputs("tiny", O, None)
    q = I0 * np.exp(-p.forward_project(np.zeros(p.N)))
    g_ref = p.back_project(q)
    b_ref = p.back_project(d)
    for r in range(world):
        gq, gd, obj, z0, rows = out[r]
        assert np.allclose(gq, g_ref, rtol=1e-12, atol=0)
        assert np.allclose(gd, b_ref, rtol=1e-12, atol=0)
        assert abs(obj - O.i_divergence(d, q)) <= 1e-9 * abs(obj)
    # replicated update is identical on both ranks (same all-reduced inputs)
    assert np.array_equal(out[0][0], out[1][0]) and out[0][3] == out[1][3]
    p.am_init(d, I0)
    assert out[0][3] == p.am_get()["Z0"]
    # the replicated multiplicative AM update from the all-reduced sums equals
    # the single-rank oracle's first iterate
    gq, gd = out[0][0], out[0][1]
    z0 = out[0][3]
    mu = np.where((gd > 0) & (gq > 0), np.maximum(0.0, np.log(np.where(gd > 0, gq / np.where(gd > 0, gd, 1), 1)) / z0), 0.0)
    p.am_iterate(1)
    assert np.allclose(mu, p.am_get()["mu"], rtol=1e-10, atol=1e-14)


def _p2p_worker(rank, world, port, out):
    """bench.Plumbing over gloo: the IPC-handle blobs every rank exports are
    gathered in RANK ORDER and concatenated (wamgpu_p2p_import's layout), and
    the tile protocol of kernels_ar.cuh (owner = tile % R, owner sums the R
    contributions in rank order, broadcasts) gives every rank the same result."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import torch
    pl = bench.Plumbing(rank, world)
    blob = bytes([rank]) * 256                            # WAMGPU_P2P_BLOB bytes
    blobs = b"".join(pl.all_gather_bytes(blob))
    # host model of the protocol over gloo: staging = all_gather of partials
    n, T = 1000, 256
    rng = np.random.default_rng(rank)
    part = rng.standard_normal(n)
    parts = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(part))
    res = np.empty(n)
    owned = []
    for t in range((n + T - 1) // T):
        if t % world != rank:
            continue
        owned.append(t)
        sl = slice(t * T, min(n, (t + 1) * T))
        s = np.zeros(sl.stop - sl.start)
        for k in range(world):                               # rank order
            s = s + parts[k].numpy()[sl]
        res[sl] = s
    # broadcast of owned tiles: every rank assembles the full result
    full = torch.zeros(n, dtype=torch.float64)
    mine = torch.zeros(n, dtype=torch.float64)
    for t in owned:
        sl = slice(t * T, min(n, (t + 1) * T))
        mine[sl] = torch.from_numpy(res[sl])
    dist.all_reduce(mine)                                    # disjoint tiles: a gather
    full += mine
    out[rank] = (blobs, full.numpy().copy(), [p.numpy().copy() for p in parts])
    pl.close()


def test_two_rank_p2p_blob_exchange_and_tile_protocol():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_p2p_worker, args=(world, port, out), nprocs=world, join=True, start_method="fork")
    want_blobs = bytes([0]) * 256 + bytes([1]) * 256
    for r in range(world):
        assert out[r][0] == want_blobs
    parts = out[0][2]
    s = np.zeros_like(parts[0])
    for p in parts:
        s = s + p
    assert np.array_equal(out[0][1], s) and np.array_equal(out[1][1], s)


# ---- 3D rank grid (wamgpu.cu resolve_grid / partition): Rv view groups x Rz
# z-slab groups, rank = zg*Rv + vg; partial back projections are summed over
# the VIEW group (ranks sharing a slab: ncclCommSplit(color=zg)), the
# objective over every rank.
def grid_of(rank, R, Rv, V, nz):
    Rz = R // Rv
    vg, zg = rank % Rv, rank // Rv
    v0, v1 = view_range(V, vg, Rv)
    s0, s1 = nz * zg // Rz, nz * (zg + 1) // Rz
    return vg, zg, (v0, v1), (s0, s1)


def test_grid_partition_covers_ray_slices_once():
    for V, nz in ((60, 16), (720, 64), (7, 5)):
        for R, Rv in ((1, 1), (2, 1), (2, 2), (4, 2), (8, 4), (8, 8), (8, 2), (6, 3)):
            if nz < R // Rv:
                continue
            seen = np.zeros((V, nz), np.int32)
            for r in range(R):
                _, _, (v0, v1), (s0, s1) = grid_of(r, R, Rv, V, nz)
                seen[v0:v1, s0:s1] += 1
            assert (seen == 1).all(), (V, nz, R, Rv)


def _grid_worker(rank, world, port, Rv, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    from wam_testutil import problem_inputs
    cfg, p, mu_true, I0, d = problem_inputs("tiny3d16", O, None)
    Rz = world // Rv
    # sub-groups as ncclCommSplit builds them (every rank creates every group)
    vgroups = [dist.new_group([z * Rv + v for v in range(Rv)]) for z in range(Rz)]
    pl = lib_plan("tiny3d16", rank, world, Rv, "wam", cfg["L"])   # the library's grid
    zg = pl["z_group"]
    s0, s1 = pl["slab_begin"], pl["slab_begin"] + pl["slab_slices"]
    M, N = p.M, p.N
    rp, ci, v = p.csr()          # in-plane matrix, shared by every slice (pin P2)
    r0, r1 = pl["row_begin"], pl["row_end"]
    q = (I0 * np.exp(-p.forward_project(np.zeros(N * cfg["nz"])))).reshape(cfg["nz"], M)
    g = np.zeros((s1 - s0, N))
    for y in range(r0, r1):
        sl = slice(int(rp[y]), int(rp[y + 1]))
        g[:, ci[sl].astype(np.int64)] += np.outer(q[s0:s1, y], v[sl])
    gt = torch.from_numpy(g.ravel().copy())
    dist.all_reduce(gt, group=vgroups[zg])           # S_VIEWS
    dd = d.reshape(cfg["nz"], M)
    qq = q[s0:s1, r0:r1]
    dl = dd[s0:s1, r0:r1]
    obj = torch.tensor([float(np.sum(qq - dl + dl * np.log(np.where(dl > 0, dl / qq, 1.0))))], dtype=torch.float64)
    dist.all_reduce(obj)                              # S_ALL
    out[rank] = (gt.numpy().copy(), float(obj.item()), (s0, s1))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,Rv", [(2, 2), (4, 2)])
def test_grid_sharded_back_projection_and_objective(world, Rv):
    from oracle import oracle as O
    from wam_testutil import problem_inputs
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_grid_worker, args=(world, port, Rv, out), nprocs=world, join=True, start_method="fork")
    cfg, p, mu_true, I0, d = problem_inputs("tiny3d16", O, None)
    q = I0 * np.exp(-p.forward_project(np.zeros(p.N * cfg["nz"])))
    g_ref = p.back_project(q).reshape(cfg["nz"], p.N)
    obj_ref = O.i_divergence(d, q)
    for r in range(world):
        g, obj, (s0, s1) = out[r]
        assert np.allclose(g, g_ref[s0:s1].ravel(), rtol=1e-12, atol=1e-12 * np.abs(g_ref).max())
        assert abs(obj - obj_ref) <= 1e-9 * abs(obj_ref)
        # the view shards of a slab hold identical sums (replicated update)
        for k in range(world):
            if k // Rv == r // Rv:
                assert np.array_equal(out[k][0], g)
