"""Benchmark of the wavelet-AM iteration (BASELINE.json metric: AM iterations/s and
ray-voxel updates/s vs the HBM roofline).

Default workload (N=1): BASELINE configs[1] = cfg2, 2D fan-beam 512x512 at
0.5 mm, 720 views x 1024 arc detectors, seeded luggage phantom, I0 = 2e5 with
Poisson noise, Haar L = 4, 50 wavelet-AM iterations, expansions at
{10, 20, 30, 40} (pin P4).  One "step" = one complete reconstruction
(init_state + 50 iterations + 4 tree expansions) with d and I0 resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--algo wam|am]
  python bench.py --impl reference ...    # CPU oracle port on the host cores

Multi-GPU (torchrun, one process per GPU): views are sharded across ranks and
the partial back projections are reduced in fp64 by the library's own NCCL
communicator (2D: fused back projection + all-reduce over NVLink peer memory;
3D: reduce-scatter / own-tile update / all-gather, --view-groups for a view x
z-slab grid); gloo is used only for host plumbing (barrier, unique-id
broadcast, max-over-ranks of the device times).

  python bench.py --config cfg3 --shard 8 [--view-groups 8]
      times rank 0 of an 8-rank grid alone on one GPU (detached shard, joint
      tree replayed) and projects the 8-GPU step with modelled collectives.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wamgpu", choices=["wamgpu", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--algo", default=None, choices=[None, "wam", "am"])
    ap.add_argument("--iters", type=int, default=None, help="override J")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=3, help="iterations in the GPU line's cpu_baseline sample")
    ap.add_argument("--cpu-threads", type=int, default=0, help="host threads of the CPU legs (0 = all)")
    ap.add_argument("--nz", type=int, default=None,
                    help="override the slice count of a 3D config (one z-slab shard of an R-GPU run = nz/R)")
    ap.add_argument("--view-groups", type=int, default=None,
                    help="3D rank grid: Rv view groups x R/Rv z-slab groups (default R: views only; 1 = z-slabs)")
    ap.add_argument("--shard", type=int, default=None,
                    help="N=1: time rank --shard-rank of an R-rank grid ALONE on this GPU (detached shard: "
                         "its views/slab, no exchange) and project the R-GPU step with a modelled all-reduce")
    ap.add_argument("--shard-rank", type=int, default=0)
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Plumbing:
    """Host-side coordination (gloo): barrier, broadcast, max over ranks."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=rank, world_size=world)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def bcast_bytes(self, b: bytes):
        if not self.dist:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def all_gather_bytes(self, b: bytes):
        if not self.dist:
            return [b]
        out = [None] * self.world
        self.dist.all_gather_object(out, b)
        return out

    def max(self, v: float):
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _poll(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _workload_desc(cfg, nnz, algo, J):
    dims = (f"2D fan-beam {cfg['nx']}x{cfg['ny']}" if cfg["nz"] == 1 else
            f"axial 3D stack {cfg['nx']}x{cfg['ny']}x{cfg['nz']} (rays in-plane, one H for all slices, pin P2)")
    return (f"{cfg['name']}: {dims} @ {cfg['voxel']} mm, {cfg['views']} views x "
            f"{cfg['detectors']} arc detectors (SCD 500, SDD 1000), I0={cfg['I0']:g} Poisson, "
            + (f"wavelet AM Haar L={cfg['L']} ({'separable 3D' if cfg['haar'] == 3 and cfg['nz'] > 1 else '2D per slice'}), {J} iterations, expansions {cfg['schedule']} @0.1"
               if algo == "wam" else f"image-domain AM, {J} iterations") + f", nnz(H per slice)={nnz}")


def _inputs(cfg, W, device=0):
    """Seeded phantom + Poisson data from the product's device simulator (the
    same counts as its host simulator, tests/test_gpu_simulate.py)."""
    from paper_1508_04458_b200 import configs
    g = configs.geometry(cfg, W.Geometry)
    mu_true = W.rasterize(g, configs.phantom(cfg))
    M = cfg["views"] * cfg["detectors"]
    I0 = configs.incident(cfg, M)
    d = W.simulate_device(g, mu_true, I0, cfg["seed"], device=device)
    return g, I0, d


def _baseline_metric():
    """BASELINE.json's metric string, printed verbatim by both arms."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "AM iterations/sec and ray-voxel updates/sec at 1/2/4/8 B200 vs HBM roofline"


def _oracle_module():
    """The CPU oracle (test infrastructure: only the CPU legs of this file use
    it), rebuilt with -march=native for the host it runs on when a compiler is
    present (bit-identical results: -ffp-contract=off)."""
    if "ORC_LIB" not in os.environ:
        from oracle import oracle as O0
        nat = O0.build_native(os.path.join("/tmp", f"wamgpu_orc_native_{os.getpid()}"))
        if nat:
            os.environ["ORC_LIB"] = nat
    from oracle import oracle as O
    return O


class CpuSample:
    """A bounded sample of the workload on the host cores: the reference-
    precision oracle port (f64 CSR+CSC, direct signed split), all threads.

    2D: the full problem.  Axial 3D: slices are independent in-plane problems
    (pin P2) and the separable Haar couples only the 2^L slices of a z-block,
    so a sample is the CENTRAL z-block of the stack (2^L slices, 8 for AM) with
    its own seeded Poisson draw; its time per iteration scales by
    nz / nz_sample to the whole stack (every pass is linear in the slice
    count).  Big configs use the slim CSR-only oracle.  step() runs the NEXT
    iteration of the sampled run, with the scheduled expansion after it."""

    def __init__(self, cfg, algo, threads, inputs=None):
        O = _oracle_module()
        from paper_1508_04458_b200 import configs
        self.algo, self.cfg = algo, cfg
        scfg = dict(cfg)
        if cfg["nz"] > 1:
            nzs = (1 << cfg["L"]) if algo == "wam" and cfg["haar"] == 3 else 8
            nzs = min(nzs, cfg["nz"])
            scfg["nz"] = nzs
            inputs = None
            self.scale = cfg["nz"] / nzs
            s0 = (cfg["nz"] - nzs) // 2
            self.what = (f"central z-block (slices {s0}-{s0 + nzs - 1} of {cfg['nz']}) of {cfg['name']}, "
                         f"scaled x{self.scale:g}")
        else:
            self.scale = 1.0
            self.what = f"{cfg['name']} (whole problem)"
        og = O.make_geometry(**configs.geometry(scfg))
        self.slim = cfg["nx"] * cfg["ny"] >= 1 << 20
        t0 = time.perf_counter()
        self.p = O.Problem(og, mirror=False, threads=threads, slim=self.slim)
        self.t_build = time.perf_counter() - t0
        self.nnz = self.p.nnz
        if inputs is None:
            # the phantom of the full stack restricted to the central slices:
            # centred geometries put slice s of the sample at z of slice s0+s
            mu = O.rasterize(og, configs.phantom(cfg))
            I0 = configs.incident(scfg, self.p.M)
            d = self.p.simulate(mu, I0, cfg["seed"])
        else:
            I0, d = inputs
        t0 = time.perf_counter()
        if algo == "wam":
            if scfg["nz"] > 1:
                self.p.set_haar_dim(cfg["haar"])
            self.p.wam_init(d, I0, cfg["L"])
        else:
            self.p.am_init(d, I0)
        self.t_init = time.perf_counter() - t0
        self.done = 0
        self.sched = set(cfg["schedule"]) if algo == "wam" else set()
        self.t_expand = 0.0
        self.label = "native" if os.environ.get("ORC_LIB") else "portable"

    def step(self):
        """One iteration (plus the scheduled expansion after it): seconds."""
        t0 = time.perf_counter()
        if self.algo == "wam":
            self.p.wam_iterate(1)
            self.done += 1
            if self.done in self.sched:
                self.p.wam_expand(0.1)
        else:
            self.p.am_iterate(1)
            self.done += 1
        return time.perf_counter() - t0

    def rate(self, times):
        """iterations/s of the WHOLE workload from per-iteration sample times."""
        return 1.0 / (sum(times) / len(times) * self.scale)

    def sample(self, first, n, threads):
        return (f"{self.algo.upper()} iterations {first}-{first + n - 1} (with their scheduled expansions) of "
                f"the {self.what}; f64 oracle port ({'slim CSR-only' if self.slim else 'CSR+CSC'}, "
                f"direct signed split), {threads} threads, -O3 -ffp-contract=off "
                f"{'-march=native' if self.label == 'native' else '(portable)'}; H build {self.t_build:.1f}s "
                f"and init {self.t_init:.1f}s untimed")


def _lscpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    from paper_1508_04458_b200 import configs
    cfg = configs.get(args.config)
    algo = args.algo or cfg["algo"]
    cores = os.cpu_count() or 1
    threads = args.cpu_threads or cores
    cs = CpuSample(cfg, algo, threads)
    for _ in range(args.warmup):
        cs.step()
    first = cs.done + 1
    times = [cs.step() for _ in range(args.steps)]
    val = cs.rate(times)
    J = cfg["J"]
    line = {
        "impl": "reference", "metric": _baseline_metric(), "value": val,
        "unit": "iterations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / args.steps * cs.scale, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded phantom, Poisson counts)",
        "config": {"workload": _workload_desc(cfg, cs.nnz, algo, J), "threads": threads, "cpu_model": _lscpu(),
                   "step": "one iteration of the sampled run (scaled to the whole stack)"},
        "ray_voxel_updates_per_s": 2 * cs.nnz * cfg["nz"] * val,
        "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": threads, "kind": "port",
                         "sample": cs.sample(first, args.steps, threads), "cpu_model": _lscpu()},
        "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# NCCL all-reduce bus bandwidth of 8 B200 ranks over NVSwitch at 1 GiB
# (/opt/skills/guides/B200_PROFILING.md) and a small-message latency allowance
ALLREDUCE_BUSBW_GBS = 725.0
SMALL_COLLECTIVE_US = 20.0


def _shard_projection(args, cfg, algo, J, part, ctx, ms_step, split_ms_step):
    """Projected R-GPU step of the rank grid from one detached shard timed alone:
    t_R = t_shard + J * (t_collectives of the view group + scalars).
    NCCL times of S total bytes over n ranks at bus bandwidth B: all-reduce
    S*2(n-1)/n/B; reduce-scatter and all-gather S*(n-1)/n/B.  With the split
    update (wamgpu.cu tile_update_split / am_split_update) the view group
    reduce-scatters [g || b-] (fp64) and all-gathers {mu, beta} (fp32); without
    it, it all-reduces [g || b-]."""
    R, Rv = args.shard, part["view_groups"]
    nzl = part["slab_slices"]
    P = 1 if cfg["nz"] == 1 else max(8, 1 << (nzl - 1).bit_length())
    B = ALLREDUCE_BUSBW_GBS * 1e9
    split = (os.environ.get("WAMGPU_VIEW_UPDATE") != "allreduce" and cfg["nz"] > 1 and Rv > 1 and
             ((algo == "am" and cfg["ny"] % Rv == 0) or
              (algo == "wam" and cfg["haar"] == 3 and (cfg["ny"] >> cfg["L"]) % Rv == 0)))
    if Rv == 1:
        S, kind, t_c = 0, "none", 0.0
    elif split:
        ne = ctx.N * (P if algo == "am" else nzl)
        s_rs, s_ag = (8 * ne, 4 * ne) if algo == "am" else (16 * ne, 4 * ne)
        S, kind = s_rs + s_ag, "reduce-scatter [g || b-] fp64 + all-gather mu fp32"
        t_c = (s_rs + s_ag) * (Rv - 1) / Rv / B * 1e3
        if algo == "wam":
            # once per run (wam_run's end, wamgpu.cu sync_beta): the beta
            # planes (fp32) all-gathered; per expansion: the members' marks
            # merged by an fp64 MAX all-reduce over the tree bytes
            nexp = len([x for x in cfg["schedule"] if x < J])
            L = cfg["L"]
            act_bytes = sum((cfg["nx"] >> l) * (cfg["ny"] >> l) * (nzl >> l) for l in range(1, L + 1))
            t_c += (4 * ne * (Rv - 1) / Rv + nexp * 8 * act_bytes * 2 * (Rv - 1) / Rv) / B * 1e3 / J
            kind += "; beta planes once per run; tree MAX per expansion"
            # the g half of the reduce-scatter runs on a side stream during the
            # signed split (wamgpu.cu wam_step): only what the split cannot hide counts
            t_g = 8 * ne * (Rv - 1) / Rv / B * 1e3
            t_c -= min(t_g, split_ms_step / J)
            kind += " (g half overlapped with the split)"
    else:
        S, kind = (2 if algo == "wam" else 1) * 8 * ctx.N * P, "all-reduce [g || b-] fp64"
        t_c = S * 2 * (Rv - 1) / Rv / B * 1e3
    t_small = SMALL_COLLECTIVE_US * 1e-3   # the objective SUM every iteration
    proj = ms_step + J * (t_c + t_small)
    return {"ranks": R, "rank": args.shard_rank, "view_groups": Rv, "z_groups": part["z_groups"],
            "slab": [part["slab_begin"], nzl], "rows": [ctx.row0, ctx.row1], "collective": kind,
            "collective_bytes_per_iter": S, "collective_ms_model": t_c, "small_collective_ms_model": t_small,
            "projected_ms_per_step": proj,
            "model": f"t_shard + J*(NCCL time at {ALLREDUCE_BUSBW_GBS:g} GB/s bus bandwidth + {SMALL_COLLECTIVE_US:g} us)",
            "note": "detached shard: this rank's views and slab timed alone on one B200, replaying the "
                    "joint reconstruction's tree at each scheduled expansion (criterion still computed)"}


def _joint_trees(W, cfg, g, I0, d, device, sched):
    """Trees after each scheduled expansion of the unsharded run on this GPU."""
    c = W.Context(device)
    c.set_geometry(g)
    if cfg["nz"] > 1:
        c.set_haar_dim(cfg["haar"])
    c.set_data(d, I0)
    c.wam_init(cfg["L"])
    trees, done = [], 0
    for ev in sched:
        c.wam_iterate(ev - done)
        done = ev
        c.wam_expand(0.1)
        trees.append(c.tree())
    c.close()
    return trees


def _slab_tree(tree, cfg, s0, nzl):
    """z-slab [s0, s0+nzl) of a separable-3D tree (level l: (nz>>l, ny>>l, nx>>l))."""
    out, o = [], 0
    for l in range(1, cfg["L"] + 1):
        nb = (cfg["nx"] >> l) * (cfg["ny"] >> l)
        lv = tree[o:o + nb * (cfg["nz"] >> l)].reshape(cfg["nz"] >> l, nb)
        out.append(lv[s0 >> l:(s0 + nzl) >> l].ravel())
        o += nb * (cfg["nz"] >> l)
    return np.concatenate(out)


def _parity_pass(ctx, cfg):
    """Stepwise run (iterate / expand) hashing the tree after each scheduled
    expansion; compared with tests/golden/big_<cfg>.json when present."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", f"big_{cfg['name']}.json")
    fx = None
    if os.path.exists(path):
        with open(path) as f:
            fx = json.load(f)
    ctx.wam_init(cfg["L"])
    out = {"fixture": os.path.relpath(path, ROOT) if fx else None, "expansions": []}
    z0_init = ctx.scalars()["Z0"]
    done = 0
    for k, ev in enumerate(cfg["schedule"]):
        ctx.wam_iterate(ev - done)
        done = ev
        n = ctx.wam_expand(0.1)
        sha = hashlib.sha256(np.ascontiguousarray(ctx.tree()).tobytes()).hexdigest()
        e = {"after_iter": ev, "newly": n, "tree_sha256": sha, "Z0": ctx.scalars()["Z0"]}
        if fx and k < len(fx["oracles"]["mirror"]["expansions"]):
            m = fx["oracles"]["mirror"]["expansions"][k]
            e["mirror_oracle_match"] = (m["tree_sha256"] == sha and m["newly"] == n and
                                        float.fromhex(m["Z0"]) == e["Z0"])
            f64 = fx["oracles"].get("f64")
            if f64:
                e["f64_oracle_tree_match"] = f64["expansions"][k]["tree_sha256"] == sha
        out["expansions"].append(e)
    if fx:
        out["Z0_init_mirror_match"] = float.fromhex(fx["oracles"]["mirror"]["Z0_init"]) == z0_init
        out["fixture_iterations"] = fx["J"]
    return out


def _sum_timing(ts):
    out = dict(ts[0])
    for t in ts[1:]:
        for k, v in t.items():
            if k != "split_nnz":
                out[k] += v
    out["split_nnz"] = ts[-1]["split_nnz"]
    return out


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = _dist()
    import paper_1508_04458_b200 as W
    from paper_1508_04458_b200 import configs
    cfg = configs.get(args.config)
    if args.nz:
        if cfg["nz"] == 1:
            raise SystemExit("--nz applies to 3D configs only")
        cfg["nz"] = args.nz
        cfg["name"] += f" (nz override {args.nz}: one z-slab shard)"
    algo = args.algo or cfg["algo"]
    J = args.iters or cfg["J"]
    sched = [s for s in cfg["schedule"] if s < J] if algo == "wam" else []
    plumb = Plumbing(rank, world)

    g, I0, d = _inputs(cfg, W, local)
    joint_trees = None
    if args.shard and algo == "wam":
        # the joint reconstruction's trees (the R-rank run reproduces the
        # unsharded tree bit-exactly, tests/test_gpu_sharded3d.py): the shard
        # replays them instead of growing its own from partial data
        joint_trees = _joint_trees(W, cfg, g, I0, d, local, sched)
    ctx = W.Context(local)
    if world > 1:
        uid = plumb.bcast_bytes(W.nccl_unique_id() if rank == 0 else b"")
        ctx.set_comm(uid, rank, world)
    elif args.shard:
        ctx.set_comm_local(-1, args.shard_rank, args.shard)
    if cfg["nz"] > 1:
        # 3D default: every rank a view group of its own (pure view sharding):
        # measured best at every R (profiles/shard/r03/TABLE.md)
        ctx.set_partition(args.view_groups or max(world, args.shard or 1))
    ctx.set_geometry(g)
    part = ctx.partition()
    collective = "none" if world == 1 else "nccl"
    if world > 1 and cfg["nz"] == 1 and os.environ.get("WAMGPU_P2P", "1") != "0":
        # fused back projection + all-reduce over NVLink peer memory: exchange
        # the CUDA IPC handles over the host plumbing
        try:
            blobs = plumb.all_gather_bytes(ctx.p2p_export())
            collective = "fused-p2p" if ctx.p2p_import(b"".join(blobs)) else "nccl (p2p self-check failed)"
        except Exception as e:  # no peer access: stay on NCCL
            collective = f"nccl (p2p unavailable: {e})"
    if cfg["nz"] > 1 and algo == "wam":
        ctx.set_haar_dim(cfg["haar"])
    ctx.set_data(d, I0)
    nnz_local = ctx.nnz

    if joint_trees is not None and cfg["nz"] > 1 and cfg["haar"] == 3:
        joint_trees = [_slab_tree(t, cfg, part["slab_begin"], part["slab_slices"]) for t in joint_trees]

    def step_device():
        if algo == "wam" and joint_trees is not None:   # shard: replay the joint tree
            ctx.wam_init(cfg["L"])
            t_init = ctx.timing()
            recs, tms, done = [], [], 0
            for k, ev in enumerate(sched + [J]):
                recs += ctx.wam_iterate(ev - done)
                tms.append(ctx.timing())
                done = ev
                if ev == J:
                    break
                ctx.wam_expand(float("inf"), add_tree=joint_trees[k])
                tms.append(ctx.timing())
            return t_init, _sum_timing(tms), recs
        if algo == "wam":
            ctx.wam_init(cfg["L"])
            t_init = ctx.timing()
            recs = ctx.wam_run(J, sched, 0.1)
        else:
            ctx.am_init()
            t_init = ctx.timing()
            recs = ctx.am_iterate(J)
        t_run = ctx.timing()
        return t_init, t_run, recs

    # ---- untimed parity pass: the tree after every scheduled expansion (and
    # Z0) against the committed oracle fixture of this config, when there is one
    # (tests/golden/big_<cfg>.json; bit-exact vs the fp32-mirror oracle)
    parity = None
    if algo == "wam" and world == 1 and not args.shard and not args.nz and J == cfg["J"]:
        parity = _parity_pass(ctx, cfg)

    for _ in range(args.warmup):
        step_device()

    # ---- timed region (device clock via the library's CUDA events)
    ctx.set_kernel_timing(True)
    dev_ms, fwd_ms, back_ms, launches = [], [], [], 0
    fwd_n = back_n = 0
    split_ms = upd_ms = exp_ms = comm_ms = phi_ms = cfwd_ms = cback_ms = 0.0
    phi_n = cfwd_n = cback_n = proj_updates = split_n = split_entries = 0
    split_nnz = 0
    plumb.barrier()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            ti, tr, recs = step_device()
            dev_ms.append(ti["total_ms"] + tr["total_ms"])
            for t in (ti, tr):
                fwd_ms.append(t["fwd_ms"])
                back_ms.append(t["back_ms"])
                fwd_n += t["fwd_launches"]
                back_n += t["back_launches"]
                launches += t["kernel_launches"]
                split_ms += t["split_ms"]
                upd_ms += t["update_ms"]
                exp_ms += t["expand_ms"]
                comm_ms += t["comm_ms"]
                phi_ms += t["phi_ms"]
                phi_n += t["phi_launches"]
                cfwd_ms += t["coarse_fwd_ms"]
                cback_ms += t["coarse_back_ms"]
                cfwd_n += t["coarse_fwd_launches"]
                cback_n += t["coarse_back_launches"]
                proj_updates += t["proj_updates"]
                split_n += t["split_launches"]
                split_entries += t["split_entries"]
                split_nnz = t["split_nnz"]
        wall = time.perf_counter() - t_wall
    plumb.barrier()
    ms_step = plumb.max(sum(dev_ms) / len(dev_ms))
    final_obj = recs[-1]["objective"]
    ctx.set_kernel_timing(False)

    # ---- end-to-end through the C-ABI with host buffers (H2D d, I0; D2H mu)
    plumb.barrier()
    t0 = time.perf_counter()
    # (at most 5 steps: a cfg4 step is ~8 s; the kernels are the device-timed ones above)
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        ctx.set_data(d, I0)
        step_device()
        img = ctx.image()
    e2e_s = plumb.max((time.perf_counter() - t0) / e2e_steps)
    Ml = ctx.row1 - ctx.row0
    nz = cfg["nz"]
    h2d = 2 * 4 * Ml * nz
    d2h = 4 * img.size

    iters_per_s = J / (ms_step * 1e-3)
    dev_mem = None
    try:
        import torch
        ctx_sms = torch.cuda.get_device_properties(local).multi_processor_count
    except Exception:
        ctx_sms = 148
    try:   # NVML, not torch: libwamgpu has the system NCCL loaded, torch's CUDA library wants its own
        import pynvml
        pynvml.nvmlInit()
        mi = pynvml.nvmlDeviceGetMemoryInfo(pynvml.nvmlDeviceGetHandleByIndex(local))
        dev_mem = {"used": round(mi.used / 2**30, 1), "total": round(mi.total / 2**30, 1)}
    except Exception as e:
        dev_mem = {"error": str(e)[:120]}
    line = None
    if rank == 0:
        hbm, peak_kind = _peaks()
        M, N = ctx.M, ctx.N
        nnz = nnz_local * world  # approximately equal shards; exact total below on N=1
        nnz = nnz_local if world == 1 else nnz
        if nz == 1:
            fwd_bytes = 8 * nnz_local + 4 * (Ml + 1) + 4 * N + 12 * Ml
            back_bytes = 8 * nnz_local + 4 * (N + 1) + 4 * Ml + 4 * N
        else:
            # slab kernels read H once per pass for all nz slices: the minimal
            # HBM traffic is H + the slab vectors; the 4 B/update SURVEY figure
            # (SURVEY.md §8(d) K2'/K3') is served from L1/L2 and reported as
            # gather_gbs
            fwd_bytes = 8 * nnz_local + 4 * (Ml + 1) + 4 * N * nz + 12 * Ml * nz
            back_bytes = 8 * nnz_local + 4 * (N + 1) + 4 * Ml * nz + 16 * N * nz
        fwd_avg = sum(fwd_ms) / max(fwd_n, 1)
        back_avg = sum(back_ms) / max(back_n, 1)
        fwd_gbs = fwd_bytes / (fwd_avg * 1e-3) / 1e9
        back_gbs = back_bytes / (back_avg * 1e-3) / 1e9
        fwd_name = ("k_fwd_patch<1,4,8,5> (K2 CSR forward + Beer + I-div, 4 rays/warp)" if nz == 1 else
                    "k_fwd3s / k_fwd3s_band<1,...> (K2' slab forward over the in-plane matrix + Beer + I-div; "
                    "banded when the mu slab exceeds L2)")
        back_name = ("k_back<0,12,1> (K3 CSC back projection)" if nz == 1 and algo == "wam" else
                     "k_back<1,12,1> (K3 CSC back projection + AM update)" if nz == 1 else
                     "k_back3s<...> (K3' slab back projection over the in-plane CSC)")
        dom = fwd_name if sum(fwd_ms) >= sum(back_ms) else back_name
        ach = fwd_gbs if sum(fwd_ms) >= sum(back_ms) else back_gbs
        dom_bytes = fwd_bytes if sum(fwd_ms) >= sum(back_ms) else back_bytes
        # 3D: with the block-coarsened projections the signed split can be the
        # largest phase.  Its algorithmic HBM bytes per launch: the Psi stream
        # (20 B per entry: ray + four fp32 psi), the q slab once and the 7
        # coefficient planes it writes; the q-row gathers (P x 4 B per entry)
        # are served by L2 and reported as the binding resource.
        split_dom = nz > 1 and split_n > 0 and split_ms > max(sum(fwd_ms), sum(back_ms))
        if split_dom:
            split_avg = split_ms / split_n
            ent_avg = split_entries / split_n
            P_slab = 8
            while P_slab < nz:
                P_slab *= 2
            split_bytes = 20 * ent_avg + 4 * Ml * nz + 8 * N * nz
            dom = ("k_split3c<P,E,true,4,1,4> (signed split b- over the Psi lists of the separable 3D Haar tree; "
                   "averaged over the launches of a run, the tree grows at every expansion)")
            ach = split_bytes / (split_avg * 1e-3) / 1e9
            dom_bytes = split_bytes
        traffic = None
        traffic_note = "GB per launch, ncu dram read+write (profiles/dram_traffic.json)"
        try:
            with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as f:
                tr = json.load(f)
            traffic = tr.get(cfg["name"], {}).get("k_split3c_final_tree" if split_dom else
                                                   "k_forward" if "forward" in dom else "k_back")
            if split_dom and traffic is not None:
                # one capture exists, of the LARGEST launch of a run (final tree); `achieved` above
                # averages over a run's launches, so compare this with the final tree's own bytes
                traffic_note = ("GB, ncu dram read+write of the final-tree launch (8.67e8 Psi entries, 19.2 GB "
                                "algorithmic for THAT launch: 2.8x, q rows re-fetched from DRAM when the "
                                "slab falls out of L2); profiles/r07/ncu_split3c_cfg4_chunk.txt")
        except Exception:
            pass
        # 3D: the slab passes are not HBM-bound (one DFMA + one fp32->fp64
        # conversion per ray-voxel update from L1/L2-resident slabs, DESIGN.md
        # §4.2): also report the dominant pass against the fp64-FMA issue peak
        # (64 DFMA lanes per clock per SM at the SM clock sampled under load)
        binding = None
        clocks = clk.summary()
        if split_dom:
            gather = ent_avg * P_slab * 4 / (split_avg * 1e-3)
            # not measured live: the issue-slot utilisation of the committed ncu capture of the
            # final-tree launch (profiles/r07/ncu_split3c_cfg4_chunk.txt: issue 61.7%, fp64 pipe
            # 34.9%, L2 31.6%, DRAM 10.4%); achieved = Psi entries per second of this run
            binding = {"resource": "instruction issue (per Psi entry and 128 slices: 2 cp.async + 2 LDS.128 per lane, "
                                   "8 conversions, 4 adds, 32 DFMAs per lane at level 1; q-row gathers served by L2)",
                       "achieved": ent_avg / (split_avg * 1e-3), "unit": "Psi entries/s", "peak": None,
                       "frac": 0.617, "frac_source": "ncu smsp__issue_active of the final-tree launch (committed "
                                                     "capture, not this run)",
                       "q_gather_gbs_from_l2": gather / 1e9,
                       "evidence": "profiles/r07/ncu_split3c_cfg4_chunk.txt"}
        elif nz > 1:
            mhz = clocks.get("sm_mhz") or 1965.0
            dom_ms = fwd_avg if sum(fwd_ms) >= sum(back_ms) else back_avg
            upd = nnz_local * nz / (dom_ms * 1e-3)
            peak_upd = ctx_sms * 64 * mhz * 1e6
            binding = {"resource": "fp64 FMA issue (one DFMA + one fp32->fp64 conversion per ray-voxel update; "
                                   "slab gathers served by L1/L2)",
                       "achieved": upd, "peak": peak_upd, "unit": "ray-voxel updates/s", "frac": upd / peak_upd,
                       "updates_per_clk_per_sm": upd / (ctx_sms * mhz * 1e6),
                       "evidence": "profiles/r06/ncu_cfg4_pass.txt (issue, XU, fp64, L1/L2 shares of the banded "
                                   "forward, the back projection and the split)"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.shard:
            try:
                threads = args.cpu_threads or os.cpu_count() or 1
                cs = CpuSample(cfg, algo, threads, inputs=(I0, d) if cfg["nz"] == 1 else None)
                ts = [cs.step() for _ in range(args.cpu_iters)]
                cpu = {"value": cs.rate(ts), "unit": "iterations/s", "cores": threads, "kind": "port",
                       "sample": cs.sample(1, args.cpu_iters, threads), "cpu_model": _lscpu()}
                del cs
            except Exception as e:  # the baseline is reported, never the target
                cpu = {"value": None, "unit": "iterations/s", "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {e}"}
        line = {
            "metric": _baseline_metric(),
            "value": iters_per_s, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 storage / f64 accumulation",
            "data": "synthetic (seeded luggage phantom, seeded Poisson counts; product device simulator)",
            "config": {"workload": _workload_desc(cfg, nnz, algo, J), "step": "init_state + run (all iterations"
                       " and expansions)", "l2": "working set (H CSR+CSC = 16 B/nnz) >> 126 MB L2; no flush needed",
                       "parallelism": (f"views/{world}" if cfg["nz"] == 1 else
                                       f"views/{part['view_groups']} x z-slabs/{part['z_groups']}"),
                       "collective": collective},
            # H passes only (forward + back launches; a 3D launch covers every
            # slice): the root-only iterations run over the approximation
            # columns Phi_A instead of H and are counted apart
            # (updates actually executed: the library counts entries streamed x slices
            # processed for every forward / back launch, H or a block-coarsened Hc)
            "ray_voxel_updates_per_s": proj_updates * world / args.steps / (ms_step * 1e-3),
            "h_passes_per_step": (fwd_n + back_n) / args.steps,
            "coarse_passes_per_step": (cfwd_n + cback_n) / args.steps,
            "pixel_equivalent_updates_per_s": (fwd_n + back_n + cfwd_n + cback_n) / args.steps * nnz * nz
                                              / (ms_step * 1e-3),
            "final_objective": final_obj,
            "device_memory_gib": dev_mem,   # after the timed steps: matrices (H, coarsened Hc), Psi lists, slabs
            "tree": {"active_set_by_iteration": sorted({r["active_set"] for r in recs}),
                     "coefficients": N * nz, "phi_minus_nnz": split_nnz},
            "parity": parity,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                         "traffic_note": traffic_note if traffic is not None else None,
                         "algorithmic_bytes": dom_bytes,
                         "binding": binding},
            "kernels": {"fwd_avg_ms": fwd_avg, "fwd_gbs": fwd_gbs, "fwd_frac": fwd_gbs / hbm,
                        "gather_gbs": (4 * nnz_local * nz / (fwd_avg * 1e-3) / 1e9) if nz > 1 else None,
                        "back_avg_ms": back_avg, "back_gbs": back_gbs, "back_frac": back_gbs / hbm,
                        "per_step_ms": {"forward": sum(fwd_ms) / args.steps, "back": sum(back_ms) / args.steps,
                                        "forward_coarse": cfwd_ms / args.steps, "back_coarse": cback_ms / args.steps,
                                        "split": split_ms / args.steps, "update": upd_ms / args.steps,
                                        "expand": exp_ms / args.steps, "comm": comm_ms / args.steps,
                                        "phi_a": phi_ms / args.steps},
                        "phi_a_iterations_per_step": phi_n / args.steps},
            "e2e": {"value": J / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clocks,
            "wall_s_timed": wall,
            "cpu_baseline": cpu,
        }
        if args.shard:
            line["shard"] = _shard_projection(args, cfg, algo, J, part, ctx, ms_step, split_ms / args.steps)
        print(json.dumps(line), flush=True)
    ctx.close()
    plumb.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
