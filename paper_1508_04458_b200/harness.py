"""Harness outputs around the AM iteration:

* ConvergenceRecord CSV logs: iteration, objective,
  elapsed_s, active_set, cum_updates -- written from the records the C-ABI
  returns (wamgpu_record, include/wamgpu.h);
* the active-tree text manifest ("one line per active
  coefficient: z-slice, level, subband, i, j"), from the tree bytes of
  wamgpu_get_tree and back, so a run can resume its tree through
  wamgpu_wam_expand_with (Context.wam_expand(inf, add_tree=...));
* compare_runs(log_a, log_b, image_a, image_b):
  matched-objective crossing analysis, difference image, RMSE vs truth.

Pure host code over numpy; nothing here is on the device path.
"""
from __future__ import annotations

import csv
import io

import numpy as np

RECORD_FIELDS = ("iter", "objective", "elapsed_s", "active_set", "cum_updates")
SUB2D = ("h", "v", "d")                 # detail subbands of a 2D block (approximation: "a")
SUB3D = ("llh", "lhl", "lhh", "hll", "hlh", "hhl", "hhh")   # (z, y, x) low/high of a 3D block


# ------------------------------------------------------------ ConvergenceRecord CSV
def write_records_csv(path_or_file, records, with_time=True):
    """One row per iteration; with_time=False drops the timing column (the
    SPEC's determinism contract compares logs 'timing column excepted')."""
    fields = [f for f in RECORD_FIELDS if with_time or f != "elapsed_s"]
    own = isinstance(path_or_file, str)
    f = open(path_or_file, "w", newline="") if own else path_or_file
    try:
        w = csv.writer(f)
        w.writerow(fields)
        last = 0
        for r in records:
            if r["iter"] <= last:
                raise ValueError("ConvergenceRecord: iteration must be strictly increasing")
            last = r["iter"]
            w.writerow([repr(float(r[k])) if k in ("objective", "elapsed_s") else int(r[k]) for k in fields])
    finally:
        if own:
            f.close()


def read_records_csv(path_or_file):
    own = isinstance(path_or_file, str)
    f = open(path_or_file, newline="") if own else path_or_file
    try:
        rows = list(csv.DictReader(f))
    finally:
        if own:
            f.close()
    out = []
    for r in rows:
        out.append({k: (float(v) if k in ("objective", "elapsed_s") else int(v)) for k, v in r.items()})
    return out


# ------------------------------------------------------------ tree manifest
def _levels(nx, ny, nz, L, haar):
    """(level, z-count, rows, cols) of the tree bytes, in wamgpu_get_tree order."""
    for l in range(1, L + 1):
        yield l, (nz >> l) if haar == 3 else 1, ny >> l, nx >> l


def tree_manifest(tree, nx, ny, nz, L, haar=2, with_approx=True):
    """Text manifest of an active tree: one line 'z level subband i j' per active
    coefficient.  2D model (haar=2): the tree is shared by every slice, z is
    the slice, subbands a/h/v/d.  Separable 3D model (haar=3): z is the
    z-block index at that level, subbands are the 7 (z, y, x) high/low
    combinations (the approximation 'lll' at level L)."""
    tree = np.asarray(tree, np.uint8)
    out = io.StringIO()
    zs = range(nz) if haar != 3 else None
    if with_approx:
        if haar == 3:
            for k in range(nz >> L):
                for i in range(ny >> L):
                    for j in range(nx >> L):
                        out.write(f"{k} {L} lll {i} {j}\n")
        else:
            for z in zs:
                for i in range(ny >> L):
                    for j in range(nx >> L):
                        out.write(f"{z} {L} a {i} {j}\n")
    o = 0
    for l, nk, h, w in _levels(nx, ny, nz, L, haar):
        lv = tree[o:o + nk * h * w].reshape(nk, h, w)
        o += nk * h * w
        ks, iis, jjs = np.nonzero(lv)
        if haar == 3:
            for k, i, j in zip(ks, iis, jjs):
                for sb in SUB3D:
                    out.write(f"{k} {l} {sb} {i} {j}\n")
        else:
            for z in zs:
                for i, j in zip(iis, jjs):
                    for sb in SUB2D:
                        out.write(f"{z} {l} {sb} {i} {j}\n")
    if o != tree.size:
        raise ValueError("tree size does not match the grid")
    return out.getvalue()


def parse_manifest(text, nx, ny, nz, L, haar=2):
    """Tree bytes (wamgpu_get_tree layout) from a manifest.  A block is active
    when its detail subbands are listed (all of them, and for the 2D model on
    every slice, since the tree is shared); the parent closure is checked."""
    sizes = [(l, nk, h, w) for l, nk, h, w in _levels(nx, ny, nz, L, haar)]
    offs, o = {}, 0
    for l, nk, h, w in sizes:
        offs[l] = o
        o += nk * h * w
    tree = np.zeros(o, np.uint8)
    seen = {}
    need = len(SUB3D) if haar == 3 else len(SUB2D) * nz
    for ln, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        parts = line.split()
        if len(parts) != 5:
            raise ValueError(f"manifest line {ln}: expected 'z level subband i j'")
        z, l, sb, i, j = int(parts[0]), int(parts[1]), parts[2], int(parts[3]), int(parts[4])
        if sb in ("a", "lll"):
            continue
        if not 1 <= l <= L or sb not in (SUB3D if haar == 3 else SUB2D):
            raise ValueError(f"manifest line {ln}: bad level/subband")
        _, nk, h, w = sizes[l - 1]
        k = z if haar == 3 else 0
        if not (0 <= k < nk and 0 <= i < h and 0 <= j < w and 0 <= z < (nk if haar == 3 else nz)):
            raise ValueError(f"manifest line {ln}: index out of range")
        key = (l, k, i, j)
        seen[key] = seen.get(key, 0) + 1
    for (l, k, i, j), n in seen.items():
        if n != need:
            raise ValueError(f"manifest: block (level {l}, {k}, {i}, {j}) lists {n} of {need} coefficients")
        _, nk, h, w = sizes[l - 1]
        tree[offs[l] + (k * h + i) * w + j] = 1
    # closure: a level-l block (l < L) needs its parent at level l+1
    for (l, k, i, j) in seen:
        if l < L:
            _, nk1, h1, w1 = sizes[l]
            kp = k >> 1 if haar == 3 else 0
            if not tree[offs[l + 1] + (kp * h1 + (i >> 1)) * w1 + (j >> 1)]:
                raise ValueError(f"manifest: block (level {l}, {k}, {i}, {j}) has no active parent")
    return tree


# ------------------------------------------------------------ compare_runs
def compare_runs(log_a, log_b, image_a, image_b, truth=None):
    """SPEC.md:446-453.  For the lower of the two final objectives, the first
    iteration / time at which each run reaches it; the difference image
    image_b - image_a; RMSE of each image against the ground truth."""
    a, b = list(log_a), list(log_b)
    ia, ib = np.asarray(image_a, np.float64), np.asarray(image_b, np.float64)
    if ia.shape != ib.shape or (truth is not None and np.asarray(truth).shape != ia.shape):
        raise ValueError("compare_runs: mismatched problem dimensions")
    target = min(a[-1]["objective"], b[-1]["objective"])

    def crossing(log):
        for r in log:
            if r["objective"] <= target:
                return {"iter": r["iter"], "elapsed_s": r["elapsed_s"]}
        return None

    rep = {"target_objective": target, "a": crossing(a), "b": crossing(b), "difference": ib - ia}
    if truth is not None:
        t = np.asarray(truth, np.float64)
        rep["rmse_a"] = float(np.sqrt(np.mean((ia - t) ** 2)))
        rep["rmse_b"] = float(np.sqrt(np.mean((ib - t) ** 2)))
    return rep
