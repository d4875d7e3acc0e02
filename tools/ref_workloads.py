"""The reference's own CPU path (oracle/_ref: the unmodified reference compiled
behind its facet-soup adapter) timed on this host's cores for every subsystem
the GPU workloads cover (tools/workloads.py). Calls fan out over a thread pool
(ctypes releases the GIL; the reference's per-snapshot functions are
re-entrant, and build_matrix / occlusion batches use VISRT_THREADS workers).
Long stages run on a seeded sample and are extrapolated linearly by the
unit count, labelled "extrapolated". Checker/baseline only: nothing here is
on the product path.

usage: python tools/ref_workloads.py [cfg ...] > ref_workloads.jsonl"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import bindings  # noqa: E402
from paper_2501_02747_b200 import scenes  # noqa: E402

CORES = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
os.environ.setdefault("VISRT_THREADS", str(CORES))


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def pool_map(fn, items):
    with ThreadPoolExecutor(CORES) as ex:
        return list(ex.map(fn, items))


def regions(r, src, faces):
    """illuminated_region for every (source, face) of the lists."""
    tasks = [(k, f) for k in range(len(src)) for f in faces]
    _, dt = timed(lambda: pool_map(lambda t: r.illuminated_region(src[t[0]], t[1]), tasks))
    return len(tasks), dt


def run(cfg: int) -> dict:
    wl = scenes.workload(cfg)
    soup = wl.scene
    n = soup.nfaces
    r = bindings.RefOracle(soup)
    out = {"config": cfg, "facets": n, "cores": CORES, "kind": "reference"}
    rng = np.random.default_rng(cfg)
    if cfg in (1, 2, 3):
        m1, dt = timed(lambda: r.build_matrix(1))
        out["matrix_A_s"] = round(dt, 3)
    if cfg == 1:
        m2, dt = timed(lambda: r.build_matrix(2))
        out["matrix_order2_s"] = round(dt, 3)
        src = np.concatenate([wl.tx, wl.rx])
        _, dt = timed(lambda: pool_map(lambda p: r.point_vis_table(m1, p, 1), list(src)))
        out["tables_order1_s"] = round(dt, 3)
        cnt, dt = regions(r, src, range(n))
        out["regions_s"] = round(dt, 3)
        acc = r.accel(m2, 2)
        _, dt = timed(lambda: pool_map(lambda k: r.trace(acc, wl.tx[k], wl.rx[0]), range(len(wl.tx))))
        out["trees_order2_s"] = round(dt, 3)
    if cfg in (3, 5):
        # per-facet regions: a seeded sample of (source, facet) pairs, extrapolated to every pair
        nsrc = 8 if cfg == 3 else 4
        nf = 500 if cfg == 3 else 300
        src = np.concatenate([wl.tx[rng.choice(len(wl.tx), nsrc // 2, replace=False)],
                              wl.rx[rng.choice(len(wl.rx), nsrc // 2, replace=False)]])
        faces = sorted(rng.choice(n, nf, replace=False).tolist())
        cnt, dt = regions(r, src, faces)
        total = (len(wl.tx) + len(wl.rx)) * n
        out["regions_sample"] = f"{cnt} seeded (source, facet) pairs, {nsrc} sources x {nf} facets"
        out["regions_sample_s"] = round(dt, 3)
        out["regions_s_extrapolated"] = round(dt * total / cnt, 1)
    if cfg == 3:
        # order-1 point_vis_table rows for 20 of the 2,000 snapshot sources, extrapolated
        sel = np.concatenate([wl.tx[rng.choice(len(wl.tx), 10, replace=False)],
                              wl.rx[rng.choice(len(wl.rx), 10, replace=False)]])
        _, dt = timed(lambda: pool_map(lambda p: r.point_vis_table(m1, p, 1), list(sel)))
        out["tables_order1_sample"] = "20 seeded sources"
        out["tables_order1_s_extrapolated"] = round(dt * (len(wl.tx) + len(wl.rx)) / len(sel), 1)
    if cfg in (2, 3, 4):
        # (B) all-pairs verdicts: seeded pair sample, extrapolated by T_alg share (pairs are i.i.d.)
        m = 20000 if cfg != 4 else 2000
        i = rng.integers(0, n, 2 * m)
        j = rng.integers(0, n, 2 * m)
        keep = i != j
        pi, pj = np.minimum(i, j)[keep][:m].astype(np.int32), np.maximum(i, j)[keep][:m].astype(np.int32)
        _, dt = timed(lambda: r.occlusion_batch(pi, pj, threads=CORES))
        out["matrix_B_sample"] = f"{len(pi)} seeded pairs"
        out["matrix_B_s_extrapolated"] = round(dt * (n * (n - 1) / 2) / len(pi), 1)
    return out


def all_pairs(n):
    i, j = np.triu_indices(n, 1)
    return i.astype(np.int32), j.astype(np.int32)


def run_full(cfg: int) -> dict:
    """r02: the stages SURVEY.md section 8(d) calls feasible, run IN FULL (or on the stated large
    sample) instead of extrapolated from a few hundred units: config 2 / 3 (B) on every pair,
    config 4 (A) = build_matrix(scene, 1), config-3 regions and order-1 tables for 200 of the
    2,000 sources x every facet, config-3 order-3 traces for 100 snapshots and config-5 order-3
    traces for every snapshot (both after the reference's own build_matrix(scene, 2))."""
    wl = scenes.workload(cfg)
    soup = wl.scene
    n = soup.nfaces
    r = bindings.RefOracle(soup)
    out = {"config": cfg, "facets": n, "cores": CORES, "kind": "reference", "mode": "full"}
    rng = np.random.default_rng(100 + cfg)
    if cfg in (2, 3):
        pi, pj = all_pairs(n)
        _, dt = timed(lambda: r.occlusion_batch(pi, pj, threads=CORES))
        out["matrix_B_pairs"] = len(pi)
        out["matrix_B_s"] = round(dt, 2)
    if cfg in (3, 4):
        m1, dt = timed(lambda: r.build_matrix(1))
        out["matrix_A_s"] = round(dt, 2)
    if cfg == 3:
        sel = np.concatenate([wl.tx[::10], wl.rx[::10]])   # 200 of the 2,000 sources
        _, dt = timed(lambda: pool_map(lambda p: r.point_vis_table(m1, p, 1), list(sel)))
        out["tables_order1_sources"] = len(sel)
        out["tables_order1_s"] = round(dt, 2)
        face = np.tile(np.arange(n, dtype=np.int32), len(sel))
        src = np.repeat(sel, n, axis=0)
        arr = (bindings.vref_region * len(face))()   # the C call alone (no per-record Python objects)
        flat = np.ascontiguousarray(src, np.float64).reshape(-1)
        _, dt = timed(lambda: r.lib().vref_regions_batch(r.h, len(face), flat, face, arr, CORES))
        out["regions_sources"] = len(sel)
        out["regions"] = int(len(face))
        out["regions_s"] = round(dt, 2)
    if cfg in (3, 5):
        m2, dt = timed(lambda: r.build_matrix(2))
        out["matrix_order2_s"] = round(dt, 2)
        r.lib().vref_matrix_set_max_order(m2, 3)
        acc = r.accel(m2, 3)
        ks = list(range(0, len(wl.tx), 10)) if cfg == 3 else list(range(len(wl.tx)))
        res, dt = timed(lambda: pool_map(lambda k: r.trace(acc, wl.tx[k], wl.rx[k])[1][0], ks))
        out["trees_order3_snapshots"] = len(ks)
        out["trees_order3_s"] = round(dt, 2)
        out["trees_order3_nodes"] = int(np.sum(res))
    return out


if __name__ == "__main__":
    if not bindings.have_ref():
        bindings.build(ref=True)
    args = [a for a in sys.argv[1:] if a != "--full"]
    fn = run_full if "--full" in sys.argv[1:] else run
    for c in [int(a) for a in args] or [1, 2, 3, 4, 5]:
        print(json.dumps(fn(c)), flush=True)
