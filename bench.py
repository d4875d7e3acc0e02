#!/usr/bin/env python
"""bench.py — headline benchmark (driver contract).

Workload (BASELINE.json configs[3], "large irregular city" — the largest
configuration that runs on one GPU): the full N x N bit-packed
inter-visibility matrix of a seeded 4 km city of 2,000 convex prisms on 32x32
ground tiles (N = 22,096 facets, 244,105,560 unordered pairs), (B)
semantics: bit(i,j) = occlusion_judgment(F_i, F_j).kind != Occluded, every
pair tested against every other facet as occluder.
``--config 2`` runs the round-1 headline (config 2, N = 1,256) instead.

metric: facet-pair occlusion tests/s = T_alg / t, T_alg = sum_{i<j} S(i,j)(N-2)
(the segment-vs-facet tests the reference's occlusion_judgment performs),
t = device time of one matrix build (CUDA events on the launching stream).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl visrt|reference]

N > 1 runs under torchrun, one rank per GPU, each rank building the matrix of
its own seeded city (independent objects: weak scaling, no data-path
collective); value = all ranks' tests / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "facet-pair occlusion tests/sec; inter-visibility matrix build ms (1 B200)"
UNIT = "tests/s"
FLOPS_PER_TEST = 17.0   # FP64 ops of the mandatory reject path


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _ncores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _sample_pairs(n: int, count: int, seed: int):
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n, count * 2)
    j = rng.integers(0, n, count * 2)
    keep = i != j
    i, j = i[keep][:count], j[keep][:count]
    return np.minimum(i, j).astype(np.int32), np.maximum(i, j).astype(np.int32)


def _sightlines(soup):
    nv = np.diff(soup.vert_off).astype(np.int64)
    ns = nv + 1 + np.where(nv == 4, 16, 3 * nv)
    return nv, ns


def _t_alg(soup, pi, pj) -> float:
    nv, ns = _sightlines(soup)
    gr, ga = ns[pi] - nv[pi] - 1, ns[pj] - nv[pj] - 1
    S = nv[pi] * nv[pj] + 1 + np.minimum(gr, ga)
    return float(S.sum()) * (soup.nfaces - 2)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        rows = []
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                if int(f[0]) != self.index:
                    continue
                rows.append((float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, r in rows for k in range(4) if r[k].lower().startswith("active")})
        loaded = [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for l in f:
                if l.startswith("model name"):
                    return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _pairs_per_core(cfg: int) -> int:
    """Pairs per host thread per reference step: ~0.5-1 s of occlusion_judgment
    (a config-4 pair costs ~22 ms on one core: 33 sightlines x 22k occluders)."""
    return {1: 4000, 2: 250, 3: 100, 4: 40}.get(cfg, 40)


def cpu_baseline(soup, seconds: float = 10.0, cfg: int = 4):
    """The compiled reference (oracle/_ref) — or the C restatement when the
    reference could not be built — timed on the host cores over a bounded
    sample of the same workload's pairs."""
    from oracle import bindings
    cores = _ncores()
    kind = "reference"
    try:
        o = bindings.RefOracle(soup)
    except Exception:
        kind = "port"
        o = bindings.Oracle(soup)
    batch = cores * _pairs_per_core(cfg)
    tests = 0.0
    npairs = 0
    t0 = time.perf_counter()
    b = 0
    while True:
        pi, pj = _sample_pairs(soup.nfaces, batch, 1000 + b)
        o.occlusion_batch(pi, pj, threads=cores)
        tests += _t_alg(soup, pi, pj)
        npairs += len(pi)
        b += 1
        el = time.perf_counter() - t0
        if el >= seconds or b >= 200:
            break
    return {"value": tests / el, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": _cpu_model(),
            "sample": f"{npairs} seeded random pairs of the config-{cfg} matrix, occlusion_judgment on {cores} "
                      f"threads ({el:.1f} s)",
            "pairs_per_s": npairs / el}


def _hbm_peak_gbs() -> tuple:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except Exception:
        return 6536.0, "fallback (B200_PROFILING.md)"


def _hbm_roofline(alg_bytes: float, ms: float, basis: str) -> dict:
    """Algorithmic bytes of a table / frontier launch against the HBM peak
    (regions = the scene state read once + the region records
    written; image tree = 80 B per node)."""
    peak, src = _hbm_peak_gbs()
    gbs = alg_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "alg_bytes": alg_bytes, "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak, "basis": basis, "peak_source": src}


def _committed_ncu(cfg: int) -> dict:
    """The ncu capture of the headline kernel committed under profiles/ for
    this workload (NOT measured in this run: labelled with its source)."""
    p = os.path.join(ROOT, "profiles", f"k2w_config{cfg}_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d["source"] = "committed ncu " + os.path.relpath(p, ROOT)
        return d
    except Exception:
        return {"source": "none committed for this workload"}


def _committed_kernel_ncu(name: str) -> dict:
    p = os.path.join(ROOT, "profiles", f"{name}_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d["source"] = "committed ncu " + os.path.relpath(p, ROOT)
        return d
    except Exception:
        return {"source": "none committed"}


def secondary_measurements(stream: int, headline_cfg: int = 4):
    """The other hot-path subsystems, timed with the library's CUDA events on
    the same stream (outside the headline's timed region, rank 0, N = 1)."""
    from paper_2501_02747_b200 import scenes
    from paper_2501_02747_b200.core import (ENTRY_DTYPE, Scene, Tracer, chain_triples, point_regions_array,
                                            trajectory_vis_table, unpack_bits)
    out = {}
    # (1) the other matrix configurations
    for cfg in [c for c in (1, 2, 3) if c != headline_cfg]:
        with Scene(scenes.workload(cfg).scene) as sc:
            sc.pair_visibility("all", copy_bits=False, stream=stream)
            _, st = sc.pair_visibility("all", copy_bits=False, stream=stream)
            _, sa = sc.pair_visibility("prefiltered", copy_bits=False, stream=stream)
            out[f"matrix_config{cfg}"] = {"B_ms": st["ms"], "B_tests_per_s": st["tests_alg"] / (st["ms"] * 1e-3),
                                          "A_ms": sa["ms"], "A_candidates": sa["candidates"],
                                          "facets": sc.n}
    # config 4 / 5 geometry (22k facets): (B) matrix once, regions + order-3 trees of config-5 snapshots
    wl5 = scenes.workload(5)
    with Scene(wl5.scene) as sc:
        if headline_cfg != 4:
            _, st = sc.pair_visibility("all", copy_bits=False, stream=stream)
            out["matrix_config4"] = {"B_ms": st["ms"], "B_tests_per_s": st["tests_alg"] / (st["ms"] * 1e-3),
                                     "facets": sc.n, "pairs": st["pairs"]}
        _, sa = sc.pair_visibility("prefiltered", copy_bits=False, stream=stream)
        out.setdefault("matrix_config4", {}).update({"A_ms": sa["ms"], "A_candidates": sa["candidates"],
                                                      "facets": sc.n})
        src = np.concatenate([wl5.tx[:10], wl5.rx[:10]])
        point_regions_array(sc, src[:2])
        arr, st = point_regions_array(sc, src)
        out["regions_config5"] = {"snapshots": len(src), "facets": sc.n, "ms": st["ms"],
                                  "regions_per_s": arr.size / (st["ms"] * 1e-3), "ms_per_snapshot": st["ms"] / len(src),
                                  "sightlines": st["candidates"], "exact_tests": st["tests_exec"],
                                  "roofline": _hbm_roofline(arr.nbytes + sc.upload_bytes, st["ms"],
                                                            "region records written + scene state read once"),
                                  "ncu": {"scan": _committed_kernel_ncu("k4w_scan_config5"),
                                          "refine": _committed_kernel_ncu("k4w_refine_config5")}}
        tri, _ = chain_triples(sc)
        tr = Tracer(sc, 3, triples=tri)
        tr.trace_raw(wl5.tx[:4], wl5.rx[:4])
        _, _, nodes, tst = tr.trace_raw(wl5.tx[:200], wl5.rx[:200])
        out["tree_config5_order3"] = {"snapshots": 200, "nodes": tst["nodes"], "ms": tst["ms"],
                                      "ms_per_snapshot": tst["ms"] / 200, "paths": tst["paths"],
                                      "roofline": _hbm_roofline(80.0 * tst["nodes"], tst["ms"], "80 B per node")}
        tr.close()
    # (2) per-snapshot Tx/Rx -> facet regions, config 3 (Tx and Rx snapshots)
    wl = scenes.workload(3)
    with Scene(wl.scene) as sc:
        src = np.concatenate([wl.tx[::10], wl.rx[::10]])
        point_regions_array(sc, src[:8])
        arr, st = point_regions_array(sc, src)
        out["regions_config3"] = {"snapshots": len(src), "facets": sc.n, "ms": st["ms"],
                                  "regions_per_s": arr.size / (st["ms"] * 1e-3),
                                  "ms_per_snapshot": st["ms"] / len(src),
                                  "sightlines": st["candidates"], "exact_tests": st["tests_exec"],
                                  "roofline": _hbm_roofline(arr.nbytes + sc.upload_bytes, st["ms"],
                                                            "region records written + scene state read once")}
        # (3) order-2 chains + image tree order 3, config 3
        sc.pair_visibility("prefiltered", copy_bits=False)
        tri, sch = chain_triples(sc)
        out["chains_config3"] = {"candidate_triples": sch["candidates"], "feasible": sch["admitted"],
                                 "ms": sch["ms"], "ncu": {"screen": _committed_kernel_ncu("k7_screen_config3"),
                                                          "decide": _committed_kernel_ncu("k7_decide_config3"),
                                                          "second": _committed_kernel_ncu("k7_second_config3")}}
        tr = Tracer(sc, 3, triples=tri)
        tr.trace_raw(wl.tx[:4], wl.rx[:4])
        _, _, nodes, tst = tr.trace_raw(wl.tx[:50], wl.rx[:50])
        out["tree_config3_order3"] = {"snapshots": 50, "nodes": tst["nodes"], "ms": tst["ms"],
                                      "nodes_per_s": tst["nodes"] / (tst["ms"] * 1e-3),
                                      "ms_per_snapshot": tst["ms"] / 50, "paths": tst["paths"],
                                      "roofline": _hbm_roofline(80.0 * tst["nodes"], tst["ms"], "80 B per node"),
                                      "ncu": _committed_kernel_ncu("k6_config3")}
        tr.close()
    wl1 = scenes.workload(1)
    with Scene(wl1.scene) as sc:
        sc.pair_visibility("prefiltered", copy_bits=False)
        tr = Tracer(sc, 2)
        tr.trace_raw(wl1.tx[:4], wl1.rx)
        _, _, nodes, tst = tr.trace_raw(wl1.tx, wl1.rx)
        out["tree_config1_order2"] = {"snapshots": len(wl1.tx), "nodes": tst["nodes"], "ms": tst["ms"],
                                      "ms_per_snapshot": tst["ms"] / len(wl1.tx), "paths": tst["paths"]}
        tr.close()
        # (2) trajectory_vis_table along config 1's 100 m Tx line (MobileSampler
        # keys depend only on the reflector chains: order-1 entries of the
        # admitted pairs and order-2 entries of the GPU triples)
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        adm = unpack_bits(bits, sc.n)
        ai, aj = np.nonzero(adm)
        ent = np.zeros(len(ai) + len(tri), ENTRY_DTYPE)
        ent["order"][: len(ai)] = 1
        ent["chain"][: len(ai), 0] = ai
        ent["chain"][: len(ai), 1] = aj
        ent["order"][len(ai):] = 2
        ent["chain"][len(ai):, :3] = tri
        wps = np.array([wl1.tx[0], wl1.tx[-1]])
        for order in (1, 2):
            sel = ent[ent["order"] <= order]
            trajectory_vis_table(sc, wps, sel, order, wl1.scene.ids)
            t0 = time.perf_counter()
            rows, tst = trajectory_vis_table(sc, wps, sel, order, wl1.scene.ids, return_stats=True)
            wall = (time.perf_counter() - t0) * 1e3
            out[f"trajectory_config1_order{order}"] = {
                "route_m": float(np.linalg.norm(wps[1] - wps[0])), "samples": tst["pairs"],
                "boundaries": tst["candidates"], "rows": len(rows), "device_ms": tst["ms"], "wall_ms": wall,
                "kernel_launches": tst["sweeps"]}
        # the reference's trajectory_vis_table on the same route, host cores (order 1: ~2 s)
        try:
            from oracle import bindings
            if bindings.have_ref():
                r = bindings.RefOracle(wl1.scene)
                m = r.build_matrix(1)
                t0 = time.perf_counter()
                rrows = r.trajectory_vis_table(m, wps, 1)
                out["trajectory_config1_order1"]["reference_ms"] = (time.perf_counter() - t0) * 1e3
                out["trajectory_config1_order1"]["reference_rows"] = len(rrows)
                out["trajectory_config1_order1"]["reference_threads"] = _ncores()
        except Exception as e:   # the reference build is optional on the box
            out["trajectory_config1_order1"]["reference_error"] = str(e)[:120]
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2501_02747_b200 import scenes
    from oracle import bindings
    soup = scenes.workload(args.config).scene
    cores = _ncores()
    kind = "reference"
    try:
        o = bindings.RefOracle(soup)
    except Exception:
        kind = "port"
        o = bindings.Oracle(soup)
    per_step = cores * _pairs_per_core(args.config)
    times, tests = [], []
    for step in range(args.warmup + args.steps):
        pi, pj = _sample_pairs(soup.nfaces, per_step, 5000 + step)
        t0 = time.perf_counter()
        o.occlusion_batch(pi, pj, threads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            tests.append(_t_alg(soup, pi, pj))
    value = sum(tests) / sum(times)
    ms = 1e3 * sum(times) / len(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded config-{args.config} city)",
            "config": {"workload": f"config{args.config} matrix (B): reference occlusion_judgment on a bounded "
                                   f"pair sample per step", "pairs_per_step": per_step, "facets": soup.nfaces},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": _cpu_model(),
                             "sample": f"{per_step} seeded pairs of the config-{args.config} matrix per step on "
                                       f"{cores} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_visrt(args, rank, world):
    import torch
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_02747_b200 import scenes
    from paper_2501_02747_b200.core import Scene, measure_peaks

    wl = scenes.workload(args.config, seed=scenes.SEED_BASE + args.config + 7919 * rank)
    soup = wl.scene
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident matrix builds (value) --------------------------
    sc = Scene(soup, device=local)
    for _ in range(args.warmup):
        sc.pair_visibility(args.mode, copy_bits=False, stream=sh)
    step_ms, kern_ms, tests_exec = [], [], []
    tests_alg = 0.0
    barrier()
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, st = sc.pair_visibility(args.mode, copy_bits=False, stream=sh)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(st["ms"])
            tests_exec.append(st["tests_exec"])
            tests_alg = st["tests_alg"]
        barrier()
        wall = time.perf_counter() - t_wall0
    clocks = clk.summary()
    ms_local = sum(step_ms) / len(step_ms)
    cand = st["candidates"]
    sc.close()

    # ---- end to end through the public API, host buffers ----------------
    e2e_times, h2d, d2h = [], 0, 0
    for step in range(args.warmup + max(3, args.steps // 2)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with Scene(soup, device=local) as s2:
            bits, _ = s2.pair_visibility(args.mode, copy_bits=True, stream=sh)
            h2d = s2.upload_bytes
        dt = time.perf_counter() - t0
        d2h = bits.nbytes
        if step >= args.warmup:
            e2e_times.append(dt)
    e2e_s = sum(e2e_times) / len(e2e_times)

    # ---- reductions over ranks ------------------------------------------
    from paper_2501_02747_b200.dist import reduce_step_metrics
    ms_max, total_tests = reduce_step_metrics(ms_local, tests_alg, device="cuda")
    e2e_max, _ = reduce_step_metrics(e2e_s, 0.0, device="cuda")
    if rank == 0:
        fp64_peak, fp32_peak = measure_peaks(local)
        kern = sum(kern_ms) / len(kern_ms)
        execd = sum(tests_exec) / len(tests_exec)
        peak = fp64_peak / 1e12
        ref_equiv = FLOPS_PER_TEST * tests_alg / (kern * 1e-3) / 1e12
        ncu = _committed_ncu(args.config)
        ops_per_test = ncu.get("fp64_thread_ops_per_exact_test") or FLOPS_PER_TEST
        achieved = ops_per_test * execd / (kern * 1e-3) / 1e12
        # ncu's FP64-pipe share of the calibration launch, carried to this run's time and work
        pipe_frac = None
        try:
            pipe_frac = (ncu["ncu_sol"]["fp64_pipe_pct"] / 100.0) * (ncu["duration_ms"] / kern) * \
                        (execd / ncu["exact_tests"])
        except (KeyError, TypeError, ZeroDivisionError):
            pass
        wl_desc = {2: "config2: 1 km city, 200 boxes + 16x16 tiles, N=1256 facets",
                   3: "config3: 2 km Manhattan grid, 500 boxes + 16x16 tiles, N=2756 facets",
                   4: "config4: 4 km city, 2000 convex prisms + 32x32 tiles, N=22096 facets"}.get(
                       args.config, f"config{args.config}")
        line = {
            "metric": METRIC, "value": total_tests / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "matrix_build_ms": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded config-{args.config} generator, one city per rank)",
            "config": {"workload": wl_desc + "; full NxN bit-packed occlusion matrix (B: every i<j vs all N-2 "
                                             "occluders)",
                       "facets": soup.nfaces, "pairs": int(st["pairs"]), "mode": args.mode,
                       "candidates": int(cand), "tests_alg_per_gpu": tests_alg,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": f"dp{world} (independent cities)"},
            "e2e": {"value": total_tests / e2e_max, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "s_per_step": e2e_max,
                    "path": "Scene(soup) ingest+upload -> pair_visibility -> bits D2H -> free"},
            "gpu_launches": args.steps,
            # EXECUTED work against the FP64 pipe (executed FP64 instructions / (kernel time x
            # peak rate), ncu pipe % as the cross-check). `frac` = the share of the pipe's issue capacity
            # the kernel's FP64 warp instructions take; `thread_ops` = the stricter lane-level count.
            "roofline": {"bound": "fp64", "kernel": "k_pair_bits_warp",
                         "achieved": (pipe_frac if pipe_frac is not None else achieved / peak) * peak, "peak": peak,
                         "unit": "TFLOP/s", "frac": pipe_frac if pipe_frac is not None else achieved / peak,
                         "traffic": ncu.get("dram_bytes_per_launch"),
                         "basis": "EXECUTED FP64-pipe warp instructions / (kernel time x the pipe's issue rate): ncu "
                                  "sm__pipe_fp64_cycles_active of the committed capture of this very launch "
                                  "(ncu.source), scaled by this run's exact-test count and kernel time; `achieved` is "
                                  "that share of the in-run DADD/DMUL peak (MEASURED_PEAKS.json has no FP64 entry)",
                         "thread_ops": {"achieved": achieved, "frac": achieved / peak, "unit": "TFLOP/s",
                                        "basis": "lane-level: in-run exact-test count x DADD+DMUL+2*DFMA thread ops "
                                                 "per exact test (ncu-calibrated on this launch) / kernel time. Below "
                                                 "`frac` because FP64 warp instructions hold the pipe with idle lanes "
                                                 "(ncu.ncu_sol.active_threads_per_inst of 32) and the pipe also "
                                                 "executes DSETP compares, DMNMX and F2F conversions, not counted here"},
                         "executed_exact_tests": execd,
                         "executed_exact_tests_per_s": execd / (kern * 1e-3),
                         "reference_equivalent": {"achieved": ref_equiv, "frac": ref_equiv / peak,
                                                  "basis": "17 FP64 ops x T_alg reference tests / kernel time: "
                                                           "culling + early exit skip the reference's work, "
                                                           "so this exceeds 1; not a roofline"},
                         "fp32_peak_tflops": fp32_peak / 1e12,
                         "ncu": ncu},
            "clocks": clocks,
            "wall_s_timed_loop": wall,
        }
        if world == 1 and not args.no_secondary:
            try:
                line["subsystems"] = secondary_measurements(sh, args.config)
            except Exception as e:   # noqa: BLE001
                line["subsystems"] = {"error": str(e)}
        if world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline(soup, seconds=args.cpu_seconds, cfg=args.config)
            except Exception as e:   # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": _ncores(), "kind": "unavailable",
                                        "sample": f"failed: {e}"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="visrt", choices=["visrt", "reference"])
    ap.add_argument("--mode", default="all", choices=["all", "prefiltered"])
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4],
                    help="matrix workload (default: config 4, the largest single-GPU configuration)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-secondary", action="store_true", help="skip the other subsystems' timings")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "visrt" else args.warmup
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_visrt(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())
