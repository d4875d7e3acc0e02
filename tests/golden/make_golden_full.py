"""Full-size reference fixtures for configs 3-5 (TEST INFRASTRUCTURE ONLY).

Every output here comes from the UNMODIFIED reference compiled by
oracle/Makefile into oracle/_ref (bindings.RefOracle), driven on the seeded
BASELINE scenes of paper_2501_02747_b200/scenes.py.  The GPU tests
(tests/test_fullsize_ref_gpu.py) re-run the same workloads on the B200 and
compare against these files; /root/reference is never read there.

Run here (needs /root/reference to build oracle/_ref), one stage at a time or
all of them (each stage writes tests/golden/full/<stage>*.npz and is skipped
when its file exists):

    nice -n 19 python tests/golden/make_golden_full.py [stage ...]

Stages (reference functions cited against /root/reference/proj):
  c3B        occlusion_judgment on ALL 3,796,390 config-3 pairs i<j
             (src/vismatrix.cpp:253-302): the (B) bit = kind != Occluded,
             packed over np.triu_indices order.
  c3A        build_matrix(scene, 1) (src/vismatrix.cpp:638-675): the order-1
             entries [ref, aim, plane] in the matrix's own order; the (A)
             bit is pair_admitted = has an order-1 entry.
  c4A        same for config 4 (22,096 facets, 2.44e8 pairs).
  c4B        occlusion_judgment on 100,000 seeded config-4 pairs.
  c3regions  illuminated_region (src/vistable.cpp:287-334) for 100 seeded
             config-3 sources (50 Tx + 50 Rx) x ALL 2,756 faces: per source
             a sha256 of the canonical region array (golden_util.region_digest)
             plus the present/has/clipped arrays and the sub doubles.
  c3tables   point_vis_table(src, build_matrix(scene,1), scene, 1)
             (src/vistable.cpp:478-521) for 50 seeded config-3 sources: every
             row as (entry index, Full, ref primed, aim primed).
  c3traj     trajectory_vis_table (src/vistable.cpp:845-987) on a 100 m
             stretch of the config-3 Tx street, order 1.
  c5trace    TraceAccelerator::trace (src/raytracer.cpp:496-514) at order 3
             with build_matrix(scene, 2) + set_max_order(3) for 100 seeded
             config-5 snapshots: node counts + every path.
  c3trace    the same for 100 seeded config-3 snapshots.
  c3chains   every order-2 chain of build_matrix(scene, 2) on config 3
             (src/vismatrix.cpp:715-797): count, sha256 and a 1/997 sample of
             the sorted unique (p, t, a) triples.
  c5regions  illuminated_region for 100 seeded config-5 sources (50 Tx +
             50 Rx) x ALL 22,096 faces, in chunks of 4 sources
             (c5regions_<k>.npz): digests + present arrays, records of the
             first chunk.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import bindings  # noqa: E402
from paper_2501_02747_b200 import scenes  # noqa: E402
import golden_util as G  # noqa: E402

OUT = os.path.join(HERE, "full")
THREADS = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 1))


def scene_sha(soup) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(soup.vert_off, np.int32).tobytes())
    h.update(np.ascontiguousarray(soup.verts, np.float64).tobytes())
    return h.hexdigest()


def save(name: str, **arrays) -> None:
    os.makedirs(OUT, exist_ok=True)
    tmp = os.path.join(OUT, name + ".tmp.npz")
    np.savez_compressed(tmp, **arrays)
    os.replace(tmp, os.path.join(OUT, name + ".npz"))
    print(f"  wrote {name}.npz ({os.path.getsize(os.path.join(OUT, name + '.npz')) / 1e6:.2f} MB)", flush=True)


def done(name: str) -> bool:
    return os.path.exists(os.path.join(OUT, name + ".npz"))


_REF = {}


def ref(cfg: int):
    if cfg not in _REF:
        wl = scenes.workload(cfg)
        _REF[cfg] = (wl, bindings.RefOracle(wl.scene))
    return _REF[cfg]


_MAT = {}


def matrix(cfg: int, order: int):
    if (cfg, order) not in _MAT:
        os.environ["VISRT_THREADS"] = str(THREADS)
        _MAT[(cfg, order)] = ref(cfg)[1].build_matrix(order)
    return _MAT[(cfg, order)]


def pmap(fn, items):
    with cf.ThreadPoolExecutor(THREADS) as ex:   # ctypes calls release the GIL
        return list(ex.map(fn, items))


# ---------------------------------------------------------------------------

def stage_matrix_B_all(cfg: int):
    wl, r = ref(cfg)
    n = wl.scene.nfaces
    pi, pj = G.pairs(n)
    kinds = r.occlusion_batch(pi, pj, THREADS)
    assert (kinds >= 0).all()
    save(f"c{cfg}B", scene_sha=np.array(scene_sha(wl.scene)), n=np.array(n),
         bits=np.packbits(kinds != 2), kind_counts=np.bincount(kinds, minlength=3))


def stage_matrix_B_sampled(cfg: int, m: int):
    wl, r = ref(cfg)
    n = wl.scene.nfaces
    rng = np.random.default_rng(2501027470 + 40 + cfg)
    i = rng.integers(0, n, 2 * m)
    j = rng.integers(0, n, 2 * m)
    keep = i != j
    pi = np.minimum(i, j)[keep][:m].astype(np.int32)
    pj = np.maximum(i, j)[keep][:m].astype(np.int32)
    kinds = r.occlusion_batch(pi, pj, THREADS)
    assert (kinds >= 0).all()
    save(f"c{cfg}B", scene_sha=np.array(scene_sha(wl.scene)), n=np.array(n), pi=pi, pj=pj, kinds=kinds)


def order1_entries(r, m):
    ents = r.matrix_entries(m)
    return np.array([[e["chain"][0], e["chain"][1], e["plane"]] for e in ents if e["order"] == 1],
                    np.int32).reshape(-1, 3)


def stage_matrix_A(cfg: int):
    wl, r = ref(cfg)
    m = matrix(cfg, 1)
    E = order1_entries(r, m)
    save(f"c{cfg}A", scene_sha=np.array(scene_sha(wl.scene)), n=np.array(wl.scene.nfaces), entries=E)


def sources(wl, k: int, seed: int):
    rng = np.random.default_rng(seed)
    it = np.sort(rng.choice(len(wl.tx), k // 2, replace=False))
    ir = np.sort(rng.choice(len(wl.rx), k - k // 2, replace=False))
    return np.concatenate([wl.tx[it], wl.rx[ir]]), np.concatenate([it, ir + 100000])


def ref_regions(r, src, n):
    """Reference regions of sources x all faces as the REGION_DTYPE fields."""
    faces = np.tile(np.arange(n, dtype=np.int32), len(src))
    S = np.repeat(src, n, axis=0)
    out = r.regions_batch(S, faces, THREADS)
    P = np.array([o["present"] for o in out], np.int8).reshape(len(src), n)
    H = np.array([o["has"] for o in out], np.int8).reshape(len(src), n, 3)
    Cl = np.array([o["clipped"] for o in out], np.int8).reshape(len(src), n, 3)
    Sb = np.array([o["sub"] for o in out], np.float64).reshape(len(src), n, 6)
    return P, H, Cl, Sb


def stage_regions(cfg: int, k: int, chunk: int = 0, records_chunks: int = 1 << 30):
    wl, r = ref(cfg)
    n = wl.scene.nfaces
    src, tag = sources(wl, k, 2501027470 + 50 + cfg)
    ranges = [(0, len(src))] if not chunk else [(a, min(a + chunk, len(src))) for a in range(0, len(src), chunk)]
    for c, (a, b) in enumerate(ranges):
        name = f"c{cfg}regions" if not chunk else f"c{cfg}regions_{c:02d}"
        if done(name):
            continue
        t = time.time()
        P, H, Cl, Sb = ref_regions(r, src[a:b], n)
        dig = np.array([G.region_digest(P[q], H[q], Cl[q], Sb[q]) for q in range(b - a)])
        extra = {}
        if c < records_chunks:
            pres = P == 1
            extra = dict(has=H, clipped=Cl, sub=Sb[pres])
        save(name, scene_sha=np.array(scene_sha(wl.scene)), src=src[a:b], tag=tag[a:b], digest=dig, present=P,
             **extra)
        print(f"  {name}: {b - a} sources in {time.time() - t:.0f} s, present {int((P == 1).sum())}", flush=True)


def stage_tables(cfg: int, k: int):
    wl, r = ref(cfg)
    m = matrix(cfg, 1)
    E = order1_entries(r, m)
    index = {(int(a), int(b), int(p)): q for q, (a, b, p) in enumerate(E)}
    src, tag = sources(wl, k, 2501027470 + 60 + cfg)
    ids = wl.scene.ids

    def one(s):
        return r.point_vis_table(m, np.asarray(s), 1)

    rows = pmap(one, list(src))
    off = [0]
    ent, full, rp, ap = [], [], [], []
    for q, rs in enumerate(rows):
        recs = []
        for x in rs:
            key = (x["chain"][0], x["aim"], x["plane"])
            assert x["ref_display"] in (ids[x["chain"][0]], ids[x["chain"][0]] + "'")
            recs.append((index[key], x["verdict"] == 0, x["ref_display"] == ids[x["chain"][0]] + "'",
                         x["aim_display"] == ids[x["aim"]] + "'"))
        recs.sort()   # by entry index (the rows' own order is the reference's name sort)
        prev = 0
        for e, fu, r_, a_ in recs:
            ent.append(e - prev)   # delta-coded per source (first = absolute)
            prev = e
            full.append(fu)
            rp.append(r_)
            ap.append(a_)
        off.append(len(ent))
    # the entry list itself is c{cfg}A.npz's (the same build_matrix(scene, 1))
    save(f"c{cfg}tables", scene_sha=np.array(scene_sha(wl.scene)), src=src, tag=tag,
         off=np.array(off, np.int64), entry_delta=np.array(ent, np.int32), full=np.array(full, bool),
         ref_primed=np.array(rp, bool), aim_primed=np.array(ap, bool))


def stage_traj(cfg: int, length: int):
    wl, r = ref(cfg)
    m = matrix(cfg, 1)
    E = order1_entries(r, m)
    wps = np.array([wl.tx[0], wl.tx[length]], np.float64)
    rows = r.trajectory_vis_table(m, wps, 1)
    keys = ["order", "node", "node_display", "s_start", "s_end", "label_start", "label_end", "parent", "blockage"]
    strs = "\n".join("\t".join(str(x[k]) if k not in ("s_start", "s_end") else float(x[k]).hex() for k in keys)
                     for x in rows)
    save(f"c{cfg}traj", scene_sha=np.array(scene_sha(wl.scene)), waypoints=wps,
         rows=np.frombuffer(strs.encode(), np.uint8))   # entries: c{cfg}A.npz
    print(f"  {len(rows)} rows", flush=True)


def stage_trace(cfg: int, k: int):
    wl, r = ref(cfg)
    t = time.time()
    m = matrix(cfg, 2)
    r.lib().vref_matrix_set_max_order(m, 3)
    print(f"  build_matrix(scene, 2): {time.time() - t:.0f} s", flush=True)
    acc = r.accel(m, 3)
    rng = np.random.default_rng(2501027470 + 70 + cfg)
    ks = np.sort(rng.choice(len(wl.tx), k, replace=False))

    def one(q):
        return r.trace(acc, wl.tx[q], wl.rx[q])

    res = pmap(one, list(ks))
    nodes = np.array([st[0] for _, st in res], np.int64)
    stats = np.array([list(st) for _, st in res], np.int64)
    off, faces, pts, length = [0], [], [], []
    for paths, _ in res:
        for p in paths:
            f = p["faces"] + [-1] * (4 - len(p["faces"]))
            faces.append(f)
            pt = p["points"] + [0.0] * (18 - len(p["points"]))
            pts.append(pt)
            length.append(p["length"])
        off.append(len(faces))
    save(f"c{cfg}trace", scene_sha=np.array(scene_sha(wl.scene)), snap=ks, nodes=nodes, stats=stats,
         off=np.array(off, np.int64), faces=np.array(faces, np.int32).reshape(-1, 4),
         points=np.array(pts, np.float64).reshape(-1, 18), length=np.array(length, np.float64))
    print(f"  {len(ks)} snapshots in {time.time() - t:.0f} s, {off[-1]} paths, {nodes.sum()} nodes", flush=True)


def stage_chains(cfg: int):
    """Every order-2 chain (p, t, a) of build_matrix(scene, 2) (src/vismatrix.cpp:
    715-797): the unique triples sorted lexicographically, kept as their count,
    a sha256 of the int32 array and every 997th triple (the full set of config 3
    is ~180 MB)."""
    wl, r = ref(cfg)
    t = time.time()
    m = matrix(cfg, 2)
    print(f"  build_matrix(scene, 2): {time.time() - t:.0f} s", flush=True)
    c = r.matrix_chains(m, 2)
    c = np.unique(c, axis=0).astype(np.int32)
    save(f"c{cfg}chains", scene_sha=np.array(scene_sha(wl.scene)), count=np.array(len(c)),
         sha=np.array(hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest()),
         sample_idx=np.arange(0, len(c), 997, dtype=np.int64), sample=c[::997])


STAGES = {
    "c3B": lambda: stage_matrix_B_all(3),
    "c3A": lambda: stage_matrix_A(3),
    "c4A": lambda: stage_matrix_A(4),
    "c4B": lambda: stage_matrix_B_sampled(4, 100000),
    "c3regions": lambda: stage_regions(3, 100),
    "c3tables": lambda: stage_tables(3, 50),
    "c3traj": lambda: stage_traj(3, 100),
    "c5trace": lambda: stage_trace(5, 100),
    "c3trace": lambda: stage_trace(3, 100),
    "c5regions": lambda: stage_regions(5, 100, chunk=4, records_chunks=1),
    "c3chains": lambda: stage_chains(3),
}


def main(argv) -> None:
    bindings.build(ref=True)
    todo = argv or list(STAGES)
    for s in todo:
        if s != "c5regions" and done(s):
            print(f"{s}: exists", flush=True)
            continue
        t = time.time()
        print(f"{s} ...", flush=True)
        STAGES[s]()
        print(f"{s}: {time.time() - t:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
