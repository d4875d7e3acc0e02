"""Python host mirror of the reference's hot-path API over the C-ABI.

Names, argument meaning and error behaviour follow the reference's C++ API
(namespace ``rt``): ``occlusion_judgment`` (include/rt/vismatrix.hpp:113),
``build_matrix`` pair loop (vismatrix.hpp:141), ``illuminated_region``
(include/rt/vistable.hpp:116-117), ``TraceAccelerator::trace``
(include/rt/raytracer.hpp:96-118). Every call goes through
``libvisrt_cuda.so``; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import check, lib
from .scenes import FacetSoup

KIND_NAMES = ("Visible", "PartiallyVisible", "Occluded")


def _stats_dict(st: _capi.visrt_stats) -> Dict[str, float]:
    return {"pairs": st.pairs, "candidates": st.candidates, "admitted": st.admitted,
            "tests_alg": st.tests_alg, "tests_exec": st.tests_exec, "ms": st.ms,
            "sweeps": st.sweeps, "tiles": st.tiles}


class Scene:
    """A facet scene resident on one GPU (``visrt_scene_create``)."""

    def __init__(self, soup: FacetSoup, device: int = 0) -> None:
        L = lib()
        self.soup = soup
        self.n = soup.nfaces
        self._vert_off = np.ascontiguousarray(soup.vert_off, dtype=np.int32)
        self._verts = np.ascontiguousarray(soup.verts, dtype=np.float64).reshape(-1)
        self._building = (None if soup.building is None
                          else np.ascontiguousarray(soup.building, dtype=np.int32))
        f = _capi.visrt_facets_v1(self.n, self._vert_off.ctypes.data, self._verts.ctypes.data,
                                  None if self._building is None else self._building.ctypes.data)
        h = C.c_void_p()
        check(L.visrt_scene_create(C.byref(f), device, C.byref(h)))
        self.h = h
        self.words = (self.n + 63) // 64
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().visrt_scene_destroy(self.h)
            self.h = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def upload_bytes(self) -> int:
        return int(lib().visrt_scene_upload_bytes(self.h))

    # -- ingest products (host copies) ----------------------------------------
    def ingest(self):
        n = self.n
        normal = np.zeros(3 * n)
        orient = np.zeros(n, np.int32)
        seg = np.zeros(18 * n)
        ok = np.zeros(3 * n, np.int32)
        check(lib().visrt_scene_ingest(self.h, normal.ctypes.data, orient.ctypes.data, seg.ctypes.data,
                                       ok.ctypes.data))
        return normal.reshape(n, 3), orient, seg.reshape(n, 3, 6), ok.reshape(n, 3)

    # -- (1) matrix -------------------------------------------------------------
    def pair_visibility(self, mode: str = "all", copy_bits: bool = True, stream: int = 0,
                        rows: Optional[Tuple[int, int]] = None
                        ) -> Tuple[Optional[np.ndarray], Dict[str, float]]:
        """(B) ``mode="all"``: bit(i,j) = occlusion_judgment(F_i, F_j).kind != Occluded for all
        i<j. (A) ``mode="prefiltered"``: pair_admitted(i, j) of build_matrix(scene, 1).
        ``rows=(r0, r1)`` ((B) only): decide the pairs of reference rows r0 <= i < r1 alone; the
        returned full-size matrix is zero elsewhere, so the blocks of a partition
        (dist.pair_row_blocks) OR into the whole matrix — one scene sharded over several GPUs."""
        flags = {"all": _capi.VISRT_PAIRS_ALL, "prefiltered": _capi.VISRT_PAIRS_PREFILTERED}[mode]
        bits = np.zeros(self.n * self.words, np.uint64) if copy_bits else None
        st = _capi.visrt_stats()
        bp = None if bits is None else bits.ctypes.data
        sp = C.c_void_p(stream) if stream else None
        if rows is None:
            check(lib().visrt_pair_visibility(self.h, flags, bp, C.byref(st), sp))
        else:
            check(lib().visrt_pair_visibility_rows(self.h, flags, int(rows[0]), int(rows[1]), bp, C.byref(st), sp))
        return (None if bits is None else bits.reshape(self.n, self.words)), _stats_dict(st)

    def candidates(self):
        L = lib()
        m = L.visrt_candidates(self.h, None, None, None)
        ci = np.zeros(m, np.int32)
        cj = np.zeros(m, np.int32)
        ad = np.zeros(m, np.uint8)
        L.visrt_candidates(self.h, ci.ctypes.data, cj.ctypes.data, ad.ctypes.data)
        return ci, cj, ad

    def pair_detail(self, ci: Sequence[int], cj: Sequence[int]):
        """occlusion_judgment(F_ci, F_cj) for a pair list: kinds + blocker index sets."""
        ci = np.ascontiguousarray(ci, np.int32)
        cj = np.ascontiguousarray(cj, np.int32)
        m = len(ci)
        kind = np.zeros(m, np.int8)
        off = np.zeros(m + 1, np.int64)
        st = _capi.visrt_stats()
        check(lib().visrt_pair_detail(self.h, m, ci, cj, kind, off, None, 0, C.byref(st), None))
        idx = np.zeros(max(int(off[-1]), 1), np.int32)
        check(lib().visrt_pair_detail(self.h, m, ci, cj, kind, off, idx.ctypes.data, len(idx), C.byref(st),
                                      None))
        blockers = [idx[off[k]:off[k + 1]].tolist() for k in range(m)]
        return kind, blockers, _stats_dict(st)


REGION_DTYPE = np.dtype([("present", np.int8), ("has", np.int8, 3), ("clipped", np.int8, 3), ("pad", np.int8),
                         ("sub", np.float64, 6)])


def point_regions_array(scene: Scene, src: np.ndarray, stream: int = 0, out: Optional[np.ndarray] = None):
    """illuminated_region(src[k], face f) for every (k, f) — one batched GPU call
    (rt::illuminated_region, include/rt/vistable.hpp:116-117). Returns a
    structured array [nsrc, nfaces] (present: 1 region / 0 none / -1 source on
    the face plane, the reference's VisibilityError) and the call stats."""
    src = np.ascontiguousarray(np.asarray(src, np.float64).reshape(-1, 3))
    # every record is written by the call; `out` (C-contiguous REGION_DTYPE,
    # >= len(src) * n records) lets batch loops reuse one resident buffer
    if out is None:
        out = np.empty((len(src), scene.n), REGION_DTYPE)
    else:
        if out.dtype != REGION_DTYPE or not out.flags.c_contiguous or out.size < len(src) * scene.n:
            raise ValueError("out must be a C-contiguous REGION_DTYPE array of at least len(src) * n records")
        out = out.reshape(-1)[: len(src) * scene.n].reshape(len(src), scene.n)
    st = _capi.visrt_stats()
    check(lib().visrt_point_regions(scene.h, len(src), src.reshape(-1),
                                    out.ctypes.data_as(C.POINTER(_capi.visrt_region)), C.byref(st),
                                    C.c_void_p(stream) if stream else None))
    return out, _stats_dict(st)


def point_regions(scene: Scene, src: np.ndarray) -> List[List[dict]]:
    arr, _ = point_regions_array(scene, src)
    return [[{"present": int(r["present"]), "has": [int(x) for x in r["has"]],
              "clipped": [int(x) for x in r["clipped"]], "sub": [float(x) for x in r["sub"]]}
             for r in row] for row in arr]


ENTRY_DTYPE = np.dtype([("order", np.int32), ("chain", np.int32, 5), ("plane", np.int32)])


def point_tables(scene: Scene, src: np.ndarray, entries: np.ndarray, want_regions: bool = False,
                 packed: bool = False):
    """For every (source k, matrix entry e) of order 1/2: does TableBuilder::reach
    succeed (row of point_vis_table) and is the beam Full in the entry's
    plane — GPU regions + beam cascade in one batched call. Returns
    (rows[nsrc, nent] bool, full[nsrc, nent] bool, regions or None, stats);
    with packed=True rows / full stay the library's bit rows (uint32
    [nsrc, ceil(nent / 32)], bit e % 32 of word e // 32) — no host expansion
    of big tables (config 3: 1.1e9 entries per table)."""
    src = np.ascontiguousarray(np.asarray(src, np.float64).reshape(-1, 3))
    ent = np.ascontiguousarray(entries, ENTRY_DTYPE)
    nsrc, nent = len(src), len(ent)
    words = (nent + 31) // 32
    rows = np.zeros((nsrc, max(words, 1)), np.uint32)
    full = np.zeros((nsrc, max(words, 1)), np.uint32)
    regs = np.zeros((nsrc, scene.n), REGION_DTYPE) if want_regions else None
    st = _capi.visrt_stats()
    check(lib().visrt_point_tables(scene.h, nsrc, src.reshape(-1), nent, ent.ctypes.data, rows.ctypes.data,
                                   full.ctypes.data, None if regs is None else regs.ctypes.data, C.byref(st), None))
    if packed:
        return rows, full, regs, _stats_dict(st)
    unpack = lambda b: np.unpackbits(b.view(np.uint8), axis=1, bitorder="little")[:, :nent].astype(bool)
    return unpack(rows), unpack(full), regs, _stats_dict(st)


def segments_clear(scene: Scene, a: np.ndarray, b: np.ndarray):
    """Batched sightline_clear(a, b, skip=-1) on the GPU."""
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, 3))
    b = np.ascontiguousarray(np.asarray(b, np.float64).reshape(-1, 3))
    out = np.zeros(len(a), np.uint8)
    st = _capi.visrt_stats()
    check(lib().visrt_segments_clear(scene.h, len(a), a.reshape(-1), b.reshape(-1), out.ctypes.data, C.byref(st),
                                     None))
    return out.astype(bool), _stats_dict(st)


def chain_reach(scene: Scene, src: np.ndarray, chains: np.ndarray):
    """TableBuilder::reach for a query list: (source q, reflector chain q) ->
    (reach[q], full[q]) — MobileSampler::member for face nodes."""
    src = np.ascontiguousarray(np.asarray(src, np.float64).reshape(-1, 3))
    ch = np.ascontiguousarray(chains, ENTRY_DTYPE)
    reach = np.zeros(len(src), np.uint8)
    full = np.zeros(len(src), np.uint8)
    st = _capi.visrt_stats()
    check(lib().visrt_chain_reach(scene.h, len(src), src.reshape(-1), ch.ctypes.data, reach.ctypes.data,
                                  full.ctypes.data, C.byref(st), None))
    return reach.astype(bool), full.astype(bool), _stats_dict(st)


MOBILE_ROW_DTYPE = np.dtype([("order", np.int32), ("node", np.int32), ("vertex", np.int32), ("parent", np.int32),
                             ("s_start", np.float64), ("s_end", np.float64), ("label_start", np.int32),
                             ("label_end", np.int32), ("prime_start", np.int32), ("prime_end", np.int32),
                             ("blockage", np.int32), ("pad", np.int32)])


def _ranks(strings: Sequence[str]) -> Dict[str, int]:
    return {s: r for r, s in enumerate(sorted(set(strings)))}


def trajectory_vis_table(scene: Scene, waypoints, entries: np.ndarray, max_order: int, ids: Sequence[str],
                         labels_xy: Optional[Sequence[str]] = None, building: Optional[Sequence[int]] = None,
                         building_names: Optional[Sequence[str]] = None, matrix_max_order: Optional[int] = None,
                         return_stats: bool = False):
    """rt::trajectory_vis_table (include/rt/vistable.hpp:143-148,
    src/vistable.cpp:822-960) on the GPU: rows as dicts with the reference's
    MobileVisEntry fields (order, node, node_display, s_start, s_end,
    label_start, label_end, parent, blockage). ``entries`` are the matrix
    entries (ENTRY_DTYPE) in matrix order; ``labels_xy`` the faces' XY labels
    ("" = use the id); ``building``/``building_names`` give building_of()."""
    n = scene.n
    wp = np.ascontiguousarray(np.asarray(waypoints, np.float64)[:, :3]).reshape(-1)
    if matrix_max_order is not None and matrix_max_order < max_order:
        raise _capi.VisibilityError(f"matrix holds orders up to {matrix_max_order}, requested {max_order}")
    # the reference's string orders as integer ranks (SigKey / row sorts);
    # cached per scene and naming, since they cost more than the GPU work on
    # 20k-facet scenes
    nkey = (tuple(ids), None if labels_xy is None else tuple(labels_xy),
            None if building is None else tuple(int(b) for b in building),
            None if building_names is None else tuple(building_names))
    cache = scene.__dict__.setdefault("_traj_names", {})
    if nkey not in cache:
        nv = np.diff(scene.soup.vert_off)
        corner = {(f, k): f"{ids[f]}#{k}" for f in range(n) for k in range(int(nv[f]))}
        kr = _ranks(list(ids) + list(corner.values()) + ["transmitter"])
        key_rank = np.zeros(9 * n + 1, np.int32)
        key_rank[:n] = [kr[i] for i in ids]
        for (f, k), s in corner.items():
            key_rank[n + 8 * f + k] = kr[s]
        key_rank[9 * n] = kr["transmitter"]
        lab = [(labels_xy[f] if labels_xy is not None and labels_xy[f] else ids[f]) for f in range(n)]
        pr = _ranks(lab + ["transmitter"])
        parent_rank = np.array([pr[s] for s in lab] + [pr["transmitter"]], np.int32)
        bname = [("ground" if building is None or building[f] < 0 or not building_names
                  else building_names[building[f]]) for f in range(n)]
        br = _ranks(bname)
        building_rank = np.array([br[s] for s in bname], np.int32)
        cache.clear()
        cache[nkey] = (key_rank, parent_rank, building_rank, lab, br)
    key_rank, parent_rank, building_rank, lab, br = cache[nkey]
    names = _capi.visrt_names(key_rank.ctypes.data, parent_rank.ctypes.data, building_rank.ctypes.data)
    ent = np.ascontiguousarray(entries, ENTRY_DTYPE)
    h = C.c_void_p()
    st = _capi.visrt_stats()
    L = lib()
    check(L.visrt_trajectory_table(scene.h, len(wp) // 3, wp, len(ent), ent.ctypes.data, max_order, C.byref(names),
                                   C.byref(h), C.byref(st), None))
    try:
        nrows = L.visrt_mobile_table_rows(h, None, 0)
        rows = np.zeros(max(nrows, 1), MOBILE_ROW_DTYPE)
        L.visrt_mobile_table_rows(h, rows.ctypes.data, nrows)
    finally:
        L.visrt_mobile_table_destroy(h)
    inv_b = {r: s for s, r in br.items()}

    def label(i, p):
        return "-" if i == 0 else f"P{i}" + ("'" if p else "")

    out = []
    for r in rows[:nrows]:
        f, v, p = int(r["node"]), int(r["vertex"]), int(r["parent"])
        out.append({"order": int(r["order"]), "node": ids[f] if v < 0 else f"{ids[f]}#{v}",
                    "node_display": lab[f] if v < 0 else f"{lab[f]}#{v}",
                    "s_start": float(r["s_start"]), "s_end": float(r["s_end"]),
                    "label_start": label(int(r["label_start"]), int(r["prime_start"])),
                    "label_end": label(int(r["label_end"]), int(r["prime_end"])),
                    "parent": "transmitter" if p < 0 else lab[p],
                    "blockage": "-" if r["blockage"] < 0 else inv_b[int(r["blockage"])]})
    return (out, _stats_dict(st)) if return_stats else out


def point_vis_table(scene: Scene, src, entries: np.ndarray, ids: Sequence[str], labels=None):
    """rt::point_vis_table rows (src/vistable.cpp:478-521) for one source and
    the given matrix entries: (order, chain ids, aim id, plane, verdict,
    ref_display, aim_display), sorted like the reference."""
    rows, full, regs, _ = point_tables(scene, np.asarray(src).reshape(1, 3), entries, want_regions=True)
    reg = regs[0]

    def display(f, plane):
        name = ids[f] if labels is None else (labels[f][0] if plane == 0 else labels[f][1]) or ids[f]
        r = reg[f]
        if r["present"] == 1 and r["has"][plane] and r["clipped"][plane]:
            name += "'"
        return name

    out = []
    for e, ok in enumerate(rows[0]):
        if not ok:
            continue
        E = entries[e]
        refl = [int(x) for x in E["chain"][: E["order"]]]
        aim = int(E["chain"][E["order"]])
        pl = int(E["plane"])
        out.append({"order": int(E["order"]), "chain": [ids[f] for f in refl], "aim": ids[aim], "plane": pl,
                    "verdict": "Full" if full[0, e] else "Partial", "ref_display": display(refl[-1], pl),
                    "aim_display": display(aim, pl)})
    out.sort(key=lambda r: (r["order"], r["chain"], r["aim"], r["plane"]))
    return out


def chain_triples(scene: Scene, admitted_bits: Optional[np.ndarray] = None):
    """Order-2 chains (p, t, a) of build_matrix(scene, 2) computed on the GPU
    (chain_triple_feasible + second_order_check per shared plane), sorted."""
    bits = None if admitted_bits is None else np.ascontiguousarray(admitted_bits, np.uint64)
    cnt = C.c_int64()
    st = _capi.visrt_stats()
    L = lib()
    check(L.visrt_chain_triples(scene.h, None if bits is None else bits.ctypes.data, None, 0, C.byref(cnt),
                                C.byref(st), None))
    out = np.empty((max(cnt.value, 1), 3), np.int32)   # the first cnt rows are written by the call
    check(L.visrt_chain_triples(scene.h, None if bits is None else bits.ctypes.data, out.ctypes.data,
                                cnt.value, C.byref(cnt), C.byref(st), None))
    return out[: cnt.value], _stats_dict(st)


class Tracer:
    """rt::TraceAccelerator (include/rt/raytracer.hpp:96-118) over the GPU image
    tree: the chain filter is the admitted matrix (pair_admitted) plus the
    order-2 chains (p, t, a) for max_refl 3. ``trace`` runs a whole batch of
    snapshots. ``edges`` (the scene's edges in order, {id, a, b}) enable
    ``allow_diffraction``: per snapshot the receiver's closest diffraction
    edge adds the sequences ending at its Fermat point (facet soups carry no
    edges)."""

    def __init__(self, scene: Scene, max_refl: int, admitted_bits: Optional[np.ndarray] = None,
                 triples: Optional[np.ndarray] = None, edges: Optional[Sequence[dict]] = None) -> None:
        self.scene = scene
        self.max_refl = max_refl
        if max_refl >= 3 and triples is None:
            # the ChainFilter needs the order-2 chains: grow them on the GPU
            triples, _ = chain_triples(scene, admitted_bits)
        bits = None if admitted_bits is None else np.ascontiguousarray(admitted_bits, np.uint64)
        tri = None if triples is None else np.ascontiguousarray(np.asarray(triples, np.int32).reshape(-1, 3))
        h = C.c_void_p()
        check(lib().visrt_tracer_create(scene.h, max_refl, None if bits is None else bits.ctypes.data,
                                        0 if tri is None else len(tri), None if tri is None else tri.ctypes.data,
                                        C.byref(h)))
        self.h = h
        self.edges = list(edges) if edges else []
        if self.edges:
            ab = np.ascontiguousarray(np.array([list(e["a"]) + list(e["b"]) for e in self.edges], np.float64))
            rank = _ranks([e["id"] for e in self.edges])
            er = np.ascontiguousarray(np.array([rank[e["id"]] for e in self.edges], np.int32))
            check(lib().visrt_tracer_set_edges(h, len(self.edges), ab.ctypes.data, er.ctypes.data))

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().visrt_tracer_destroy(self.h)
            self.h = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def trace_raw(self, tx: np.ndarray, rx: np.ndarray, stream: int = 0, allow_diffraction: bool = False,
                  brute_force: bool = False):
        tx = np.ascontiguousarray(np.asarray(tx, np.float64).reshape(-1, 3))
        rx = np.ascontiguousarray(np.asarray(rx, np.float64).reshape(-1, 3))
        flags = 1 if len(rx) == 1 and len(tx) != 1 else 0
        if allow_diffraction:
            flags |= 2
        if brute_force:
            flags |= 4
        st = _capi.visrt_trace_stats()
        check(lib().visrt_trace(self.h, len(tx), tx.reshape(-1), rx.reshape(-1), flags, C.byref(st),
                                C.c_void_p(stream) if stream else None))
        L = lib()
        npaths = L.visrt_trace_results(self.h, None, None, 0, None)
        off = np.zeros(len(tx) + 1, np.int64)
        nodes = np.zeros(len(tx), np.int64)
        paths = (_capi.visrt_path * max(npaths, 1))()
        L.visrt_trace_results(self.h, off.ctypes.data, C.cast(paths, C.c_void_p), npaths, nodes.ctypes.data)
        return off, paths, nodes, {"nodes": st.nodes, "sequences": st.sequences, "paths": st.paths,
                                   "leg_tests": st.leg_tests, "ms": st.ms}

    def trace(self, tx: np.ndarray, rx: np.ndarray, allow_diffraction: bool = False, brute_force: bool = False):
        """Per snapshot: list of paths {faces, edge (-1: none), points, length}
        ordered by face sequence, plus per-snapshot node counts and stats."""
        off, paths, nodes, st = self.trace_raw(tx, rx, allow_diffraction=allow_diffraction, brute_force=brute_force)
        out = []
        for k in range(len(off) - 1):
            row = []
            for q in range(off[k], off[k + 1]):
                p = paths[q]
                npts = p.nrefl + 2 + (1 if p.edge >= 0 else 0)
                row.append({"faces": list(p.faces[: p.nrefl]), "edge": int(p.edge),
                            "points": list(p.points[: 3 * npts]), "length": p.length})
            out.append(row)
        return out, nodes, st


def resolve_keys(scene: Scene, tx, rx, keys: Sequence[Sequence[Tuple[Sequence[int], int]]],
                 edges: Optional[Sequence[dict]] = None):
    """resolve_keys (src/raytracer.cpp:554-570) batched: keys[k] = the fixed
    sequences (faces, edge index or -1) to re-solve at sample k (tx[k], rx[k];
    one rx = fixed receiver). Returns per sample the valid paths
    {faces, edge, points, length} in key order, and the stats."""
    tx = np.ascontiguousarray(np.asarray(tx, np.float64).reshape(-1, 3))
    rx = np.ascontiguousarray(np.asarray(rx, np.float64).reshape(-1, 3))
    ns = len(tx)
    flags = 1 if len(rx) == 1 and ns != 1 else 0
    off = np.zeros(ns + 1, np.int64)
    off[1:] = np.cumsum([len(kk) for kk in keys])
    nk = int(off[-1])
    karr = (_capi.visrt_seqkey * max(nk, 1))()
    q = 0
    for kk in keys:
        for faces, edge in kk:
            karr[q].nrefl = len(faces)
            for i, f in enumerate(faces):
                karr[q].faces[i] = int(f)
            karr[q].edge = int(edge)
            q += 1
    ab = np.ascontiguousarray(np.array([list(e["a"]) + list(e["b"]) for e in (edges or [])], np.float64).reshape(-1))
    ok = np.zeros(max(nk, 1), np.uint8)
    paths = (_capi.visrt_path * max(nk, 1))()
    st = _capi.visrt_stats()
    check(lib().visrt_resolve_keys(scene.h, ns, tx.reshape(-1), rx.reshape(-1), flags, off.ctypes.data,
                                   C.cast(karr, C.c_void_p), len(edges or []), ab.ctypes.data if len(ab) else None,
                                   ok.ctypes.data, C.cast(paths, C.c_void_p), C.byref(st), None))
    out = []
    for k in range(ns):
        row = []
        for q in range(off[k], off[k + 1]):
            if not ok[q]:
                continue
            p = paths[q]
            npts = p.nrefl + 2 + (1 if p.edge >= 0 else 0)
            row.append({"faces": list(p.faces[: p.nrefl]), "edge": int(p.edge), "points": list(p.points[: 3 * npts]),
                        "length": p.length})
        out.append(row)
    return out, _stats_dict(st)


def save_matrix_cache(scene: Scene, path: str, admitted_bits: np.ndarray, triples: Optional[np.ndarray] = None,
                      max_order: int = 2) -> None:
    """Binary matrix / pair-graph cache (replaces the text save_matrix,
    src/vismatrix.cpp:849-894): admitted bits + feasible order-2 triples."""
    bits = np.ascontiguousarray(admitted_bits, np.uint64)
    tri = np.ascontiguousarray(np.zeros((0, 3), np.int32) if triples is None else triples, np.int32).reshape(-1, 3)
    check(lib().visrt_cache_save(path.encode(), scene.h, max_order, bits.ctypes.data, len(tri),
                                 tri.ctypes.data if len(tri) else None))


def load_matrix_cache(scene: Scene, path: str):
    """-> (admitted bits [N, words] uint64, triples [T, 3] int32, max_order);
    SceneError if the cache was built for another scene."""
    mo = C.c_int32()
    nt = C.c_int64()
    L = lib()
    check(L.visrt_cache_load(path.encode(), scene.h, C.byref(mo), None, None, 0, C.byref(nt)))
    bits = np.zeros((scene.n, scene.words), np.uint64)
    tri = np.zeros((max(nt.value, 1), 3), np.int32)
    check(L.visrt_cache_load(path.encode(), scene.h, C.byref(mo), bits.ctypes.data, tri.ctypes.data, nt.value,
                             C.byref(nt)))
    return bits, tri[: nt.value], mo.value


def ray_gains(scene: Scene, paths: Sequence[dict], materials, edges: Sequence[dict] = (),
              edge_faces: Sequence[Sequence[int]] = (), frequency: float = 5.5e9, tx_gain_dbi: float = 0.0,
              rx_gain_dbi: float = 0.0, polarization: str = "TE"):
    """rt::ray_gains (include/rt/em.hpp:92-96) on the GPU for a list of paths
    (the dicts Tracer.trace returns). materials: [nfaces][2] (permittivity,
    conductivity). Returns (complex amplitudes, delays)."""
    n = len(paths)
    arr = (_capi.visrt_path * max(n, 1))()
    for q, p in enumerate(paths):
        arr[q].nrefl = len(p["faces"])
        for i, f in enumerate(p["faces"]):
            arr[q].faces[i] = int(f)
        arr[q].edge = int(p.get("edge", -1))
        for i, v in enumerate(p["points"]):
            arr[q].points[i] = float(v)
        arr[q].length = float(p["length"])
    mat = np.ascontiguousarray(np.asarray(materials, np.float64).reshape(-1, 2))
    ab = np.ascontiguousarray(np.array([list(e["a"]) + list(e["b"]) for e in edges], np.float64).reshape(-1))
    ef = np.ascontiguousarray(np.asarray(edge_faces, np.int32).reshape(-1))
    cfg = _capi.visrt_em_config(frequency, tx_gain_dbi, rx_gain_dbi, 1 if polarization == "TM" else 0, 0)
    amp = np.zeros(2 * max(n, 1), np.float64)
    dl = np.zeros(max(n, 1), np.float64)
    st = _capi.visrt_stats()
    check(lib().visrt_ray_gains(scene.h, n, C.cast(arr, C.c_void_p), mat.reshape(-1), len(edges),
                                ab.ctypes.data if len(ab) else None, ef.ctypes.data if len(ef) else None,
                                C.byref(cfg), amp.ctypes.data, dl.ctypes.data, C.byref(st), None))
    return amp[: 2 * n].view(np.complex128), dl[:n]


def channel_stats(scene: Scene, amps: Sequence[np.ndarray], delays: Sequence[np.ndarray]):
    """rt::channel_stats (include/rt/em.hpp:98-101) per snapshot on the GPU:
    (outage, path_loss_db, rms_delay_spread) arrays."""
    ns = len(amps)
    off = np.zeros(ns + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in amps])
    amp = np.ascontiguousarray(np.concatenate([np.asarray(a, np.complex128) for a in amps]) if ns else np.zeros(0, np.complex128))
    dl = np.ascontiguousarray(np.concatenate([np.asarray(d, np.float64) for d in delays]) if ns else np.zeros(0))
    outage = np.zeros(max(ns, 1), np.int8)
    loss = np.zeros(max(ns, 1), np.float64)
    rms = np.zeros(max(ns, 1), np.float64)
    check(lib().visrt_channel_stats(scene.h, ns, off, amp.ctypes.data if len(amp) else None,
                                    dl.ctypes.data if len(dl) else None, outage.ctypes.data, loss.ctypes.data,
                                    rms.ctypes.data, None))
    return outage[:ns].astype(bool), loss[:ns], rms[:ns]


def brute_force_trace(scene: Scene, tx, rx, max_refl: int, allow_diffraction: bool = False,
                      edges: Optional[Sequence[dict]] = None):
    """rt::brute_force_trace (include/rt/raytracer.hpp:78-83): the conventional
    image method — every face but the immediate repeat at every level, no
    chain filter, no image prune — batched over snapshots on the GPU."""
    if max_refl < 0:
        raise _capi.VisibilityError("reflection order must be non-negative")
    zero = np.zeros((scene.n, scene.words), np.uint64)
    tr = Tracer(scene, max_refl, admitted_bits=zero, triples=np.zeros((0, 3), np.int32), edges=edges)
    try:
        return tr.trace(tx, rx, allow_diffraction=allow_diffraction, brute_force=True)
    finally:
        tr.close()


def image_tree(scene: Scene, source, max_depth: int, ids: Optional[Sequence[str]] = None):
    """rt::image_tree (include/rt/raytracer.hpp:51-61): the unfiltered
    front-side mirror hierarchy in the reference's depth-first node order.
    Returns a list of {face, image, parent, depth} (face = id when ``ids``)."""
    src = np.ascontiguousarray(np.asarray(source, np.float64).reshape(3))
    cnt = C.c_int64()
    st = _capi.visrt_stats()
    L = lib()
    check(L.visrt_image_tree(scene.h, src, max_depth, None, None, None, None, 0, C.byref(cnt), C.byref(st), None))
    n = cnt.value
    face = np.zeros(max(n, 1), np.int32)
    parent = np.zeros(max(n, 1), np.int32)
    depth = np.zeros(max(n, 1), np.int32)
    image = np.zeros((max(n, 1), 3), np.float64)
    check(L.visrt_image_tree(scene.h, src, max_depth, face.ctypes.data, parent.ctypes.data, depth.ctypes.data,
                             image.ctypes.data, n, C.byref(cnt), C.byref(st), None))
    return [{"face": ids[face[k]] if ids is not None else int(face[k]), "image": image[k].tolist(),
             "parent": int(parent[k]), "depth": int(depth[k])} for k in range(n)]


def closest_diffraction_edges(scene: Scene, receivers, edges: Sequence[dict]):
    """rt::closest_diffraction_edge (include/rt/vistable.hpp:131-137) for a batch
    of receivers; ``edges`` = the scene's edges in order ({id, a, b}). Returns
    per receiver the edge index or -1."""
    rx = np.ascontiguousarray(np.asarray(receivers, np.float64).reshape(-1, 3))
    ab = np.ascontiguousarray(np.array([list(e["a"]) + list(e["b"]) for e in edges], np.float64).reshape(-1))
    rank = _ranks([e["id"] for e in edges])
    er = np.ascontiguousarray(np.array([rank[e["id"]] for e in edges], np.int32))
    out = np.full(len(rx), -1, np.int32)
    st = _capi.visrt_stats()
    check(lib().visrt_closest_edges(scene.h, len(rx), rx.reshape(-1), len(edges), ab.ctypes.data if len(edges) else None,
                                    er.ctypes.data if len(edges) else None, out, C.byref(st), None))
    return out


def path_identity(ids: Sequence[str], faces: Sequence[int], edge_id: Optional[str] = None) -> str:
    """Path::identity (src/raytracer.cpp:448-456): "LOS" or "R:<face>/.../D:<edge>"."""
    parts = ["R:" + ids[f] for f in faces] + ([f"D:{edge_id}"] if edge_id is not None else [])
    return "LOS" if not parts else "/".join(parts)


def measure_peaks(device: int = 0) -> Tuple[float, float]:
    """(FP64 non-FMA ops/s, FP32 FFMA flop/s) measured on `device`."""
    f64 = C.c_double()
    f32 = C.c_double()
    check(lib().visrt_measure_peaks(device, C.byref(f64), C.byref(f32)))
    return f64.value, f32.value


def unpack_bits(bits: np.ndarray, n: int) -> np.ndarray:
    """[n, words] uint64 -> [n, n] bool."""
    b = bits.view(np.uint8).reshape(n, -1)
    return np.unpackbits(b, axis=1, bitorder="little")[:, :n].astype(bool)


def occlusion_judgment(scene: Scene, ref: int, aim: int) -> Tuple[str, List[int]]:
    """rt::occlusion_judgment (include/rt/vismatrix.hpp:113) on the GPU."""
    kind, blockers, _ = scene.pair_detail([ref], [aim])
    return KIND_NAMES[int(kind[0])], blockers[0]
