"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* :class:`Oracle`   — the C restatement (oracle/_build/libvisrt_oracle.so).
* :class:`RefOracle` — the compiled, unmodified reference behind the facet-soup
  adapter (oracle/_ref/libvisrt_ref.so, built from /root/reference by
  oracle/Makefile; the built .so travels to the GPU box, the sources do not).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libvisrt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvisrt_ref.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the checkers (the reference only where /root/reference exists)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8"] + targets, check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


class vo_region(C.Structure):
    _fields_ = [("present", C.c_int32), ("has", C.c_int32 * 3), ("clipped", C.c_int32 * 3),
                ("sub", C.c_double * 6)]


class vo_path(C.Structure):
    _fields_ = [("nrefl", C.c_int32), ("faces", C.c_int32 * 4), ("points", C.c_double * 18),
                ("length", C.c_double)]


_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def chain_filter_arrays(n: int, admitted, triples=None):
    """Chain filter in the oracle's layout: the admitted aims as CSR (off1,
    idx1 ascending per face) and the order-2 continuations as CSR over the
    directed admitted pairs in the same order. `admitted`: [n, n] bool matrix
    or an (i, j) pair list of directed admitted pairs; `triples`: (p, t, a)
    order-2 chains (None: order <= 2 only)."""
    if isinstance(admitted, np.ndarray) and admitted.ndim == 2 and admitted.shape == (n, n):
        pi, pj = np.nonzero(admitted)
    else:
        pi, pj = (np.asarray(x) for x in admitted)
        o = np.lexsort((pj, pi))
        pi, pj = pi[o], pj[o]
    pi = pi.astype(np.int64)
    pj = pj.astype(np.int32)
    off1 = np.zeros(n + 1, np.int64)
    np.add.at(off1, pi + 1, 1)
    off1 = np.cumsum(off1)
    idx1 = np.ascontiguousarray(pj if len(pj) else np.zeros(1, np.int32), np.int32)
    off2 = np.zeros(len(pj) + 1, np.int64)
    idx2 = np.zeros(1, np.int32)
    if triples is not None and len(triples):
        t = np.asarray(triples, np.int64).reshape(-1, 3)
        key = pi * n + pj
        rank = np.searchsorted(key, t[:, 0] * n + t[:, 1])
        o = np.lexsort((t[:, 2], rank))
        rank, aim = rank[o], t[o, 2]
        keep = np.ones(len(rank), bool)
        keep[1:] = (rank[1:] != rank[:-1]) | (aim[1:] != aim[:-1])
        rank, aim = rank[keep], aim[keep]
        np.add.at(off2, rank + 1, 1)
        off2 = np.cumsum(off2)
        idx2 = np.ascontiguousarray(aim.astype(np.int32))
    return (np.ascontiguousarray(off1), idx1, np.ascontiguousarray(off2), idx2)


class Oracle:
    """C restatement of the reference hot path (see oracle/visrt_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            L = C.CDLL(ORACLE_SO)
            L.vo_scene_create.restype = C.c_void_p
            L.vo_scene_create.argtypes = [C.c_int32, _i32p, _f64p]
            L.vo_scene_free.argtypes = [C.c_void_p]
            L.vo_face_info.argtypes = [C.c_void_p, C.c_int32, _f64p, C.POINTER(C.c_int32)]
            L.vo_plane_segment.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _f64p]
            L.vo_segment_hits_face.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int32]
            L.vo_mutually_front.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vo_required_planes.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vo_prefilter.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vo_occlusion.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _i32p, C.c_int32,
                                       C.POINTER(C.c_int32)]
            L.vo_occlusion_batch.argtypes = [C.c_void_p, C.c_int64, _i32p, _i32p, _i8p, C.c_int32]
            L.vo_sightline_count.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vo_illuminated_region.argtypes = [C.c_void_p, _f64p, C.c_int32, C.POINTER(vo_region)]
            L.vo_prefilter_all.restype = C.c_int64
            L.vo_prefilter_all.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]
            L.vo_trace.restype = C.c_int64
            L.vo_trace.argtypes = [C.c_void_p, _i64p, _i32p, _i64p, _i32p, C.c_int32, _f64p, _f64p,
                                   C.POINTER(vo_path), C.c_int64, _i64p]
            cls._lib = L
        return cls._lib

    def __init__(self, soup) -> None:
        L = self.lib()
        self.soup = soup
        self.n = soup.nfaces
        self.h = L.vo_scene_create(self.n, np.ascontiguousarray(soup.vert_off, dtype=np.int32),
                                   np.ascontiguousarray(soup.verts, dtype=np.float64).reshape(-1))
        if not self.h:
            raise ValueError("oracle rejected the facet soup")

    def __del__(self):
        if getattr(self, "h", None) and self._lib is not None:
            self._lib.vo_scene_free(self.h)
            self.h = None

    def orientation(self) -> np.ndarray:
        out = np.zeros(self.n, np.int32)
        nrm = np.zeros(3)
        o = C.c_int32()
        for i in range(self.n):
            self.lib().vo_face_info(self.h, i, nrm, C.byref(o))
            out[i] = o.value
        return out

    def plane_segment(self, i: int, plane: int):
        o = np.zeros(6)
        return o if self.lib().vo_plane_segment(self.h, i, plane, o) else None

    def prefilter(self, i: int, j: int) -> bool:
        return bool(self.lib().vo_prefilter(self.h, i, j))

    def required_planes(self, i: int, j: int) -> int:
        return int(self.lib().vo_required_planes(self.h, i, j))

    def prefilter_all(self, threads: int = 0):
        """(i, j) of every pair passing first_order_pair's gate, in order."""
        L = self.lib()
        th = threads or os.cpu_count() or 1
        m = L.vo_prefilter_all(self.h, None, None, 0, th)
        pi = np.zeros(m, np.int32)
        pj = np.zeros(m, np.int32)
        L.vo_prefilter_all(self.h, pi.ctypes.data, pj.ctypes.data, m, th)
        return pi, pj

    def occlusion(self, i: int, j: int):
        buf = np.zeros(max(self.n, 1), np.int32)
        nb = C.c_int32()
        k = self.lib().vo_occlusion(self.h, i, j, buf, len(buf), C.byref(nb))
        return int(k), buf[: nb.value].tolist()

    def occlusion_batch(self, pi: np.ndarray, pj: np.ndarray, threads: int = 0) -> np.ndarray:
        pi = np.ascontiguousarray(pi, np.int32)
        pj = np.ascontiguousarray(pj, np.int32)
        out = np.zeros(len(pi), np.int8)
        self.lib().vo_occlusion_batch(self.h, len(pi), pi, pj, out, threads or os.cpu_count() or 1)
        return out

    def sightline_count(self, i: int, j: int) -> int:
        return int(self.lib().vo_sightline_count(self.h, i, j))

    def illuminated_region(self, src, face: int) -> dict:
        r = vo_region()
        self.lib().vo_illuminated_region(self.h, np.ascontiguousarray(src, np.float64), face, C.byref(r))
        return {"present": r.present, "has": list(r.has), "clipped": list(r.clipped), "sub": list(r.sub)}

    def trace(self, filt, max_refl: int, tx, rx):
        """TraceAccelerator::trace (no diffraction) with the chain filter
        `filt` = chain_filter_arrays(...). Returns (paths, stats) with paths
        as dicts {faces, points, length}; stats = nodes, sequences, paths."""
        off1, idx1, off2, idx2 = filt
        cap = 1 << 16
        out = (vo_path * cap)()
        st = np.zeros(3, np.int64)
        n = self.lib().vo_trace(self.h, off1, idx1, off2, idx2, max_refl,
                                np.ascontiguousarray(tx, np.float64), np.ascontiguousarray(rx, np.float64),
                                out, cap, st)
        if n < 0:
            raise ValueError("PlacementError: transmitter and receiver coincide")
        paths = [{"faces": list(out[k].faces[: out[k].nrefl]),
                  "points": list(out[k].points[: 3 * (out[k].nrefl + 2)]), "length": out[k].length}
                 for k in range(min(n, cap))]
        return paths, st


# ---------------------------------------------------------------------------
# compiled reference (oracle/_ref)
# ---------------------------------------------------------------------------

class vref_entry(C.Structure):
    _fields_ = [("order", C.c_int32), ("chain", C.c_int32 * 5), ("chain_len", C.c_int32),
                ("plane", C.c_int32), ("kind", C.c_int32), ("verdict", C.c_int32),
                ("has_criterion", C.c_int32), ("nblockers", C.c_int32), ("nsub", C.c_int32),
                ("naim_image", C.c_int32), ("ranges", C.c_double * 12), ("criterion", C.c_double * 4),
                ("sub", C.c_double * 8), ("aim_image", C.c_double * 24), ("blockers", C.c_int32 * 64),
                ("edge_a", C.c_char * 64), ("edge_b", C.c_char * 64)]


class vref_region(C.Structure):
    _fields_ = [("present", C.c_int32), ("nplanes", C.c_int32), ("plane", C.c_int32 * 3),
                ("clipped", C.c_int32 * 3), ("sub", C.c_double * 6), ("image", C.c_double * 6),
                ("sub_ab", C.c_double * 12), ("angles", C.c_double * 12)]


class vref_row(C.Structure):
    _fields_ = [("order", C.c_int32), ("chain", C.c_int32 * 4), ("chain_len", C.c_int32),
                ("aim", C.c_int32), ("plane", C.c_int32), ("verdict", C.c_int32),
                ("ref_display", C.c_char * 32), ("aim_display", C.c_char * 32),
                ("parent_display", C.c_char * 32)]


class vref_mobile_row(C.Structure):
    _fields_ = [("order", C.c_int32), ("pad", C.c_int32), ("s_start", C.c_double), ("s_end", C.c_double),
                ("node", C.c_char * 64), ("node_display", C.c_char * 64), ("label_start", C.c_char * 16),
                ("label_end", C.c_char * 16), ("parent", C.c_char * 64), ("blockage", C.c_char * 64)]


class vref_dyn_sample(C.Structure):
    _fields_ = [("s", C.c_double), ("segment", C.c_int32), ("retraced", C.c_int32), ("npaths", C.c_int32),
                ("first", C.c_int32)]


class vref_path(C.Structure):
    _fields_ = [("ninter", C.c_int32), ("face", C.c_int32 * 6), ("is_diff", C.c_int32 * 6),
                ("points", C.c_double * 24), ("length", C.c_double), ("delay", C.c_double),
                ("identity", C.c_char * 256)]


class RefOracle:
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} missing (built by oracle/Makefile where "
                                        "/root/reference exists)")
            L = C.CDLL(REF_SO)
            L.vref_last_error.restype = C.c_char_p
            L.vref_scene_from_soup.restype = C.c_void_p
            L.vref_scene_from_soup.argtypes = [C.c_int32, _i32p, _f64p, C.c_char_p]
            L.vref_scene_load.restype = C.c_void_p
            L.vref_scene_load.argtypes = [C.c_char_p]
            L.vref_scene_free.argtypes = [C.c_void_p]
            L.vref_nfaces.argtypes = [C.c_void_p]
            L.vref_nedges.argtypes = [C.c_void_p]
            L.vref_face_export.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32, C.c_char_p,
                                           C.c_int32, C.c_char_p, C.c_char_p, C.c_int32, _f64p,
                                           C.c_int32, _f64p]
            L.vref_edge_export.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32, _f64p]
            L.vref_occlusion.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _i32p, C.c_int32,
                                         C.POINTER(C.c_int32)]
            L.vref_occlusion_batch.argtypes = [C.c_void_p, C.c_int64, _i32p, _i32p, _i8p, C.c_int32]
            L.vref_mutually_front.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vref_required_planes.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
            L.vref_plane_segment.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _f64p]
            L.vref_triple_feasible.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]
            L.vref_segment_hits_face.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int32]
            L.vref_segments_blocked.argtypes = [C.c_void_p, C.c_int64, _f64p, _f64p, _u8p, C.c_int32]
            L.vref_build_matrix.restype = C.c_void_p
            L.vref_build_matrix.argtypes = [C.c_void_p, C.c_int32]
            L.vref_matrix_free.argtypes = [C.c_void_p]
            L.vref_matrix_set_max_order.argtypes = [C.c_void_p, C.c_int32]
            L.vref_matrix_size.restype = C.c_int64
            L.vref_matrix_size.argtypes = [C.c_void_p]
            L.vref_matrix_entry.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(vref_entry)]
            L.vref_matrix_chains.restype = C.c_int64
            L.vref_matrix_chains.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _i32p, C.c_int64]
            L.vref_illuminated_region.argtypes = [C.c_void_p, _f64p, C.c_int32, C.POINTER(vref_region)]
            L.vref_regions_batch.argtypes = [C.c_void_p, C.c_int64, _f64p, _i32p, C.POINTER(vref_region),
                                             C.c_int32]
            L.vref_point_vis_table.restype = C.c_int64
            L.vref_point_vis_table.argtypes = [C.c_void_p, C.c_void_p, _f64p, C.c_int32,
                                               C.POINTER(vref_row), C.c_int64]
            L.vref_accel_create.restype = C.c_void_p
            L.vref_accel_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
            L.vref_accel_free.argtypes = [C.c_void_p]
            L.vref_accel_trace.restype = C.c_int64
            L.vref_accel_trace.argtypes = [C.c_void_p, C.c_void_p, _f64p, _f64p, C.c_int32,
                                           C.POINTER(vref_path), C.c_int64, _i64p]
            L.vref_brute_trace.restype = C.c_int64
            L.vref_brute_trace.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int32, C.c_int32,
                                           C.POINTER(vref_path), C.c_int64, _i64p]
            L.vref_accel_trace_batch.restype = C.c_int64
            L.vref_accel_trace_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, _f64p, _f64p,
                                                 C.c_int32, C.c_int32, _i64p, _i64p]
            L.vref_scene_from_shells.restype = C.c_void_p
            L.vref_scene_from_shells.argtypes = [C.c_int32, _i32p, _f64p, C.c_char_p, _i32p, C.c_int32,
                                                 C.c_char_p]
            L.vref_closest_edge.argtypes = [C.c_void_p, _f64p]
            L.vref_face_material.argtypes = [C.c_void_p, C.c_int32, _f64p]
            L.vref_edge_faces.argtypes = [C.c_void_p, C.c_int32, _i32p]
            L.vref_trace_em.restype = C.c_int64
            L.vref_trace_em.argtypes = [C.c_void_p, C.c_void_p, _f64p, _f64p, C.c_int32, C.c_double, C.c_double,
                                        C.c_double, C.c_int32, _f64p, _f64p, _f64p, C.c_int64]
            L.vref_dynamic_trace.restype = C.c_int64
            L.vref_dynamic_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _f64p, _f64p, C.c_int32, C.c_int32,
                                             C.c_double, C.POINTER(vref_dyn_sample), C.c_int64, C.POINTER(vref_path),
                                             C.c_int64, C.POINTER(C.c_int64)]
            L.vref_trajectory_table.restype = C.c_int64
            L.vref_trajectory_table.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _f64p, C.c_int32,
                                                C.POINTER(vref_mobile_row), C.c_int64]
            L.vref_image_tree.restype = C.c_int64
            L.vref_image_tree.argtypes = [C.c_void_p, _f64p, C.c_int32, _i32p, _i32p, _i32p, _f64p,
                                          C.c_int64]
            cls._lib = L
        return cls._lib

    def __init__(self, soup=None, path: Optional[str] = None) -> None:
        L = self.lib()
        if path is not None:
            self.h = L.vref_scene_load(path.encode())
        elif getattr(soup, "building", None) is not None and getattr(soup, "building_ids", None):
            # closed shells through the reference's own Scene::finalize
            ids = b"".join(s.encode() + b"\0" for s in soup.ids)
            bids = b"".join(s.encode() + b"\0" for s in soup.building_ids)
            self.h = L.vref_scene_from_shells(soup.nfaces, np.ascontiguousarray(soup.vert_off, np.int32),
                                              np.ascontiguousarray(soup.verts, np.float64).reshape(-1), ids,
                                              np.ascontiguousarray(soup.building, np.int32),
                                              len(soup.building_ids), bids)
        else:
            ids = b"".join(s.encode() + b"\0" for s in soup.ids)
            self.h = L.vref_scene_from_soup(soup.nfaces, np.ascontiguousarray(soup.vert_off, np.int32),
                                            np.ascontiguousarray(soup.verts, np.float64).reshape(-1), ids)
        if not self.h:
            raise RuntimeError("reference scene: " + L.vref_last_error().decode())
        self.n = L.vref_nfaces(self.h)
        self._matrices = []

    def __del__(self):
        if getattr(self, "h", None) and self._lib is not None:
            for m in self._matrices:
                self._lib.vref_matrix_free(m)
            self._lib.vref_scene_free(self.h)
            self.h = None

    # -- scene export (fixture conversion) -----------------------------------
    def export(self):
        L = self.lib()
        faces = []
        for i in range(self.n):
            fid, bld, lx, lv = (C.create_string_buffer(128) for _ in range(4))
            pts = np.zeros(3 * 64)
            nrm = np.zeros(3)
            nv = L.vref_face_export(self.h, i, fid, 128, bld, 128, lx, lv, 128, pts, 64, nrm)
            faces.append({"id": fid.value.decode(), "building": bld.value.decode(),
                          "label_xy": lx.value.decode(), "label_vert": lv.value.decode(),
                          "pts": pts[: 3 * nv].reshape(nv, 3).tolist(), "normal": nrm.tolist()})
        edges = []
        for e in range(L.vref_nedges(self.h)):
            eid = C.create_string_buffer(128)
            ab = np.zeros(6)
            L.vref_edge_export(self.h, e, eid, 128, ab)
            edges.append({"id": eid.value.decode(), "a": ab[:3].tolist(), "b": ab[3:].tolist()})
        return faces, edges

    # -- (1) ----------------------------------------------------------------
    def occlusion(self, i: int, j: int):
        buf = np.zeros(max(self.n, 1), np.int32)
        nb = C.c_int32()
        k = self.lib().vref_occlusion(self.h, i, j, buf, len(buf), C.byref(nb))
        if k < 0:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return int(k), buf[: nb.value].tolist()

    def occlusion_batch(self, pi, pj, threads: int = 0) -> np.ndarray:
        pi = np.ascontiguousarray(pi, np.int32)
        pj = np.ascontiguousarray(pj, np.int32)
        out = np.zeros(len(pi), np.int8)
        self.lib().vref_occlusion_batch(self.h, len(pi), pi, pj, out, threads or os.cpu_count() or 1)
        return out

    def segments_blocked(self, a, b, threads: int = 0) -> np.ndarray:
        """sightline_clear's negation for a batch of segments (any face hits)."""
        a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, 3))
        b = np.ascontiguousarray(np.asarray(b, np.float64).reshape(-1, 3))
        out = np.zeros(len(a), np.uint8)
        self.lib().vref_segments_blocked(self.h, len(a), a.reshape(-1), b.reshape(-1), out,
                                         threads or os.cpu_count() or 1)
        return out.astype(bool)

    def mutually_front(self, i, j) -> bool:
        return bool(self.lib().vref_mutually_front(self.h, i, j))

    def triple_feasible(self, p: int, t: int, a: int) -> bool:
        """build_matrix's triple_ext feasibility through the reference's public functions."""
        r = self.lib().vref_triple_feasible(self.h, p, t, a)
        if r < 0:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return bool(r)

    def required_planes(self, i, j) -> int:
        return int(self.lib().vref_required_planes(self.h, i, j))

    def plane_segment(self, i: int, plane: int):
        o = np.zeros(6)
        return o if self.lib().vref_plane_segment(self.h, i, plane, o) else None

    def build_matrix(self, order: int):
        m = self.lib().vref_build_matrix(self.h, order)
        if not m:
            raise RuntimeError(self.lib().vref_last_error().decode())
        self._matrices.append(m)
        return m

    def matrix_chains(self, m, order: int) -> np.ndarray:
        """Chains (face indices) of every entry of one order, [k][order + 1]."""
        L = self.lib()
        n = L.vref_matrix_chains(self.h, m, order, np.zeros(1, np.int32), 0)
        out = np.zeros((max(n, 1), order + 1), np.int32)
        L.vref_matrix_chains(self.h, m, order, out, n)
        return out[:n]

    def matrix_entries(self, m) -> List[dict]:
        L = self.lib()
        out = []
        e = vref_entry()
        for k in range(L.vref_matrix_size(m)):
            L.vref_matrix_entry(self.h, m, k, C.byref(e))
            out.append({"order": e.order, "chain": list(e.chain[: e.chain_len]), "plane": e.plane,
                        "kind": e.kind, "verdict": e.verdict, "has_criterion": e.has_criterion,
                        "ranges": list(e.ranges), "criterion": list(e.criterion),
                        "sub": list(e.sub[: 2 * e.nsub]), "blockers": list(e.blockers[: e.nblockers]),
                        "aim_image": list(e.aim_image[: 3 * e.naim_image]),
                        "edge_a": e.edge_a.decode(), "edge_b": e.edge_b.decode()})
        return out

    # -- (2) ----------------------------------------------------------------
    def illuminated_region(self, src, face: int) -> dict:
        r = vref_region()
        self.lib().vref_illuminated_region(self.h, np.ascontiguousarray(src, np.float64), face, C.byref(r))
        return _region_dict(r)

    def regions_batch(self, src: np.ndarray, face: np.ndarray, threads: int = 0) -> List[dict]:
        n = len(face)
        arr = (vref_region * n)()
        self.lib().vref_regions_batch(self.h, n, np.ascontiguousarray(src, np.float64).reshape(-1),
                                      np.ascontiguousarray(face, np.int32), arr, threads or os.cpu_count() or 1)
        return [_region_dict(arr[k]) for k in range(n)]

    def point_vis_table(self, m, src, max_order: int) -> List[dict]:
        L = self.lib()
        cap = 1 << 16
        rows = (vref_row * cap)()
        n = L.vref_point_vis_table(self.h, m, np.ascontiguousarray(src, np.float64), max_order, rows, cap)
        if n < 0:
            raise RuntimeError(L.vref_last_error().decode())
        return [{"order": r.order, "chain": list(r.chain[: r.chain_len]), "aim": r.aim, "plane": r.plane,
                 "verdict": r.verdict, "ref_display": r.ref_display.decode(),
                 "aim_display": r.aim_display.decode(), "parent_display": r.parent_display.decode()}
                for r in rows[:n]]

    def image_tree(self, src, depth: int):
        L = self.lib()
        src = np.ascontiguousarray(src, np.float64)
        cap = 1 << 22
        face, parent, dep = (np.zeros(cap, np.int32) for _ in range(3))
        image = np.zeros(3 * cap, np.float64)
        n = L.vref_image_tree(self.h, src, depth, face, parent, dep, image, cap)
        return face[:n], parent[:n], dep[:n], image[:3 * n].reshape(n, 3)

    def dynamic_trace(self, m, waypoints, rx, max_refl: int, diffraction: bool, step: float):
        """rt::dynamic_trace (fixed receiver): samples with their paths."""
        L = self.lib()
        scap, pcap = 1 << 14, 1 << 18
        smp = (vref_dyn_sample * scap)()
        pth = (vref_path * pcap)()
        npth = C.c_int64()
        wp = np.ascontiguousarray(np.asarray(waypoints, np.float64)[:, :3]).reshape(-1)
        ns = L.vref_dynamic_trace(self.h, m, len(wp) // 3, wp, np.ascontiguousarray(rx, np.float64), max_refl,
                                  int(diffraction), step, smp, scap, pth, pcap, C.byref(npth))
        if ns < 0:
            raise RuntimeError(L.vref_last_error().decode())
        out = []
        for k in range(ns):
            d = smp[k]
            ps = [pth[d.first + q] for q in range(d.npaths)]
            out.append({"s": d.s, "segment": d.segment, "retraced": bool(d.retraced),
                        "paths": [{"identity": p.identity.decode(), "points": list(p.points[: 3 * (p.ninter + 2)]),
                                   "length": p.length} for p in ps]})
        return out

    def face_materials(self):
        out = np.zeros((self.n, 2), np.float64)
        for i in range(self.n):
            v = np.zeros(2, np.float64)
            self.lib().vref_face_material(self.h, i, v)
            out[i] = v
        return out

    def edge_faces(self):
        L = self.lib()
        out = []
        for e in range(L.vref_nedges(self.h)):
            f2 = np.zeros(2, np.int32)
            L.vref_edge_faces(self.h, e, f2)
            out.append(f2.tolist())
        return out

    def trace_em(self, accel, tx, rx, diffraction, freq, tx_gain, rx_gain, tm):
        cap = 1 << 14
        amp = np.zeros(2 * cap, np.float64)
        dl = np.zeros(cap, np.float64)
        st = np.zeros(3, np.float64)
        n = self.lib().vref_trace_em(self.h, accel, np.ascontiguousarray(tx, np.float64),
                                     np.ascontiguousarray(rx, np.float64), int(diffraction), freq, tx_gain, rx_gain,
                                     int(tm), amp, dl, st, cap)
        if n < 0:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return amp[: 2 * n].reshape(n, 2), dl[:n], st

    def closest_edge(self, rx) -> int:
        return int(self.lib().vref_closest_edge(self.h, np.ascontiguousarray(rx, np.float64)))

    def trajectory_vis_table(self, m, waypoints, max_order: int) -> List[dict]:
        """rt::trajectory_vis_table rows (proj/src/vistable.cpp:822-960)."""
        L = self.lib()
        cap = 1 << 16
        rows = (vref_mobile_row * cap)()
        wp = np.ascontiguousarray(np.asarray(waypoints, np.float64)[:, :3]).reshape(-1)
        n = L.vref_trajectory_table(self.h, m, len(wp) // 3, wp, max_order, rows, cap)
        if n < 0:
            raise RuntimeError(L.vref_last_error().decode())
        return [{"order": r.order, "node": r.node.decode(), "node_display": r.node_display.decode(),
                 "s_start": r.s_start, "s_end": r.s_end, "label_start": r.label_start.decode(),
                 "label_end": r.label_end.decode(), "parent": r.parent.decode(), "blockage": r.blockage.decode()}
                for r in rows[:n]]

    # -- (3) ----------------------------------------------------------------
    def accel(self, m, max_refl: int):
        a = self.lib().vref_accel_create(self.h, m, max_refl)
        if not a:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return a

    def trace(self, accel, tx, rx, diffraction: bool = False):
        cap = 1 << 14
        out = (vref_path * cap)()
        st = np.zeros(4, np.int64)
        n = self.lib().vref_accel_trace(self.h, accel, np.ascontiguousarray(tx, np.float64),
                                        np.ascontiguousarray(rx, np.float64), int(diffraction), out, cap, st)
        if n < 0:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return [_path_dict(out[k]) for k in range(n)], st

    def brute_trace(self, tx, rx, max_refl: int, diffraction: bool = False):
        cap = 1 << 14
        out = (vref_path * cap)()
        st = np.zeros(4, np.int64)
        n = self.lib().vref_brute_trace(self.h, np.ascontiguousarray(tx, np.float64),
                                        np.ascontiguousarray(rx, np.float64), max_refl, int(diffraction),
                                        out, cap, st)
        if n < 0:
            raise RuntimeError(self.lib().vref_last_error().decode())
        return [_path_dict(out[k]) for k in range(n)], st


def _region_dict(r) -> dict:
    d = {"present": r.present, "has": [0, 0, 0], "clipped": [0, 0, 0], "sub": [0.0] * 6,
         "image": [0.0] * 6, "sub_ab": [0.0] * 12}
    for p in range(r.nplanes):
        t = r.plane[p]
        d["has"][t] = 1
        d["clipped"][t] = r.clipped[p]
        d["sub"][2 * t], d["sub"][2 * t + 1] = r.sub[2 * p], r.sub[2 * p + 1]
        d["image"][2 * t], d["image"][2 * t + 1] = r.image[2 * p], r.image[2 * p + 1]
        d["sub_ab"][4 * t: 4 * t + 4] = list(r.sub_ab[4 * p: 4 * p + 4])
    return d


def _path_dict(p) -> dict:
    return {"faces": [p.face[q] for q in range(p.ninter)], "is_diff": [p.is_diff[q] for q in range(p.ninter)],
            "points": list(p.points[: 3 * (p.ninter + 2)]), "length": p.length,
            "identity": p.identity.decode()}
