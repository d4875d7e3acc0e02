"""Load the committed golden fixtures (tests/golden/*.json, made by
tests/golden/make_golden.py from the compiled reference)."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2501_02747_b200.scenes import FacetSoup

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = ["two_buildings", "street_canyon", "screened_wall", "open_field", "manhattan", "config1"]


def load(name: str) -> dict:
    with open(os.path.join(GOLDEN, name + ".json")) as fh:
        return json.load(fh)


def unhex(v):
    if isinstance(v, list):
        return [unhex(x) for x in v]
    return float.fromhex(v)


def soup(d: dict, with_buildings: bool = True) -> FacetSoup:
    faces = d["faces"]
    off = np.zeros(len(faces) + 1, np.int32)
    off[1:] = np.cumsum([len(f["pts"]) for f in faces])
    verts = np.array([p for f in faces for p in f["pts"]], np.float64).reshape(-1, 3)
    b = np.array([f["building"] for f in faces], np.int32)
    return FacetSoup(ids=[f["id"] for f in faces], vert_off=off, verts=verts,
                     building=b if with_buildings and (b >= 0).any() else None, name=d["name"])


def pairs(n: int):
    pi, pj = np.triu_indices(n, 1)
    return pi.astype(np.int32), pj.astype(np.int32)


def kinds(d: dict) -> np.ndarray:
    return np.frombuffer(d["kinds"].encode(), np.uint8) - ord("0")


def admitted_matrix(d: dict) -> np.ndarray:
    n = len(d["faces"])
    m = np.zeros((n, n), bool)
    for e in d["matrix1"]:
        m[e["ref"], e["aim"]] = True
    return m


def region_tuple(row):
    present, has, clipped, sub = row
    return (int(present), list(has), list(clipped), unhex(sub))


def region_canonical(P, H, Cl, S):
    """Canonical bytes of one source's regions over all faces (present int8
    [n], has/clipped int8 [n,3], sub float64 [n,6]): fields that the present /
    has flags make meaningless are zeroed, so the reference's and the GPU's
    arrays hash alike exactly when every bit-exact field agrees."""
    P = np.ascontiguousarray(P, np.int8)
    pres = (P == 1)[:, None]
    H2 = np.where(pres, np.asarray(H, np.int8), 0).astype(np.int8)
    hb = H2.astype(bool)
    Cl2 = np.where(hb, np.asarray(Cl, np.int8), 0).astype(np.int8)
    S2 = np.where(np.repeat(hb, 2, axis=1), np.asarray(S, np.float64), 0.0)
    return P.tobytes() + H2.tobytes() + Cl2.tobytes() + np.ascontiguousarray(S2, np.float64).tobytes()


def region_digest(P, H, Cl, S) -> str:
    import hashlib
    return hashlib.sha256(region_canonical(P, H, Cl, S)).hexdigest()
