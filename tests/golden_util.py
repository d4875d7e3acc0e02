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
