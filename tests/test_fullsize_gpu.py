"""Parity at the BASELINE sizes (configs 2-5): the GPU runs the full workload;
the CPU oracle / compiled reference re-decides a seeded sample (the full CPU
passes take minutes to days), plus size-independent checks
(symmetry, candidate-list identity)."""
import numpy as np
import pytest

from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import (Scene, Tracer, chain_triples, path_identity, point_regions_array,
                                        unpack_bits)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _sample_pairs(n, m, seed):
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n, 2 * m)
    j = rng.integers(0, n, 2 * m)
    keep = i != j
    return np.minimum(i, j)[keep][:m].astype(np.int32), np.maximum(i, j)[keep][:m].astype(np.int32)


@pytest.mark.parametrize("cfg,m", [(3, 3000), (4, 600)])
def test_matrix_B_sampled(oracle_built, cfg, m):
    soup = scenes.workload(cfg).scene
    with Scene(soup) as sc:
        bits, st = sc.pair_visibility("all")
    M = unpack_bits(bits, soup.nfaces)
    assert np.array_equal(M, M.T)
    pi, pj = _sample_pairs(soup.nfaces, m, 100 + cfg)
    kinds = oracle_built.Oracle(soup).occlusion_batch(pi, pj)
    np.testing.assert_array_equal(M[pi, pj], kinds != 2)


@pytest.mark.parametrize("cfg", [3, 4])
def test_matrix_A_candidates_full(oracle_built, cfg):
    """The full first_order_pair candidate list equals the oracle's; the
    admitted bit of a seeded sample (all of config 4's) is re-decided."""
    soup = scenes.workload(cfg).scene
    o = oracle_built.Oracle(soup)
    with Scene(soup) as sc:
        sc.pair_visibility("prefiltered")
        ci, cj, ad = sc.candidates()
    pi, pj = o.prefilter_all()
    np.testing.assert_array_equal(ci, pi)
    np.testing.assert_array_equal(cj, pj)
    sel = np.arange(len(ci)) if len(ci) < 5000 else np.random.default_rng(5).choice(len(ci), 5000, replace=False)
    kinds = o.occlusion_batch(ci[sel], cj[sel])
    # no degenerate bouncing ranges in these scenes: admitted == not Occluded
    np.testing.assert_array_equal(ad[sel].astype(bool), kinds != 2)


@pytest.mark.parametrize("cfg", [2, 3])
def test_chain_triples_sampled(oracle_built, cfg):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup = scenes.workload(cfg).scene
    with Scene(soup) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, st = chain_triples(sc)
    adm = unpack_bits(bits, soup.nfaces)
    r = oracle_built.RefOracle(soup)
    rng = np.random.default_rng(cfg)
    got = set(map(tuple, tri.tolist()))
    # feasible ones the GPU reports, and random candidate triples of admitted pairs
    for k in rng.choice(len(tri), 300, replace=False):
        assert r.triple_feasible(*map(int, tri[k]))
    ai, aj = np.nonzero(adm)
    for k in rng.choice(len(ai), 300, replace=False):
        p, t = int(ai[k]), int(aj[k])
        aims = np.nonzero(adm[t])[0]
        a = int(aims[rng.integers(len(aims))])
        assert r.triple_feasible(p, t, a) == ((p, t, a) in got), (p, t, a)


@pytest.mark.parametrize("cfg,nsrc,nface", [(3, 4, 120), (5, 3, 80)])
def test_regions_sampled(oracle_built, cfg, nsrc, nface):
    wl = scenes.workload(cfg)
    soup = wl.scene
    rng = np.random.default_rng(cfg)
    src = np.concatenate([wl.tx[rng.choice(len(wl.tx), nsrc // 2 + 1)], wl.rx[rng.choice(len(wl.rx), nsrc // 2)]])
    with Scene(soup) as sc:
        arr, _ = point_regions_array(sc, src)
    o = oracle_built.Oracle(soup)
    # every present region plus a random sample of the rest
    for k in range(len(src)):
        faces = set(np.nonzero(arr[k]["present"] == 1)[0][:nface].tolist())
        faces |= set(rng.choice(soup.nfaces, nface, replace=False).tolist())
        for f in sorted(faces):
            e = o.illuminated_region(src[k], f)
            g = arr[k, f]
            assert (int(g["present"]), [int(x) for x in g["has"]], [int(x) for x in g["clipped"]],
                    [float(x) for x in g["sub"]]) == (e["present"], e["has"], e["clipped"], e["sub"]), (k, f)


@pytest.mark.parametrize("cfg,nsnap", [(3, 2), (5, 3)])
def test_trace_order3_sampled(oracle_built, cfg, nsnap):
    """Order-3 image trees with the GPU chain filter ((A) bits + K7 chains,
    both pinned above) vs the oracle restatement on the same filter."""
    wl = scenes.workload(cfg)
    soup = wl.scene
    rng = np.random.default_rng(cfg)
    ks = sorted(rng.choice(len(wl.tx), nsnap, replace=False).tolist())
    with Scene(soup) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc)
        tr = Tracer(sc, 3, admitted_bits=bits, triples=tri)
        paths, nodes, _ = tr.trace(wl.tx[ks], wl.rx[ks])
    adm = unpack_bits(bits, soup.nfaces)
    filt = oracle_built.chain_filter_arrays(soup.nfaces, np.nonzero(adm), tri)
    o = oracle_built.Oracle(soup)
    for q, k in enumerate(ks):
        exp, est = o.trace(filt, 3, wl.tx[k], wl.rx[k])
        key = lambda p: (len(p["faces"]), tuple(p["faces"]), tuple(p["points"]), p["length"])
        assert sorted(map(key, paths[q])) == sorted(map(key, exp))
        assert nodes[q] == est[0]


def test_matrix_config2_full_vs_reference(oracle_built):
    """The WHOLE config-2 matrix against the unmodified reference (oracle/_ref,
    all host threads): (B) occlusion_judgment on all 788,140 pairs and (A)
    build_matrix(scene, 1).pair_admitted — bit-identical, no sampling."""
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup = scenes.workload(2).scene
    n = soup.nfaces
    with Scene(soup) as sc:
        bits_b, _ = sc.pair_visibility("all")
        bits_a, _ = sc.pair_visibility("prefiltered")
    r = oracle_built.RefOracle(soup)
    pi, pj = np.triu_indices(n, 1)
    kinds = r.occlusion_batch(pi.astype(np.int32), pj.astype(np.int32))
    M = unpack_bits(bits_b, n)
    np.testing.assert_array_equal(M[pi, pj], kinds != 2)
    adm = np.zeros((n, n), bool)
    for e in r.matrix_entries(r.build_matrix(1)):
        if e["order"] == 1:
            adm[e["chain"][0], e["chain"][1]] = True
    np.testing.assert_array_equal(unpack_bits(bits_a, n), adm)
