"""Order-2 chain growth (build_matrix(scene, 2)'s Markov-2 filter) on the GPU
vs the compiled reference, and the fully GPU-built order-3 trace."""
import numpy as np
import pytest

from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, Tracer, chain_triples, path_identity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    return scenes.workload(1)


def test_chain_triples_config1_vs_reference(oracle_built, cfg1):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup = cfg1.scene
    r = oracle_built.RefOracle(soup)
    ents = r.matrix_entries(r.build_matrix(2))
    exp = sorted({tuple(e["chain"]) for e in ents if e["order"] == 2})
    with Scene(soup) as sc:
        sc.pair_visibility("prefiltered")
        tri, st = chain_triples(sc)
    got = sorted(map(tuple, tri.tolist()))
    assert got == exp
    assert len(got) == st["admitted"]


def test_trace_order3_fully_gpu_config1(oracle_built, cfg1):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup = cfg1.scene
    r = oracle_built.RefOracle(soup)
    m = r.build_matrix(2)
    r.lib().vref_matrix_set_max_order(m, 3)
    acc = r.accel(m, 3)
    with Scene(soup) as sc:
        sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc)
        tr = Tracer(sc, 3, triples=tri)
        sel = list(range(3, len(cfg1.tx), 13))
        paths, nodes, _ = tr.trace(cfg1.tx[sel], cfg1.rx)
    for q, k in enumerate(sel):
        exp, est = r.trace(acc, cfg1.tx[k], cfg1.rx[0])
        got = sorted((path_identity(soup.ids, p["faces"]), p["points"], p["length"]) for p in paths[q])
        assert got == sorted((p["identity"], p["points"], p["length"]) for p in exp), k
        assert nodes[q] == est[0]
