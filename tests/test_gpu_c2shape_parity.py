"""Search parity at config-2 shape against the UNMODIFIED reference
(tests/golden/make_c2shape_golden.py): 100k x 768 seeded embeddings
(tests/golden/c2shape.py), GPU-built graph (M=32, hub 2%) and PQ m=64 that
the reference's own load_graph/load_pq validated, the reference's run_search
over MatrixSource(E) for 256 queries at (k=3, ef=64, 30%) and (k=10, ef=96,
70%). Device ids, distance bits and counters must be identical — with host
np.dot query norms and with the device ones."""
from __future__ import annotations

import json
import sys

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
FIX = GOLDEN / "c2shape"


@pytest.fixture(scope="module")
def fx():
    import __graft_entry__ as ge
    ge.build()
    sys.path.insert(0, str(GOLDEN))
    import c2shape
    import paper_2506_08276_b200 as lv
    meta = json.loads((FIX / "reference_results.json").read_text())
    E, Q = c2shape.make()
    return dict(lv=lv, meta=meta, E=E, Q=Q[:meta["n_queries"]], g=lv.load_graph(FIX / "graph.bin"),
                pq=lv.load_pq(FIX / "pq.bin"))


@pytest.mark.parametrize("device_qn", [False, True])
def test_c2shape_matrix_mode_bit_exact(fx, device_qn):
    import torch
    lv = fx["lv"]
    model, codes = fx["pq"]
    dev = lv.search.device_index_for(fx["g"], model, codes)
    Et = torch.from_numpy(fx["E"]).cuda()
    Qt = torch.from_numpy(fx["Q"]).cuda()
    qn = None if device_qn else torch.from_numpy(lv.search.query_norms(fx["Q"])).cuda()
    for case in fx["meta"]["cases"]:
        out = dev.search_device(Qt, lv.SearchParams(**case["params"]), lv.MatrixSource(Et), qn=qn)
        ids = out["ids"].cpu().numpy()
        dist = out["dist"].cpu().numpy().view(np.uint32)
        cnt = out["counters"].cpu().numpy()
        for b, exp in enumerate(case["reports"]):
            assert list(ids[b]) == exp["ids"], (case["params"], b)
            assert list(dist[b]) == exp["dist"], (case["params"], b)
            assert cnt[b, 0] == exp["recomputations"] and cnt[b, 1] == exp["approx_lookups"]


@pytest.mark.parametrize("k", [3, 10])
def test_c2shape_ground_truth_matches_reference(fx, k):
    from paper_2506_08276_b200.evaluation import ground_truth
    assert ground_truth(fx["E"], fx["Q"], k, "cosine") == fx["meta"][f"ground_truth_{k}"]


def test_c2shape_ground_truth_with_deletes_matches_oracle(fx):
    """Inactive rows are skipped like the reference's active mask (evaluation.py:88-94)."""
    from oracle import numerics
    from paper_2506_08276_b200.evaluation import ground_truth
    E, Q = fx["E"], fx["Q"][:8]
    active = np.ones(E.shape[0], dtype=bool)
    active[np.asarray(fx["meta"]["ground_truth_3"][:8]).ravel()] = False   # delete the top hits
    got = ground_truth(E, Q, 3, "cosine", active=active)
    for q, g in zip(Q, got):
        d = numerics.distance_many(E, q, "cosine").astype(np.float64)
        d = np.where(active, d, np.inf)
        assert g == [int(i) for i in np.lexsort((np.arange(E.shape[0]), d))[:3]]


def test_c2shape_smem_lut_path_bit_exact(fx):
    """LV_SMEM_LUT (each query's table staged in shared memory by one bulk copy)
    returns the same bits as the default per-lookup path and the reference."""
    import torch
    lv = fx["lv"]
    model, codes = fx["pq"]
    dev = lv.search.device_index_for(fx["g"], model, codes)
    case = fx["meta"]["cases"][0]
    out = dev.search_device(torch.from_numpy(fx["Q"]).cuda(), lv.SearchParams(**case["params"]),
                            lv.MatrixSource(torch.from_numpy(fx["E"]).cuda()), smem_lut=True)
    ids = out["ids"].cpu().numpy()
    dist = out["dist"].cpu().numpy().view(np.uint32)
    for b, exp in enumerate(case["reports"]):
        assert list(ids[b]) == exp["ids"] and list(dist[b]) == exp["dist"]


def test_c2shape_hash_visited_sets_bit_exact(fx):
    """LV_HASH_VISITED (bounded per-query hash sets instead of n-bit bitmaps —
    the automatic choice at 10M nodes x 16k queries) returns the reference's
    bits, in matrix mode and across repeated calls (tables reset per query)."""
    import torch
    lv = fx["lv"]
    model, codes = fx["pq"]
    dev = lv.search.device_index_for(fx["g"], model, codes)
    for _ in range(2):
        for case in fx["meta"]["cases"]:
            out = dev.search_device(torch.from_numpy(fx["Q"]).cuda(),
                                    lv.SearchParams(**case["params"]),
                                    lv.MatrixSource(torch.from_numpy(fx["E"]).cuda()),
                                    hash_visited=True, max_inflight=64)
            ids = out["ids"].cpu().numpy()
            dist = out["dist"].cpu().numpy().view(np.uint32)
            cnt = out["counters"].cpu().numpy()
            for b, exp in enumerate(case["reports"]):
                assert list(ids[b]) == exp["ids"] and list(dist[b]) == exp["dist"]
                assert cnt[b, 0] == exp["recomputations"]
