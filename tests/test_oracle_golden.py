"""Pin the CPU oracle (oracle/) against golden vectors from the unmodified reference.

Golden files were produced by tests/golden/make_golden.py, which imports the
reference (slimvec) and runs its own search / ADC / distance code. Bit-exact
comparison: ids, float32 distance bits, counters, batch logs, visit order.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, f32_from_hex, load_fixture_dir
from oracle import numerics
from oracle import search_port as sp


def _check_case(fx, params, reports, cached=None, deleted=None):
    g = fx["graph"]
    if deleted is not None:
        g.deleted = deleted
    else:
        g.deleted = np.zeros(g.n, dtype=bool)
    src = sp.MatrixRows(fx["matrix"])
    p = dict(params)
    p.pop("cache_percent", None)
    prm = sp.SearchParams(**p)
    for qi, (q, exp) in enumerate(zip(fx["queries"], reports)):
        rep = sp.run_search(g, q, prm, src, fx["pq"]["metric"], fx["pq"]["codebooks"],
                            fx["pq"]["codes"], qn=fx["qn"][qi], cached=cached)
        assert [i for i, _ in rep.results] == exp["ids"], (params, qi)
        assert [np.float32(d).view(np.uint32) for _, d in rep.results] == \
            [np.float32(f32_from_hex(h)).view(np.uint32) for h in exp["dist_hex"]]
        assert rep.recomputations == exp["recomputations"]
        assert rep.approx_lookups == exp["approx_lookups"]
        assert rep.batches == exp["batches"]
        assert rep.cache_hits == exp["cache_hits"]
        if "visits" in exp:
            assert rep.visits == exp["visits"]


@pytest.mark.parametrize("case", ["small_cos", "small_l2", "small_ip"])
def test_oracle_matches_reference_search(search_cases, case):
    fx = load_fixture_dir(case)
    for entry in search_cases[case]:
        _check_case(fx, entry["params"], entry["reports"])


def test_oracle_matches_reference_with_deletes(search_cases):
    fx = load_fixture_dir("small_cos")
    for entry in search_cases["small_cos_deleted"]:
        _check_case(fx, entry["params"], entry["reports"], deleted=fx["deleted"])


def test_oracle_matches_reference_with_cache(search_cases):
    fx = load_fixture_dir("small_cos")
    g = fx["graph"]
    # build_embedding_cache (search.py:130-142): top ceil(f*n/100) by (degree desc, id asc)
    count = int(np.ceil(10.0 / 100.0 * g.n))
    order = np.lexsort((np.arange(g.n), -g.out_degrees(0)))
    cached = set(int(i) for i in order[:count])
    for entry in search_cases["small_cos_cache10"]:
        _check_case(fx, entry["params"], entry["reports"], cached=cached)


def test_oracle_reproduces_published_standard_fixture(standard_cases):
    """test_output.txt:216,219 — recall 0.900 @ ef=120 with 322.4 recomputes/query."""
    fx = load_fixture_dir("standard")
    for entry in standard_cases:
        _check_case(fx, entry["params"], entry["reports"])
    rec = np.mean([r["recomputations"] for r in standard_cases[0]["reports"]])
    assert abs(rec - 322.39) < 1e-6


def test_path_graph_hand_trace():
    """test_search.py:103-114: visits [2,3,4,1,0], batches [1,2,1,1], result (4, 0.04)."""
    g = sp.read_lgr1(GOLDEN / "path" / "graph.bin")
    matrix = np.arange(5, dtype=np.float32).reshape(5, 1)
    rep = sp.best_first(g, np.array([4.2], np.float32), sp.SearchParams(k=1, ef=5,
                        mode="exact_bestfirst"), sp.MatrixRows(matrix), "l2")
    assert rep.visits == [2, 3, 4, 1, 0]
    assert rep.batches == [1, 2, 1, 1]
    assert rep.recomputations == 5
    assert rep.results[0][0] == 4 and abs(rep.results[0][1] - 0.04) < 1e-5


@pytest.mark.parametrize("dim", [1, 3, 8, 12, 17, 32, 100, 256, 768, 1024])
@pytest.mark.parametrize("metric", ["l2", "ip", "cosine"])
def test_distance_many_bit_exact(dim, metric):
    rows = np.load(GOLDEN / f"num_rows_{dim}.npy")
    q = np.load(GOLDEN / f"num_q_{dim}.npy")
    exp = np.load(GOLDEN / f"num_dist_{metric}_{dim}.npy")
    got = numerics.distance_many(rows, q, metric)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("tag", ["32_8_cosine", "256_32_cosine", "768_64_cosine",
                                 "40_5_l2", "24_6_ip", "30_4_cosine"])
def test_adc_bit_exact(tag):
    cb = np.load(GOLDEN / f"adc_cb_{tag}.npy")
    q = np.load(GOLDEN / f"adc_q_{tag}.npy")
    codes = np.load(GOLDEN / f"adc_codes_{tag}.npy")
    metric = tag.split("_")[2]
    table = numerics.adc_build(cb, q.shape[0], metric, q)
    assert np.array_equal(table.view(np.uint32), np.load(GOLDEN / f"adc_table_{tag}.npy").view(np.uint32))
    approx = numerics.approx_distance_many(table, codes)
    assert np.array_equal(approx.view(np.uint32), np.load(GOLDEN / f"adc_approx_{tag}.npy").view(np.uint32))


def test_einsum_order_matches_this_hosts_numpy():
    """Re-pin App. A on whatever host runs the tests (catches a numpy/SIMD change)."""
    rng = np.random.default_rng(5)
    for d in (2, 5, 8, 16, 17, 33, 64, 100, 768, 1024):
        a = rng.normal(size=(500, d)).astype(np.float32)
        b = rng.normal(size=d).astype(np.float32)
        assert np.array_equal(np.einsum("ij,j->i", a, b).view(np.uint32),
                              numerics.einsum_dot(a, b).view(np.uint32))
        c = rng.normal(size=(500, d)).astype(np.float32)
        assert np.array_equal(np.einsum("ij,ij->i", a, c).view(np.uint32),
                              numerics.einsum_dot(a, c).view(np.uint32))


def test_cutoff_rank_uses_float_product():
    """0.07*100 = 7.000000000000001 -> ceil gives 8, not 7."""
    assert sp.cutoff_rank(7.0, 100) == 8
    assert sp.cutoff_rank(30.0, 10) == 3
    assert sp.cutoff_rank(100.0, 1) == 1
    assert sp.cutoff_rank(0.5, 1) == 1


def test_oracle_matches_reference_on_encoder_fixture():
    """The oracle port reproduces the reference's run_search on the fp32-encoder
    fixture (tests/golden/make_encoder_golden.py)."""
    import json
    from oracle import search_port as sp
    d = GOLDEN / "enc_fp32"
    meta = json.loads((d / "reference_results.json").read_text())
    g = sp.read_lgr1(d / "graph.bin")
    pq = sp.read_lpq1(d / "pq.bin")
    E = np.load(d / "embeddings_ref.npy")
    Q = np.load(d / "queries_ref.npy")
    for case in meta["cases"]:
        p = sp.SearchParams(**case["params"])
        for q, exp in list(zip(Q, case["reports"]))[:40]:
            rep = sp.two_level(g, q, p, pq["codebooks"], pq["codes"], sp.MatrixRows(E), "cosine")
            assert [i for i, _ in rep.results] == exp["ids"]
            assert [float(x) for _, x in rep.results] == exp["dist"]
            assert rep.recomputations == exp["recomputations"]


@pytest.mark.parametrize("n", [32, 64, 96, 128, 256, 768, 1024])
def test_sdot_order(n):
    """np.dot of float32 vectors (OpenBLAS SkylakeX sdot) == the restated order
    that lv_query_norms / lv_merge_pending run on the device."""
    rng = np.random.default_rng(n)
    for _ in range(60):
        x = rng.standard_normal(n).astype(np.float32)
        y = rng.standard_normal(n).astype(np.float32)
        assert numerics.sdot_openblas(x, y).view(np.uint32) == np.dot(x, y).view(np.uint32)
        assert numerics.sdot_openblas(x, x).view(np.uint32) == np.dot(x, x).view(np.uint32)


def _engine_fixture():
    import json
    d = GOLDEN / "engine_pending"
    g = sp.read_lgr1(d / "graph.bin")
    g.deleted = sp.read_ldl1(d / "deleted.bin", g.n)
    return dict(d=d, g=g, pq=sp.read_lpq1(d / "pq.bin"), matrix=np.load(d / "matrix.npy"),
                pids=np.load(d / "pending_ids.npy"), pvec=np.load(d / "pending_vecs.npy"),
                Q=np.load(d / "queries.npy"), meta=json.loads((d / "cases.json").read_text()))


def test_oracle_engine_pending_merge():
    """Engine.search with a pending buffer (index.py:305-328): oracle search +
    oracle buffer_scan merge == the reference Engine's reports, bit for bit."""
    fx = _engine_fixture()
    src = sp.MatrixRows(fx["matrix"])
    for case in fx["meta"]["cases"]:
        prm = sp.SearchParams(**case["params"])
        for q, exp in zip(fx["Q"], case["reports"]):
            rep = sp.run_search(fx["g"], q, prm, src, fx["pq"]["metric"], fx["pq"]["codebooks"],
                                fx["pq"]["codes"], qn=numerics.query_norm(q))
            res = sp.merge_pending(rep.results, q, fx["pids"], fx["pvec"], "cosine", prm.k)
            assert [i for i, _ in res] == exp["ids"]
            assert [int(np.float32(d).view(np.uint32)) for _, d in res] == exp["dist"]
            assert rep.recomputations == exp["recomputations"]


def test_oracle_matches_reference_at_config1():
    """Config-1 at full size (10k x 256-d, M=32, PQ m=32; make_c1_golden.py):
    the oracle port reproduces the reference's ids, distance bits and
    counters (first 40 queries of each case — CPU time)."""
    import json
    d = GOLDEN / "c1"
    meta = json.loads((d / "reference_results.json").read_text())
    g = sp.read_lgr1(d / "graph.bin")
    pq = sp.read_lpq1(d / "pq.bin")
    E, Q = np.load(d / "embeddings_ref.npy"), np.load(d / "queries_ref.npy")
    src = sp.MatrixRows(E)
    for case in meta["cases"]:
        prm = sp.SearchParams(**case["params"])
        for q, exp in list(zip(Q, case["reports"]))[:40]:
            rep = sp.run_search(g, q, prm, src, "cosine", pq["codebooks"], pq["codes"],
                                qn=numerics.query_norm(q))
            assert [i for i, _ in rep.results] == exp["ids"]
            assert [np.float32(x).view(np.uint32) for _, x in rep.results] == \
                [np.float32(x).view(np.uint32) for x in exp["dist"]]
            assert rep.recomputations == exp["recomputations"]
            assert rep.approx_lookups == exp["approx_lookups"]


def test_oracle_matches_reference_at_config2_shape():
    """Config-2 shape (100k x 768, GPU-built M=32 graph, PQ m=64;
    make_c2shape_golden.py): the oracle port reproduces the reference's ids,
    distance bits and counters (first 12 queries per case — CPU time)."""
    import json
    import sys
    sys.path.insert(0, str(GOLDEN))
    import c2shape
    d = GOLDEN / "c2shape"
    meta = json.loads((d / "reference_results.json").read_text())
    g = sp.read_lgr1(d / "graph.bin")
    pq = sp.read_lpq1(d / "pq.bin")
    E, Q = c2shape.make()
    src = sp.MatrixRows(E)
    for case in meta["cases"]:
        prm = sp.SearchParams(**case["params"])
        for q, exp in list(zip(Q, case["reports"]))[:12]:
            rep = sp.run_search(g, q, prm, src, "cosine", pq["codebooks"], pq["codes"],
                                qn=numerics.query_norm(q))
            assert [i for i, _ in rep.results] == exp["ids"]
            assert [int(np.float32(x).view(np.uint32)) for _, x in rep.results] == exp["dist"]
            assert rep.recomputations == exp["recomputations"]
