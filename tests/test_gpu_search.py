"""GPU parity: the sm_100a search path against golden vectors from the unmodified
reference (tests/golden/make_golden.py) — ids, float32 distance bits, counters,
batch logs and the base-layer expansion order, bit-exact."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, f32_from_hex, load_fixture_dir

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lv():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as mod
    return mod


def _load(lv, name):
    d = GOLDEN / name
    g = lv.load_graph(d / "graph.bin")
    m, c = lv.load_pq(d / "pq.bin")
    return g, m, c, np.load(d / "matrix.npy"), np.load(d / "queries.npy"), np.load(d / "qn.npy")


def _compare(reps, expected, check_visits=True):
    for qi, (rep, exp) in enumerate(zip(reps, expected)):
        assert [i for i, _ in rep.results] == exp["ids"], qi
        got_bits = [np.float32(d).view(np.uint32) for _, d in rep.results]
        exp_bits = [np.float32(f32_from_hex(h)).view(np.uint32) for h in exp["dist_hex"]]
        assert got_bits == exp_bits, qi
        assert rep.recomputations == exp["recomputations"], qi
        assert rep.approx_lookups == exp["approx_lookups"], qi
        assert rep.batches == exp["batches"], qi
        assert rep.cache_hits == exp["cache_hits"], qi
        if check_visits and "visits" in exp:
            assert rep.visits == exp["visits"], qi


def _params(lv, p):
    p = dict(p)
    p.pop("cache_percent", None)
    return lv.SearchParams(**p)


@pytest.mark.parametrize("case", ["small_cos", "small_l2", "small_ip"])
def test_device_search_matches_reference(lv, search_cases, case):
    g, m, c, matrix, queries, qn = _load(lv, case)
    for entry in search_cases[case]:
        reps = lv.search_batch(g, queries, _params(lv, entry["params"]), lv.MatrixSource(matrix),
                               m.metric, m, c, qn=qn, trace=True)
        _compare(reps, entry["reports"])


def test_device_search_with_deletes(lv, search_cases):
    g, m, c, matrix, queries, qn = _load(lv, "small_cos")
    g.deleted = lv.load_deleted(GOLDEN / "small_cos" / "deleted.bin", g.n)
    for entry in search_cases["small_cos_deleted"]:
        reps = lv.search_batch(g, queries, _params(lv, entry["params"]), lv.MatrixSource(matrix),
                               "cosine", m, c, qn=qn, trace=True)
        _compare(reps, entry["reports"])


def test_device_search_with_cache(lv, search_cases):
    g, m, c, matrix, queries, qn = _load(lv, "small_cos")
    cache = lv.build_embedding_cache(g, 10.0)
    for entry in search_cases["small_cos_cache10"]:
        reps = lv.search_batch(g, queries, _params(lv, entry["params"]), lv.MatrixSource(matrix),
                               "cosine", m, c, cache=cache, qn=qn, trace=True)
        _compare(reps, entry["reports"])


def test_device_standard_fixture_published_numbers(lv, standard_cases):
    """test_output.txt:216,219: recall 0.900 @ ef=120, 322.39 recomputes/query."""
    g, m, c, matrix, queries, qn = _load(lv, "standard")
    for entry in standard_cases:
        reps = lv.search_batch(g, queries, _params(lv, entry["params"]), lv.MatrixSource(matrix),
                               "cosine", m, c, qn=qn)
        _compare(reps, entry["reports"], check_visits=False)
    reps = lv.search_batch(g, queries, lv.SearchParams(k=3, ef=120), lv.MatrixSource(matrix),
                           "cosine", m, c, qn=qn)
    assert abs(np.mean([r.recomputations for r in reps]) - 322.39) < 1e-9


def test_batch_composition_and_inflight_slots_do_not_change_results(lv):
    g, m, c, matrix, queries, qn = _load(lv, "small_cos")
    dev = lv.search.device_index_for(g, m, c)
    p = lv.SearchParams(k=3, ef=48)
    base = dev.search(queries, p, lv.MatrixSource(matrix), qn=qn, max_inflight=1)
    for slots in (2, 7, 30):
        reps = dev.search(queries, p, lv.MatrixSource(matrix), qn=qn, max_inflight=slots)
        assert [r.results for r in reps] == [r.results for r in base]
        assert [r.recomputations for r in reps] == [r.recomputations for r in base]
    single = [dev.search(q[None], p, lv.MatrixSource(matrix), qn=qn[i:i + 1])[0]
              for i, q in enumerate(queries[:5])]
    assert [r.results for r in single] == [r.results for r in base[:5]]


def test_path_graph_hand_trace(lv):
    """test_search.py:103-114 on the device."""
    g = lv.load_graph(GOLDEN / "path" / "graph.bin")
    matrix = np.arange(5, dtype=np.float32).reshape(5, 1)
    q = np.array([[4.2]], np.float32)
    rep = lv.search_batch(g, q, lv.SearchParams(k=1, ef=5, mode="exact_bestfirst"),
                          lv.MatrixSource(matrix), "l2", trace=True)[0]
    assert rep.visits == [2, 3, 4, 1, 0]
    assert rep.batches == [1, 2, 1, 1]
    assert rep.recomputations == 5
    assert rep.results[0][0] == 4 and rep.results[0][1] == pytest.approx(0.04, abs=1e-5)


def test_single_node_graph(lv):
    g = lv.PrunedGraph(n=1, max_degree=2, entry_point=0, levels=np.zeros(1, np.uint16),
                       level_offsets=[np.array([0, 0], np.uint64)],
                       level_neighbors=[np.empty(0, np.uint32)])
    rep = lv.search_batch(g, np.array([[1.0]], np.float32),
                          lv.SearchParams(k=1, ef=1, mode="exact_bestfirst"),
                          lv.MatrixSource(np.array([[3.0]], np.float32)), "l2")[0]
    assert rep.results == [(0, 4.0)]
    assert rep.recomputations == 1


def test_aq_overflow_is_retried_transparently(lv, search_cases):
    """ef=n drives the approximate queue past its default capacity (exactness ceiling)."""
    g, m, c, matrix, queries, qn = _load(lv, "small_cos")
    entry = [e for e in search_cases["small_cos"] if e["params"].get("ef") == 600][0]
    reps = lv.search_batch(g, queries, _params(lv, entry["params"]), lv.MatrixSource(matrix),
                           "cosine", m, c, qn=qn)
    _compare(reps, entry["reports"], check_visits=False)


@pytest.mark.parametrize("dim", [1, 3, 8, 12, 17, 32, 100, 256, 768, 1024])
@pytest.mark.parametrize("metric", ["l2", "ip", "cosine"])
def test_distance_kernel_bit_exact(lv, dim, metric):
    from paper_2506_08276_b200 import _lib
    rows = np.load(GOLDEN / f"num_rows_{dim}.npy")
    q = np.load(GOLDEN / f"num_q_{dim}.npy")
    exp = np.load(GOLDEN / f"num_dist_{metric}_{dim}.npy")
    qn = lv.query_norm(q)
    out = np.empty(rows.shape[0], np.float32)
    _lib.check(_lib.lib().lv_distance_many(_lib.LV_METRIC[metric], rows.ctypes.data, rows.shape[0],
                                           dim, q.ctypes.data, float(qn), out.ctypes.data, 0, None))
    assert np.array_equal(out.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("tag", ["32_8_cosine", "256_32_cosine", "768_64_cosine", "40_5_l2",
                                 "24_6_ip", "30_4_cosine"])
def test_adc_kernels_bit_exact(lv, tag):
    cb = np.load(GOLDEN / f"adc_cb_{tag}.npy")
    q = np.load(GOLDEN / f"adc_q_{tag}.npy")
    codes = np.load(GOLDEN / f"adc_codes_{tag}.npy")
    dim, m, metric = int(tag.split("_")[0]), int(tag.split("_")[1]), tag.split("_")[2]
    padded = cb.shape[1 - 1 + 1 - 1 + 2] * m if False else cb.shape[2] * m
    model = lv.PQModel(dim=dim, padded_dim=padded, m_pq=m, metric=metric, codebooks=cb)
    n = codes.shape[0]
    g = lv.PrunedGraph(n=n, max_degree=1, entry_point=0, levels=np.zeros(n, np.uint16),
                       level_offsets=[np.zeros(n + 1, np.uint64)],
                       level_neighbors=[np.zeros(0, np.uint32)])
    dev = lv.DeviceIndex(g, model, lv.PQCodes(codes))
    table = dev.adc_tables(q[None], np.array([lv.query_norm(q)], np.float32))[0]
    assert np.array_equal(table.view(np.uint32), np.load(GOLDEN / f"adc_table_{tag}.npy").view(np.uint32))
    approx = dev.adc_score(table, np.arange(n))
    assert np.array_equal(approx.view(np.uint32), np.load(GOLDEN / f"adc_approx_{tag}.npy").view(np.uint32))


@pytest.mark.parametrize("m", [32, 64, 96])
def test_streaming_adc_bit_exact_vs_oracle(lv, m):
    """lv_adc_score's streaming kernel (LUT in shared memory, 16-byte code
    loads; m = 32/64/96) keeps numpy's fp64 pairwise order (pq.py:186-189)."""
    from oracle.numerics import approx_distance_many
    rng = np.random.default_rng(m)
    n, dim = 5000, 768
    cb = rng.standard_normal((m, 256, -(-dim // m)), dtype=np.float32)
    model = lv.PQModel(dim=dim, padded_dim=cb.shape[2] * m, m_pq=m, metric="cosine", codebooks=cb)
    codes = rng.integers(0, 256, (n, m), dtype=np.uint8)
    g = lv.PrunedGraph(n=n, max_degree=1, entry_point=0, levels=np.zeros(n, np.uint16),
                       level_offsets=[np.zeros(n + 1, np.uint64)],
                       level_neighbors=[np.zeros(0, np.uint32)])
    dev = lv.DeviceIndex(g, model, lv.PQCodes(codes))
    table = (rng.standard_normal((m, 256)) * 0.1).astype(np.float32)
    ids = rng.permutation(n)
    got = dev.adc_score(table, ids)
    ref = approx_distance_many(table, codes[ids])
    assert np.array_equal(got.view(np.uint32), np.asarray(ref, dtype=np.float32).view(np.uint32))


def test_empty_batch_returns_nothing(lv):
    d = GOLDEN / "small_cos"
    g = lv.load_graph(d / "graph.bin")
    model, codes = lv.load_pq(d / "pq.bin")
    E = np.load(d / "matrix.npy")
    reps = lv.search_batch(g, np.zeros((0, E.shape[1]), np.float32), lv.SearchParams(k=3, ef=8),
                           lv.MatrixSource(E), "cosine", model, codes)
    assert reps == []


def test_ef_n_full_rerank_equals_brute_force(lv):
    """ef = n, rerank 100% reduces to exhaustive search (reference
    test_search.py:196-205): the results are the reference-order brute force."""
    from paper_2506_08276_b200.evaluation import ground_truth
    d = GOLDEN / "small_cos"
    g = lv.load_graph(d / "graph.bin")
    model, codes = lv.load_pq(d / "pq.bin")
    E, Q = np.load(d / "matrix.npy"), np.load(d / "queries.npy")
    reps = lv.search_batch(g, Q, lv.SearchParams(k=5, ef=g.n, rerank_percent=100.0),
                           lv.MatrixSource(E), "cosine", model, codes)
    gt = ground_truth(E, Q, 5, "cosine")
    assert [[i for i, _ in r.results] for r in reps] == gt


def test_all_deleted_returns_no_results_but_traverses(lv):
    """Deleted nodes stay traversable and are filtered only at k_best
    (search.py:324,426): with every node deleted the result list is empty."""
    d = GOLDEN / "small_cos"
    g = lv.load_graph(d / "graph.bin")
    model, codes = lv.load_pq(d / "pq.bin")
    E, Q = np.load(d / "matrix.npy"), np.load(d / "queries.npy")
    g.deleted = np.ones(g.n, dtype=bool)
    reps = lv.search_batch(g, Q[:8], lv.SearchParams(k=3, ef=16), lv.MatrixSource(E), "cosine",
                           model, codes)
    assert all(r.results == [] and r.recomputations > 0 for r in reps)
    g.deleted = np.zeros(g.n, dtype=bool)
