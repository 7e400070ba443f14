"""The reference's own objects through the device path:
a HOST provider behind a ProviderSource (the reference's Synthetic/External
providers: lv_index_set_fetch callback), a reference-shaped EmbeddingCache
({id: vector}), an OverlayGraph-shaped graph (base + overrides), and a
provider failure surfacing as SearchError with the partial report
(search.py:169-172). Results must equal the matrix-source run bit for bit."""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    d = GOLDEN / "small_cos"
    g = lv.load_graph(d / "graph.bin")
    model, codes = lv.load_pq(d / "pq.bin")
    return dict(lv=lv, g=g, model=model, codes=codes, E=np.load(d / "matrix.npy"),
                Q=np.load(d / "queries.npy"), qn=np.load(d / "qn.npy"))


class HostProvider:
    """vectors.py:201-211 duck type: embed_batch(requests) -> f32[n, dim]."""

    def __init__(self, E, fail_after=None):
        self.E = E
        self.config = SimpleNamespace(dim=E.shape[1], max_batch=64, kind="synthetic")
        self.calls = 0
        self.fail_after = fail_after

    def embed_batch(self, requests):
        from paper_2506_08276_b200.errors import ProviderError
        self.calls += 1
        if self.fail_after is not None and self.calls > self.fail_after:
            raise ProviderError("provider down", retries=2)
        return self.E[[int(r.content.decode()) for r in requests]]


def _same(a, b):
    for x, y in zip(a, b):
        assert x.results == y.results
        assert x.recomputations == y.recomputations
        assert x.approx_lookups == y.approx_lookups


@pytest.mark.parametrize("mode", ["two_level", "exact_bestfirst"])
def test_host_provider_callback_equals_matrix(fx, mode):
    lv = fx["lv"]
    p = lv.SearchParams(k=3, ef=32, rerank_percent=30.0, mode=mode)
    pq = (fx["model"], fx["codes"]) if mode == "two_level" else (None, None)
    ref = lv.search_batch(fx["g"], fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", *pq,
                          qn=fx["qn"])
    prov = HostProvider(fx["E"])
    src = lv.ProviderSource(prov, lambda i: str(i).encode())
    got = lv.search_batch(fx["g"], fx["Q"], p, src, "cosine", *pq, qn=fx["qn"])
    _same(ref, got)
    assert prov.calls > 0


def test_reference_shaped_cache_is_transparent(fx):
    lv = fx["lv"]
    p = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    src = lv.ProviderSource(HostProvider(fx["E"]), lambda i: str(i).encode())
    plain = lv.search_batch(fx["g"], fx["Q"], p, src, "cosine", fx["model"], fx["codes"],
                            qn=fx["qn"])
    ids = lv.build_embedding_cache(fx["g"], 10.0).ids
    cache = SimpleNamespace(vectors={int(i): fx["E"][i] for i in ids})   # reference layout
    cached = lv.search_batch(fx["g"], fx["Q"], p, src, "cosine", fx["model"], fx["codes"],
                             qn=fx["qn"], cache=cache)
    hits = 0
    for a, b in zip(plain, cached):
        assert a.results == b.results
        assert a.recomputations == b.recomputations + b.cache_hits
        hits += b.cache_hits
    assert hits > 0


def test_provider_error_becomes_search_error(fx):
    lv = fx["lv"]
    from paper_2506_08276_b200.errors import SearchError
    src = lv.ProviderSource(HostProvider(fx["E"], fail_after=1), lambda i: str(i).encode())
    with pytest.raises(SearchError) as err:
        lv.search_batch(fx["g"], fx["Q"], lv.SearchParams(k=3, ef=32), src, "cosine",
                        fx["model"], fx["codes"], qn=fx["qn"])
    assert "provider down" in str(err.value)
    assert err.value.partial_report is not None


class Overlay:
    """OverlayGraph's observable surface (update.py:93-191): base CSR, per-level
    override rows, the delete list and freeze(max_degree)."""

    def __init__(self, base):
        self.base = base
        self.n, self.max_degree, self.entry_point = base.n, base.max_degree, base.entry_point
        self._deleted = list(base.deleted.tolist())
        self.overrides = [{} for _ in range(base.level_count)]

    def neighbor_list(self, v, level):
        row = self.overrides[level].get(v)
        return list(row) if row is not None else base_row(self.base, v, level)

    def freeze(self, max_degree):
        from paper_2506_08276_b200.graph import PrunedGraph
        offs, nbrs = [], []
        for lvl in range(len(self.overrides)):
            rows = [self.neighbor_list(v, lvl) for v in range(self.n)]
            offs.append(np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.uint64))
            nbrs.append(np.asarray([w for r in rows for w in r], dtype=np.uint32))
        return PrunedGraph(self.n, max_degree, self.entry_point, self.base.levels.copy(), offs,
                           nbrs, np.asarray(self._deleted, dtype=bool))


def base_row(g, v, level):
    return g.neighbors(v, level).tolist()


def test_overlay_graph_equals_its_frozen_csr(fx):
    lv = fx["lv"]
    p = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    ov = Overlay(fx["g"])
    plain = lv.search_batch(ov, fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", fx["model"],
                            fx["codes"], qn=fx["qn"])
    _same(lv.search_batch(fx["g"], fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", fx["model"],
                          fx["codes"], qn=fx["qn"]), plain)
    # override a few level-0 rows (an add's rewiring) and delete a node
    rng = np.random.default_rng(0)
    for v in rng.choice(fx["g"].n, 20, replace=False):
        ov.overrides[0][int(v)] = [int(w) for w in rng.choice(fx["g"].n, 8, replace=False)
                                   if w != v]
    ov._deleted[int(plain[0].results[0][0])] = True
    frozen = ov.freeze(ov.max_degree)
    a = lv.search_batch(ov, fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", fx["model"],
                        fx["codes"], qn=fx["qn"])
    b = lv.search_batch(frozen, fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", fx["model"],
                        fx["codes"], qn=fx["qn"])
    _same(a, b)
    assert a[0].results[0][0] != plain[0].results[0][0]


def test_failed_search_leaves_no_stale_visited_bits(fx):
    """A provider failure aborts lv_search_batch mid-traversal with queries in
    flight; the next search on the same handle must clear their visited sets
    (workspace dirty flag) and return the reference results."""
    lv = fx["lv"]
    from paper_2506_08276_b200.errors import SearchError
    p = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    ref = lv.search_batch(fx["g"], fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", fx["model"],
                          fx["codes"], qn=fx["qn"])
    bad = lv.ProviderSource(HostProvider(fx["E"], fail_after=2), lambda i: str(i).encode())
    with pytest.raises(SearchError):
        lv.search_batch(fx["g"], fx["Q"], p, bad, "cosine", fx["model"], fx["codes"], qn=fx["qn"])
    good = lv.ProviderSource(HostProvider(fx["E"]), lambda i: str(i).encode())
    _same(ref, lv.search_batch(fx["g"], fx["Q"], p, good, "cosine", fx["model"], fx["codes"],
                               qn=fx["qn"]))


def test_zero_query_rejected_for_cosine_two_level(fx):
    """adc_build raises for a zero query under cosine (pq.py:163-166)."""
    lv = fx["lv"]
    from paper_2506_08276_b200.errors import InvalidArgumentError
    Q = fx["Q"][:4].copy()
    Q[2] = 0.0
    with pytest.raises(InvalidArgumentError):
        lv.search_batch(fx["g"], Q, lv.SearchParams(k=3, ef=32), lv.MatrixSource(fx["E"]),
                        "cosine", fx["model"], fx["codes"])
