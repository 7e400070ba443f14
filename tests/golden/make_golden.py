"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

Usage: python tests/golden/make_golden.py [--standard]

Imports slimvec from /root/reference/pkg/src (read-only; no bytecode written),
builds small indexes with the reference builder, runs the reference's own
search / ADC / distance functions and writes their outputs under
tests/golden/. These files pin both the CPU oracle (oracle/) and the CUDA path.
Nothing here runs on the GPU box.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from slimvec.builder import BuildParams, build_index, embed_items  # noqa: E402
from slimvec.evaluation import STANDARD_FIXTURE, fixture_items, fixture_queries  # noqa: E402
from slimvec.graph import PrunedGraph, save_graph, save_deleted  # noqa: E402
from slimvec.pq import save_pq, adc_build, approx_distance_many, pq_train, pq_encode  # noqa: E402
from slimvec.search import (MatrixSource, SearchParams, run_search,  # noqa: E402
                            build_embedding_cache)
from slimvec.vectors import (EmbeddingRequest, ProviderConfig, embed_all,  # noqa: E402
                             make_provider, distance_many)

OUT = Path(__file__).resolve().parent


class _Recorder:
    """Graph proxy recording base-layer expansions (as test_search.py:24-52)."""

    def __init__(self, g):
        self._g = g
        self.visits = []

    def __getattr__(self, name):
        return getattr(self._g, name)

    @property
    def level_count(self):
        return self._g.level_count

    @property
    def entry_point(self):
        return self._g.entry_point

    @property
    def n(self):
        return self._g.n

    def neighbors(self, v, level=0):
        if level == 0:
            self.visits.append(int(v))
        return self._g.neighbors(v, level)

    def is_deleted(self, v):
        return self._g.is_deleted(v)


def _f32hex(x) -> str:
    return np.float32(x).view(np.uint32).item().to_bytes(4, "little").hex()


def _report(rep, visits):
    return {
        "ids": [int(i) for i, _ in rep.results],
        "dist_hex": [_f32hex(d) for _, d in rep.results],
        "recomputations": rep.recomputations,
        "approx_lookups": rep.approx_lookups,
        "batches": list(rep.batches),
        "cache_hits": rep.cache_hits,
        "visits": visits,
    }


def build_fixture(name, n, n_queries, dim, metric, m_pq, seed=42, max_degree=16,
                  low_degree=5, hub=8.0, efc=64):
    config = ProviderConfig(kind="synthetic", dim=dim, seed=seed, max_batch=64)
    provider = make_provider(config)
    items = fixture_items(n)
    matrix = embed_items(items, provider)
    params = BuildParams(ef_construction=efc, max_degree=max_degree, low_degree=low_degree,
                         hub_percent=hub, metric=metric, seed=seed, pq_subspaces=m_pq)
    res = build_index(items, params, provider)
    queries = embed_all([EmbeddingRequest(-1, q) for q in fixture_queries(n_queries)], provider)
    d = OUT / name
    d.mkdir(exist_ok=True)
    save_graph(res.graph, d / "graph.bin")
    save_pq(res.pq_model, res.pq_codes, d / "pq.bin")
    np.save(d / "matrix.npy", matrix)
    np.save(d / "queries.npy", queries)
    qn = np.array([np.float32(np.sqrt(np.dot(q, q))) for q in queries], dtype=np.float32)
    np.save(d / "qn.npy", qn)
    return res, matrix, queries, d


def run_grid(name, res, matrix, queries, metric, grid, d, deleted=None, cache_pct=None):
    src = MatrixSource(matrix)
    g = res.graph
    cache = build_embedding_cache(g, cache_pct, src) if cache_pct else None
    out = []
    for p in grid:
        params = SearchParams(**p)
        reps = []
        for q in queries:
            rec = _Recorder(g)
            rep = run_search(rec, q, params, src, metric, res.pq_model, res.pq_codes, cache)
            reps.append(_report(rep, rec.visits))
        out.append({"params": p, "reports": reps})
    return out


def small_fixtures():
    cases = {}
    grid = [
        dict(k=3, ef=16, rerank_percent=30.0),
        dict(k=3, ef=32, rerank_percent=30.0),
        dict(k=3, ef=48, rerank_percent=30.0, batch_size=16),
        dict(k=3, ef=64, rerank_percent=30.0, batch_size=8),
        dict(k=3, ef=48, rerank_percent=7.0),
        dict(k=3, ef=48, rerank_percent=14.0),
        dict(k=10, ef=64, rerank_percent=5.0),
        dict(k=3, ef=32, rerank_percent=100.0, batch_size=1),
        dict(k=10, ef=120, rerank_percent=55.0),
        dict(k=3, ef=600, rerank_percent=100.0),
        dict(k=3, ef=8, mode="exact_bestfirst"),
        dict(k=3, ef=32, mode="exact_bestfirst"),
        dict(k=5, ef=64, mode="exact_bestfirst"),
    ]
    res, matrix, queries, d = build_fixture("small_cos", 600, 30, 32, "cosine", 8)
    cases["small_cos"] = run_grid("small_cos", res, matrix, queries, "cosine", grid, d)
    # deleted: mark every 7th node deleted
    deleted = np.zeros(res.graph.n, dtype=bool)
    deleted[::7] = True
    save_deleted(deleted, d / "deleted.bin")
    res.graph.deleted = deleted
    cases["small_cos_deleted"] = run_grid("small_cos", res, matrix, queries, "cosine",
                                          grid[:4] + grid[10:12], d)
    res.graph.deleted = np.zeros(res.graph.n, dtype=bool)
    cases["small_cos_cache10"] = run_grid("small_cos", res, matrix, queries, "cosine",
                                          [dict(k=3, ef=48, rerank_percent=30.0, batch_size=16,
                                                cache_percent=10.0)], d, cache_pct=10.0)
    small_grid = [dict(k=3, ef=16, rerank_percent=30.0), dict(k=3, ef=40, rerank_percent=27.0),
                  dict(k=5, ef=64, rerank_percent=100.0), dict(k=3, ef=24, mode="exact_bestfirst")]
    res, matrix, queries, d = build_fixture("small_l2", 400, 20, 16, "l2", 4, seed=7)
    cases["small_l2"] = run_grid("small_l2", res, matrix, queries, "l2", small_grid, d)
    res, matrix, queries, d = build_fixture("small_ip", 400, 20, 20, "ip", 3, seed=9)
    cases["small_ip"] = run_grid("small_ip", res, matrix, queries, "ip", small_grid, d)
    (OUT / "search_cases.json").write_text(json.dumps(cases))


def path_graph():
    rows = [[1], [0, 2], [1, 3], [2, 4], [3]]
    offsets = np.zeros(6, dtype=np.uint64)
    flat = []
    for v, row in enumerate(rows):
        flat.extend(row)
        offsets[v + 1] = len(flat)
    g = PrunedGraph(n=5, max_degree=2, entry_point=2, levels=np.zeros(5, dtype=np.uint16),
                    level_offsets=[offsets], level_neighbors=[np.asarray(flat, dtype=np.uint32)])
    d = OUT / "path"
    d.mkdir(exist_ok=True)
    save_graph(g, d / "graph.bin")


def numerics():
    rng = np.random.Generator(np.random.PCG64(1234))
    out = {}
    # distance_many for several dims / metrics (reference vectors.py:120)
    for dim in (1, 3, 8, 12, 17, 32, 100, 256, 768, 1024):
        rows = (rng.normal(size=(257, dim)) * rng.uniform(0.05, 20, size=(257, 1))).astype(np.float32)
        q = rng.normal(size=dim).astype(np.float32)
        np.save(OUT / f"num_rows_{dim}.npy", rows)
        np.save(OUT / f"num_q_{dim}.npy", q)
        for metric in ("l2", "ip", "cosine"):
            np.save(OUT / f"num_dist_{metric}_{dim}.npy", distance_many(rows, q, metric))
    # ADC tables + lookups (pq.py:153-189) on trained models
    for (dim, m, metric) in ((32, 8, "cosine"), (256, 32, "cosine"), (768, 64, "cosine"),
                             (40, 5, "l2"), (24, 6, "ip"), (30, 4, "cosine")):
        sample = rng.normal(size=(600, dim)).astype(np.float32)
        model = pq_train(sample, m, iters=3, seed=1, metric=metric)
        codes = pq_encode(model, sample)
        q = rng.normal(size=dim).astype(np.float32)
        table = adc_build(model, q)
        tag = f"{dim}_{m}_{metric}"
        np.save(OUT / f"adc_cb_{tag}.npy", model.codebooks)
        np.save(OUT / f"adc_q_{tag}.npy", q)
        np.save(OUT / f"adc_codes_{tag}.npy", codes)
        np.save(OUT / f"adc_table_{tag}.npy", table)
        np.save(OUT / f"adc_approx_{tag}.npy", approx_distance_many(table, codes))
    (OUT / "numerics.json").write_text(json.dumps({"ok": True}))


def standard():
    cfg = STANDARD_FIXTURE
    res, matrix, queries, d = build_fixture("standard", cfg["n"], cfg["n_queries"], cfg["dim"],
                                            cfg["metric"], cfg["pq_subspaces"], seed=cfg["seed"],
                                            max_degree=cfg["max_degree"],
                                            low_degree=cfg["low_degree"],
                                            hub=cfg["hub_percent"], efc=cfg["ef_construction"])
    grid = [dict(k=3, ef=120, rerank_percent=30.0), dict(k=3, ef=50, rerank_percent=30.0)]
    cases = run_grid("standard", res, matrix, queries, "cosine", grid, d)
    for c in cases:
        for r in c["reports"]:
            r.pop("visits")
    (OUT / "standard_cases.json").write_text(json.dumps(cases))


if __name__ == "__main__":
    path_graph()
    numerics()
    small_fixtures()
    if "--standard" in sys.argv:
        standard()
