"""TEST INFRASTRUCTURE ONLY. CPU restatement of the reference query engine.

Restates ``/root/reference/pkg/src/slimvec/search.py``:
  * ``SearchParams`` validation          search.py:37-56
  * exact queue (bounded, (d, id) order) search.py:194-251
  * upper-layer greedy descent           search.py:257-285
  * exact best-first (Alg. 1)            search.py:288-328
  * two-level search (Alg. 2)            search.py:331-431
  * recompute funnel / counters / cache  search.py:145-188
  * dispatch                             search.py:434-443
with the float math of ``oracle.numerics`` (pinned einsum / pairwise order).

The implementation is deliberately different from the reference (sorted
member list instead of lazy heaps, one state object) but its observable
behaviour — expansion order, results, counters, batch log — is the
reference's, which ``tests/test_oracle_golden.py`` checks against vectors
produced by the unmodified reference.
"""

from __future__ import annotations

import bisect
import math
from dataclasses import dataclass, field

import numpy as np

from . import numerics

MODES = ("exact_bestfirst", "two_level")


@dataclass
class SearchParams:
    """search.py:37-56."""

    k: int = 3
    ef: int = 50
    rerank_percent: float = 30.0
    batch_size: int = 64
    mode: str = "two_level"
    cache_percent: float | None = None

    def __post_init__(self) -> None:
        if self.k < 1 or self.ef < self.k:
            raise ValueError("need ef >= k >= 1")
        if not 0 < self.rerank_percent <= 100:
            raise ValueError("rerank_percent must be in (0, 100]")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode: {self.mode!r}")


@dataclass
class Report:
    """Observable output of one query (search.py:59-72 plus the visit trace)."""

    results: list = field(default_factory=list)
    recomputations: int = 0
    approx_lookups: int = 0
    batches: list = field(default_factory=list)
    cache_hits: int = 0
    visits: list = field(default_factory=list)   # base-layer expansion order


class MatrixRows:
    """Oracle source: exact vectors are rows of a resident matrix (search.py:78-93)."""

    def __init__(self, matrix: np.ndarray) -> None:
        self.matrix = np.asarray(matrix, dtype=np.float32)

    def fetch(self, ids: list[int]) -> np.ndarray:
        return self.matrix[ids]


class _Funnel:
    """Recompute funnel: cache split + counters (search.py:155-188)."""

    def __init__(self, source, cached: set | None, rep: Report) -> None:
        self.source = source
        self.cached = cached
        self.rep = rep

    def rows(self, ids: list[int]) -> np.ndarray:
        if self.cached:
            misses = [i for i in ids if i not in self.cached]
            self.rep.cache_hits += len(ids) - len(misses)
        else:
            misses = ids
        if misses:
            self.rep.recomputations += len(misses)
            self.rep.batches.append(len(misses))
        # values are identical whether cached or recomputed (same provider)
        return self.source.fetch(ids)


class _BoundedExact:
    """Capacity-ef set ordered by (d, id), with visited marks (search.py:194-251)."""

    def __init__(self, ef: int) -> None:
        self.ef = ef
        self.sorted: list[tuple[float, int]] = []
        self.ids: set[int] = set()
        self.visited: set[int] = set()

    def offer(self, node: int, dist: float) -> None:
        if node in self.ids:
            return
        item = (dist, node)
        if len(self.sorted) >= self.ef:
            if not item < self.sorted[-1]:
                return
            _, gone = self.sorted.pop()
            self.ids.discard(gone)
        bisect.insort(self.sorted, item)
        self.ids.add(node)

    def next_unvisited(self) -> int | None:
        for _, node in self.sorted:
            if node not in self.visited:
                self.visited.add(node)
                return node
        return None

    def best(self, k: int, active) -> list[tuple[int, float]]:
        out = []
        for d, node in self.sorted:
            if active(node):
                out.append((node, d))
                if len(out) == k:
                    break
        return out


def _dists(rows: np.ndarray, q: np.ndarray, metric: str, qn) -> list[float]:
    return numerics.distance_many(rows, q, metric, qn).tolist()


def _descend(graph, q, metric, qn, funnel, exact: dict) -> None:
    """Entry recompute + greedy over fresh neighbours per upper level (search.py:257-285)."""
    cur = int(graph.entry_point)
    cur_d = _dists(funnel.rows([cur]), q, metric, qn)[0]
    exact[cur] = cur_d
    for level in range(graph.level_count - 1, 0, -1):
        while True:
            cand = [int(w) for w in graph.neighbors(cur, level) if int(w) not in exact]
            if not cand:
                break
            best = (cur_d, cur)
            for w, dw in zip(cand, _dists(funnel.rows(cand), q, metric, qn)):
                exact[w] = dw
                best = min(best, (dw, w))
            if best == (cur_d, cur):
                break
            cur_d, cur = best


def best_first(graph, q, params: SearchParams, source, metric: str,
               qn=None, cached: set | None = None) -> Report:
    """Alg. 1: every fresh neighbour is recomputed on sight (search.py:288-328)."""
    rep = Report()
    funnel = _Funnel(source, cached, rep)
    exact: dict[int, float] = {}
    _descend(graph, q, metric, qn, funnel, exact)
    eq = _BoundedExact(params.ef)
    for node, d in exact.items():
        eq.offer(node, d)
    while (u := eq.next_unvisited()) is not None:
        rep.visits.append(u)
        fresh = [int(w) for w in graph.neighbors(u, 0) if int(w) not in exact]
        if not fresh:
            continue
        for w in fresh:
            exact[w] = math.inf
        for w, dw in zip(fresh, _dists(funnel.rows(fresh), q, metric, qn)):
            exact[w] = dw
            eq.offer(w, dw)
    rep.results = eq.best(params.k, lambda i: not graph.is_deleted(i))
    return rep


def cutoff_rank(pct: float, n_aq: int) -> int:
    """search.py:396-397 — float64 ``ceil(alpha * L)`` clamped to [1, L]."""
    alpha = pct / 100.0
    return min(n_aq, max(1, math.ceil(alpha * n_aq)))


def two_level(graph, q, params: SearchParams, codebooks: np.ndarray, codes: np.ndarray,
              source, metric: str, qn=None, cached: set | None = None,
              table: np.ndarray | None = None) -> Report:
    """Alg. 2: PQ-gated recompute with per-step promotion (search.py:331-431)."""
    rep = Report()
    funnel = _Funnel(source, cached, rep)
    if table is None:
        table = numerics.adc_build(codebooks, q.shape[0], metric, q, qn)
    exact: dict[int, float] = {}
    _descend(graph, q, metric, qn, funnel, exact)
    eq = _BoundedExact(params.ef)
    for node, d in exact.items():
        eq.offer(node, d)
    exact_known = set(exact)
    approx_sorted: list[tuple[float, int]] = []   # every approx-known node
    approx_known: set[int] = set()
    waiting: list[tuple[float, int]] = []          # eligible, not yet promoted (sorted)
    while (u := eq.next_unvisited()) is not None:
        rep.visits.append(u)
        fresh = [int(w) for w in graph.neighbors(u, 0) if int(w) not in approx_known]
        if fresh:
            aw = numerics.approx_distance_many(table, codes[fresh]).tolist()
            rep.approx_lookups += len(fresh)
            for w, a in zip(fresh, aw):
                approx_known.add(w)
                bisect.insort(approx_sorted, (a, w))
                if w not in exact_known:
                    bisect.insort(waiting, (a, w))
        step: list[int] = []
        if approx_sorted:
            cut = approx_sorted[cutoff_rank(params.rerank_percent, len(approx_sorted)) - 1]
            take = bisect.bisect_right(waiting, cut)
            for _, w in waiting[:take]:
                exact_known.add(w)
                step.append(w)
            del waiting[:take]
        if step:
            for w, dw in zip(step, _dists(funnel.rows(step), q, metric, qn)):
                exact[w] = dw
                eq.offer(w, dw)
    # batch log regrouped at batch_size boundaries (search.py:421-425)
    total = rep.recomputations
    rep.batches = [params.batch_size] * (total // params.batch_size)
    if total % params.batch_size:
        rep.batches.append(total % params.batch_size)
    rep.results = eq.best(params.k, lambda i: not graph.is_deleted(i))
    return rep


def run_search(graph, q, params: SearchParams, source, metric: str,
               codebooks=None, codes=None, qn=None, cached=None) -> Report:
    """search.py:434-443."""
    q = np.asarray(q, dtype=np.float32)
    if params.mode == "exact_bestfirst":
        return best_first(graph, q, params, source, metric, qn, cached)
    if codebooks is None or codes is None:
        raise ValueError("two_level mode requires PQ artifacts")
    return two_level(graph, q, params, codebooks, codes, source, metric, qn, cached)


def merge_pending(results, q, pending_ids, pending_vecs, metric: str, k: int):
    """Engine.search's merge (index.py:320-327) of ``buffer_scan`` (update.py:483-488):
    distance() (vectors.py:94-116) to every pending vector, (d, id)-sorted with
    the graph results, first k."""
    from .numerics import distance
    combined = [(d, i) for i, d in results]
    combined += [(distance(q, v, metric), int(i)) for i, v in zip(pending_ids, pending_vecs)]
    combined.sort()
    return [(i, d) for d, i in combined[:k]]


# --- minimal graph / file readers (graph.py:138-216, pq.py:198-244) ----------

class CsrGraph:
    """Duck-typed graph for the port (graph.py:30-73)."""

    def __init__(self, n, max_degree, entry_point, levels, offsets, neighbors,
                 deleted=None) -> None:
        self.n = int(n)
        self.max_degree = int(max_degree)
        self.entry_point = int(entry_point)
        self.levels = levels
        self.offsets = offsets
        self.nbrs = neighbors
        self.deleted = np.zeros(self.n, dtype=bool) if deleted is None else deleted

    @property
    def level_count(self) -> int:
        return len(self.offsets)

    def neighbors(self, v: int, level: int = 0) -> np.ndarray:
        off = self.offsets[level]
        return self.nbrs[level][int(off[v]):int(off[v + 1])]

    def is_deleted(self, v: int) -> bool:
        return bool(self.deleted[v])

    def out_degrees(self, level: int = 0) -> np.ndarray:
        return np.diff(self.offsets[level].astype(np.int64))


def read_lgr1(path) -> CsrGraph:
    """LGR1: ``<4sHQHHQ>`` header, u16 levels[n], per level count u64, offsets u64[n+1], nbrs u32."""
    import struct
    data = open(path, "rb").read()
    magic, version, n, max_deg, level_count, entry = struct.unpack_from("<4sHQHHQ", data)
    if magic != b"LGR1" or version != 1:
        raise ValueError("bad LGR1 header")
    pos = 26
    levels = np.frombuffer(data, "<u2", n, pos).copy()
    pos += 2 * n
    offs, nbrs = [], []
    for _ in range(level_count):
        (count,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        offs.append(np.frombuffer(data, "<u8", n + 1, pos).copy())
        pos += 8 * (n + 1)
        nbrs.append(np.frombuffer(data, "<u4", count, pos).copy())
        pos += 4 * count
    if pos != len(data):
        raise ValueError("trailing bytes")
    return CsrGraph(n, max_deg, entry, levels, offs, nbrs)


def read_lpq1(path):
    """LPQ1: ``<4sHIIHBxQ>`` header, codebooks f32[m][256][sub], codes u8[n][m]."""
    import struct
    data = open(path, "rb").read()
    magic, version, dim, padded, m, metric_tag, n = struct.unpack_from("<4sHIIHBxQ", data)
    if magic != b"LPQ1" or version != 1:
        raise ValueError("bad LPQ1 header")
    pos = 26
    cb = np.frombuffer(data, "<f4", m * 256 * (padded // m), pos).reshape(m, 256, padded // m).copy()
    pos += cb.nbytes
    codes = np.frombuffer(data, np.uint8, n * m, pos).reshape(n, m).copy()
    return dict(dim=dim, padded_dim=padded, m=m, metric=numerics.METRICS[metric_tag],
                codebooks=cb, codes=codes)


def read_ldl1(path, n: int) -> np.ndarray:
    """LDL1 delete bitset (graph.py:196-216)."""
    data = open(path, "rb").read()
    if data[:4] != b"LDL1":
        raise ValueError("bad LDL1 magic")
    return np.unpackbits(np.frombuffer(data, np.uint8, offset=12), count=n,
                         bitorder="little").astype(bool)
