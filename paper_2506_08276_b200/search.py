"""Query engine front end — the reference's search API over the B200 kernels.

Mirrors ``slimvec.search`` (search.py:37-443): ``SearchParams``,
``SearchReport``, ``MatrixSource``, ``ProviderSource``, ``EmbeddingCache``,
``build_embedding_cache``, ``run_search``, ``two_level_search``,
``best_first_search`` — same argument meaning, validation and errors. The
work itself runs in ``libleann_b200.so`` (lv_search_batch): a batch of queries
is traversed concurrently on the GPU, one warp per in-flight query, with the
recompute requests of all in-flight queries packed into one encoder forward.
There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidArgumentError

MODES = ("exact_bestfirst", "two_level")
STAGES = ("pq_lookup", "payload_fetch", "embed", "distance")


@dataclass
class SearchParams:
    """search.py:37-56 (same defaults and validation)."""

    k: int = 3
    ef: int = 50
    rerank_percent: float = 30.0
    batch_size: int = 64
    mode: str = "two_level"
    cache_percent: float | None = None

    def __post_init__(self) -> None:
        if self.k < 1 or self.ef < self.k:
            raise InvalidArgumentError("need ef >= k >= 1")
        if not 0 < self.rerank_percent <= 100:
            raise InvalidArgumentError("rerank_percent must be in (0, 100]")
        if self.batch_size < 1:
            raise InvalidArgumentError("batch_size must be >= 1")
        if self.mode not in MODES:
            raise InvalidArgumentError(f"unknown mode: {self.mode!r}")
        if self.cache_percent is not None and not 0 < self.cache_percent <= 100:
            raise InvalidArgumentError("cache_percent must be in (0, 100]")


@dataclass
class SearchReport:
    """search.py:59-72; ``visits`` is the optional base-layer expansion trace."""

    results: list = field(default_factory=list)
    recomputations: int = 0
    approx_lookups: int = 0
    batches: list = field(default_factory=list)
    cache_hits: int = 0
    stage_times: dict = field(default_factory=lambda: dict.fromkeys(STAGES, 0.0))
    wall_time: float = 0.0
    expansions: int = 0
    visits: list | None = None

    @property
    def cache_hit_rate(self) -> float:
        seen = self.cache_hits + self.recomputations
        return self.cache_hits / seen if seen else 0.0


class MatrixSource:
    """Oracle-mode source (search.py:78-93): exact vectors are rows of a resident matrix.

    ``matrix`` is a float32 numpy array or a CUDA torch tensor (n, dim).
    """

    def __init__(self, matrix) -> None:
        self.matrix = matrix


class ProviderSource:
    """Recompute source (search.py:96-110): the attached GPU encoder embeds the
    token payloads of the requested nodes. ``provider`` must be an
    :class:`paper_2506_08276_b200.encoder.EncoderProvider` bound to the
    index's token store."""

    def __init__(self, provider, payload_of=None) -> None:
        self.provider = provider
        self.payload_of = payload_of


class EmbeddingCache:
    """Pinned exact vectors of the highest-degree nodes (search.py:113-142)."""

    def __init__(self, ids) -> None:
        self.ids = np.asarray(sorted(int(i) for i in ids), dtype=np.int64)
        self._set = set(self.ids.tolist())

    def __len__(self) -> int:
        return len(self.ids)

    def __contains__(self, node_id: int) -> bool:
        return node_id in self._set


def build_embedding_cache(graph, fraction_percent: float, source=None) -> EmbeddingCache:
    """Top ceil(f*n/100) nodes by (out-degree desc, id asc) (search.py:130-142)."""
    if not 0 < fraction_percent <= 100:
        raise InvalidArgumentError("cache fraction must be in (0, 100]")
    n = graph.n
    count = min(n, math.ceil(fraction_percent / 100.0 * n))
    order = np.lexsort((np.arange(n), -graph.out_degrees(0)))
    return EmbeddingCache(order[:count])


def query_norm(q: np.ndarray) -> np.float32:
    """``np.float32(np.sqrt(np.dot(q, q)))`` on the host (vectors.py:138, pq.py:163)."""
    q = np.asarray(q, dtype=np.float32)
    return np.float32(np.sqrt(np.dot(q, q)))


def query_norms(Q: np.ndarray) -> np.ndarray:
    return np.array([query_norm(q) for q in Q], dtype=np.float32)


# --------------------------------------------------------------------------- device index

class DeviceIndex:
    """One graph + PQ index resident in HBM (an ``lv_index`` handle)."""

    def __init__(self, graph, pq_model=None, pq_codes=None, metric: str | None = None,
                 device: int = 0, dim: int | None = None) -> None:
        _lib.require_device()
        L = _lib.lib()
        if metric is None:
            if pq_model is None:
                raise InvalidArgumentError("metric required without a PQ model")
            metric = pq_model.metric
        if metric not in _lib.LV_METRIC:
            raise InvalidArgumentError(f"unknown metric: {metric!r}")
        self.metric = metric
        self.n = int(graph.n)
        self.dim = int(pq_model.dim if pq_model is not None else (dim or 0))
        if self.dim < 1:
            raise InvalidArgumentError("dim required without a PQ model")
        self._pq_m = int(pq_model.m_pq) if pq_model is not None else 0
        self.device = device
        lc = graph.level_count
        offs = [np.ascontiguousarray(o, dtype=np.uint64) for o in graph.level_offsets]
        nbrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in graph.level_neighbors]
        self._keep = (offs, nbrs)
        off_p = (C.c_void_p * lc)(*[o.ctypes.data for o in offs])
        nb_p = (C.c_void_p * lc)(*[x.ctypes.data if x.size else None for x in nbrs])
        nnz = (C.c_uint64 * lc)(*[x.shape[0] for x in nbrs])
        d = _lib.IndexDesc()
        d.n = self.n
        d.metric = _lib.LV_METRIC[metric]
        d.max_degree = int(max(1, graph.max_degree))
        d.level_count = lc
        d.entry_point = int(graph.entry_point)
        d.level_offsets = C.cast(off_p, C.POINTER(C.c_void_p))
        d.level_neighbors = C.cast(nb_p, C.POINTER(C.c_void_p))
        d.level_nnz = C.cast(nnz, C.POINTER(C.c_uint64))
        self._deleted = np.asarray(graph.deleted, dtype=bool).copy()
        dele = self._deleted.astype(np.uint8)
        d.deleted = dele.ctypes.data if self._deleted.any() else None
        if pq_model is not None:
            cb = np.ascontiguousarray(pq_model.codebooks, dtype=np.float32)
            codes = np.ascontiguousarray(pq_codes.codes, dtype=np.uint8)
            if codes.shape[0] != self.n:
                raise InvalidArgumentError("PQ codes do not match the graph size")
            d.dim = pq_model.dim
            d.pq_m = pq_model.m_pq
            d.pq_padded_dim = pq_model.padded_dim
            d.pq_codebooks = cb.ctypes.data
            d.pq_codes = codes.ctypes.data
        else:
            d.dim = self.dim
        handle = C.c_void_p()
        _lib.check(L.lv_index_create(C.byref(d), device, C.byref(handle)))
        self.handle = handle
        self._matrix_key = None
        self._matrix_ref = None
        self._cache_key = None
        self._encoder = None

    @classmethod
    def for_pq(cls, model) -> "DeviceIndex":
        """Single-node index carrying only the PQ codebooks (for adc_build)."""
        from .graph import PrunedGraph
        from .pq import PQCodes
        g = PrunedGraph(n=1, max_degree=1, entry_point=0, levels=np.zeros(1, np.uint16),
                        level_offsets=[np.zeros(2, np.uint64)],
                        level_neighbors=[np.zeros(0, np.uint32)])
        return cls(g, model, PQCodes(np.zeros((1, model.m_pq), np.uint8)))

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().lv_index_destroy(self.handle)
            self.handle = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def sync_deleted(self, deleted: np.ndarray) -> None:
        deleted = np.asarray(deleted, dtype=bool)
        if np.array_equal(deleted, self._deleted):
            return
        self._deleted = deleted.copy()
        arr = deleted.astype(np.uint8)
        _lib.check(_lib.lib().lv_index_set_deleted(self.handle, arr.ctypes.data if deleted.any()
                                                    else None, 0))

    def set_matrix(self, matrix) -> None:
        key = id(matrix)
        if key == self._matrix_key:
            return
        if hasattr(matrix, "data_ptr"):
            if tuple(matrix.shape) != (self.n, self.dim) or str(matrix.dtype) != "torch.float32":
                raise InvalidArgumentError("matrix must be float32 (n, dim)")
            _lib.check(_lib.lib().lv_index_set_matrix(self.handle, matrix.data_ptr(),
                                                      _lib.LV_IO_DEVICE))
        else:
            m = np.ascontiguousarray(matrix, dtype=np.float32)
            if m.shape != (self.n, self.dim):
                raise InvalidArgumentError(f"matrix shape {m.shape} != ({self.n}, {self.dim})")
            _lib.check(_lib.lib().lv_index_set_matrix(self.handle, m.ctypes.data, 0))
        self._matrix_key = key
        self._matrix_ref = matrix

    def attach_encoder(self, provider) -> None:
        if self._encoder is provider:
            return
        provider.attach(self)
        self._encoder = provider
        self._cache_key = None

    def set_cache(self, cache: EmbeddingCache | None) -> None:
        key = None if cache is None else id(cache)
        if key == self._cache_key:
            return
        ids = None if cache is None else np.ascontiguousarray(cache.ids, dtype=np.int64)
        _lib.check(_lib.lib().lv_index_set_cache(
            self.handle, None if ids is None else ids.ctypes.data,
            0 if ids is None else ids.shape[0], 0))
        self._cache_key = key

    # -- ADC / distances (pq.py:153-189, vectors.py:120-140)
    def adc_tables(self, Q: np.ndarray, qn: np.ndarray) -> np.ndarray:
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        qn = np.ascontiguousarray(qn, dtype=np.float32)
        m = _lib.lib()
        out = np.empty((Q.shape[0],) + self._lut_shape(), dtype=np.float32)
        _lib.check(m.lv_adc_tables(self.handle, Q.ctypes.data, qn.ctypes.data, Q.shape[0],
                                   out.ctypes.data, 0, None))
        return out

    def _lut_shape(self):
        return (self._pq_m, 256)

    def adc_score(self, table: np.ndarray, ids: np.ndarray) -> np.ndarray:
        table = np.ascontiguousarray(table, dtype=np.float32)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.empty(ids.shape[0], dtype=np.float32)
        _lib.check(_lib.lib().lv_adc_score(self.handle, table.ctypes.data, ids.ctypes.data,
                                           ids.shape[0], out.ctypes.data, 0, None))
        return out

    # -- search
    def search(self, Q, params: SearchParams, source, qn=None,
               cache: EmbeddingCache | None = None, trace: bool = False,
               max_inflight: int = 0, stream=None,
               shared_recompute: bool = True) -> list[SearchReport]:
        """Run ``len(Q)`` queries concurrently; one ``SearchReport`` per query."""
        t0 = time.perf_counter()
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        if Q.ndim == 1:
            Q = Q.reshape(1, -1)
        B = Q.shape[0]
        if Q.shape[1] != self.dim:
            raise InvalidArgumentError(f"dimension mismatch: {Q.shape[1]} vs {self.dim}")
        qn = query_norms(Q) if qn is None else np.ascontiguousarray(qn, dtype=np.float32)
        p = _lib.SearchParamsC()
        p.k, p.ef = params.k, params.ef
        p.rerank_percent = float(params.rerank_percent)
        p.batch_size = params.batch_size
        p.mode = _lib.LV_MODE[params.mode]
        p.max_inflight = max_inflight
        p.flags = 0 if shared_recompute else _lib.LV_NO_SHARED_RECOMPUTE
        if isinstance(source, MatrixSource):
            p.source = _lib.LV_SOURCE_MATRIX
            self.set_matrix(source.matrix)
        elif isinstance(source, ProviderSource):
            p.source = _lib.LV_SOURCE_ENCODER
            self.attach_encoder(source.provider)
        else:
            raise InvalidArgumentError(
                "source must be MatrixSource or ProviderSource(EncoderProvider); "
                "the device path has no CPU fallback")
        self.set_cache(cache)
        p.use_cache = 1 if cache is not None else 0
        k = params.k
        ids = np.empty((B, k), dtype=np.int64)
        dist = np.empty((B, k), dtype=np.float32)
        count = np.empty(B, dtype=np.int32)
        counters = np.empty((B, 4), dtype=np.int64)
        status = np.empty(B, dtype=np.int32)
        o = _lib.SearchOutputs()
        o.ids, o.dist, o.count = ids.ctypes.data, dist.ctypes.data, count.ctypes.data
        o.counters, o.status = counters.ctypes.data, status.ctypes.data
        blog_cap = 0
        if params.mode == "exact_bestfirst":
            blog_cap = max(256, 8 * params.ef + 256)
            blog = np.empty((B, blog_cap), dtype=np.int32)
            o.batch_log, o.batch_log_cap = blog.ctypes.data, blog_cap
        vis_cap = 0
        if trace:
            vis_cap = max(256, 4 * params.ef + 256)
            vis = np.empty((B, vis_cap), dtype=np.int32)
            o.visits, o.visits_cap = vis.ctypes.data, vis_cap
        _lib.check(_lib.lib().lv_search_batch(self.handle, Q.ctypes.data, qn.ctypes.data, B,
                                              C.byref(p), C.byref(o), stream))
        wall = time.perf_counter() - t0
        reports = []
        for b in range(B):
            rep = SearchReport()
            rep.results = [(int(ids[b, j]), float(dist[b, j])) for j in range(int(count[b]))]
            rep.recomputations = int(counters[b, 0])
            rep.approx_lookups = int(counters[b, 1])
            rep.cache_hits = int(counters[b, 2])
            rep.expansions = int(counters[b, 3])
            if params.mode == "two_level":
                total, bs = rep.recomputations, params.batch_size
                rep.batches = [bs] * (total // bs) + ([total % bs] if total % bs else [])
            else:
                row = blog[b]
                rep.batches = [int(x) for x in row[row >= 0]]
                if sum(rep.batches) != rep.recomputations:
                    raise InvalidArgumentError("batch log overflow; lower ef")
            if trace:
                row = vis[b]
                if rep.expansions > vis_cap:
                    raise InvalidArgumentError("visit trace overflow")
                rep.visits = [int(x) for x in row[:rep.expansions]]
            rep.wall_time = wall / B
            reports.append(rep)
        return reports

    def search_device(self, Q, params: SearchParams, source, qn=None,
                      cache: EmbeddingCache | None = None, max_inflight: int = 0,
                      out: dict | None = None, shared_recompute: bool = True,
                      dry_matrix=None):
        """Device-resident batch search: ``Q`` is a CUDA float32 tensor [B, dim],
        ``qn`` a CUDA tensor [B] or None (norms then computed on the device).
        Returns CUDA tensors ids [B, k] (int64, -1 padded), dist [B, k],
        count [B], counters [B, 4] (recomputations, approx_lookups, cache_hits,
        expansions). Stream-ordered on the current torch stream.
        ``dry_matrix`` (with a ProviderSource): rows the encoder would produce,
        used instead of running it (LV_DRY_RECOMPUTE) — same results, counters
        and physical-recompute statistics, for tuning."""
        import torch
        if not (Q.is_cuda and Q.dtype == torch.float32 and Q.is_contiguous() and Q.dim() == 2):
            raise InvalidArgumentError("Q must be a contiguous CUDA float32 [B, dim] tensor")
        if Q.shape[1] != self.dim:
            raise InvalidArgumentError(f"dimension mismatch: {Q.shape[1]} vs {self.dim}")
        B, k = Q.shape[0], params.k
        p = _lib.SearchParamsC()
        p.k, p.ef = k, params.ef
        p.rerank_percent = float(params.rerank_percent)
        p.batch_size = params.batch_size
        p.mode = _lib.LV_MODE[params.mode]
        p.max_inflight = max_inflight
        p.flags = _lib.LV_IO_DEVICE | (0 if shared_recompute else _lib.LV_NO_SHARED_RECOMPUTE)
        if isinstance(source, MatrixSource):
            p.source = _lib.LV_SOURCE_MATRIX
            self.set_matrix(source.matrix)
        elif isinstance(source, ProviderSource) and dry_matrix is not None:
            p.source = _lib.LV_SOURCE_ENCODER
            p.flags |= _lib.LV_DRY_RECOMPUTE
            self.set_matrix(dry_matrix)
        elif isinstance(source, ProviderSource):
            p.source = _lib.LV_SOURCE_ENCODER
            self.attach_encoder(source.provider)
        else:
            raise InvalidArgumentError("source must be MatrixSource or ProviderSource")
        self.set_cache(cache)
        p.use_cache = 1 if cache is not None else 0
        dev = Q.device
        if out is None or out["ids"].shape[0] < B or out["ids"].shape[1] != k:
            out = dict(ids=torch.empty((B, k), dtype=torch.int64, device=dev),
                       dist=torch.empty((B, k), dtype=torch.float32, device=dev),
                       count=torch.empty(B, dtype=torch.int32, device=dev),
                       counters=torch.empty((B, 4), dtype=torch.int64, device=dev),
                       status=torch.empty(B, dtype=torch.int32, device=dev))
        o = _lib.SearchOutputs()
        o.ids, o.dist = out["ids"].data_ptr(), out["dist"].data_ptr()
        o.count, o.counters = out["count"].data_ptr(), out["counters"].data_ptr()
        o.status = out["status"].data_ptr()
        st = torch.cuda.current_stream(dev).cuda_stream
        qp = None if qn is None else qn.data_ptr()
        _lib.check(_lib.lib().lv_search_batch(self.handle, Q.data_ptr(), qp, B, C.byref(p),
                                              C.byref(o), st))
        return out

    def last_stats(self) -> dict:
        st = _lib.SearchStats()
        _lib.check(_lib.lib().lv_last_search_stats(self.handle, C.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}


def device_index_for(graph, pq_model=None, pq_codes=None, metric=None,
                     dim=None) -> DeviceIndex:
    """Per-(graph, PQ) cached DeviceIndex (the index is immutable, graph.py:32)."""
    cache = graph.__dict__.setdefault("_lv_device", {})
    key = (id(pq_model), id(pq_codes), metric, dim)
    dev = cache.get(key)
    if dev is None:
        dev = DeviceIndex(graph, pq_model, pq_codes, metric, dim=dim)
        cache[key] = dev
    dev.sync_deleted(graph.deleted)
    return dev


# --------------------------------------------------------------------------- reference API

def search_batch(graph, Q, params: SearchParams, source, metric: str, pq_model=None,
                 pq_codes=None, cache: EmbeddingCache | None = None, qn=None,
                 trace: bool = False) -> list[SearchReport]:
    """Batched ``run_search``: all queries traverse concurrently on the device."""
    if params.mode == "two_level" and (pq_model is None or pq_codes is None):
        raise InvalidArgumentError("two_level mode requires PQ artifacts")
    if pq_model is not None and pq_model.metric != metric:
        raise InvalidArgumentError("metric differs from the PQ model's metric")
    Q = np.asarray(Q, dtype=np.float32)
    if pq_model is None:
        dev = device_index_for(graph, None, None, metric, dim=int(Q.shape[-1]))
    else:
        dev = device_index_for(graph, pq_model, pq_codes)
    return dev.search(Q, params, source, qn=qn, cache=cache, trace=trace)


def run_search(graph, q, params: SearchParams, source, metric: str, pq_model=None,
               pq_codes=None, cache: EmbeddingCache | None = None) -> SearchReport:
    """search.py:434-443 for one query."""
    return search_batch(graph, np.asarray(q, dtype=np.float32).reshape(1, -1), params, source,
                        metric, pq_model, pq_codes, cache)[0]


def two_level_search(graph, q, params: SearchParams, pq_model, pq_codes, source, metric: str,
                     cache: EmbeddingCache | None = None) -> SearchReport:
    """search.py:331-431."""
    if params.mode != "two_level":
        params = SearchParams(params.k, params.ef, params.rerank_percent, params.batch_size,
                              "two_level", params.cache_percent)
    return run_search(graph, q, params, source, metric, pq_model, pq_codes, cache)


def best_first_search(graph, q, params: SearchParams, source, metric: str,
                      cache: EmbeddingCache | None = None) -> SearchReport:
    """search.py:288-328."""
    if params.mode != "exact_bestfirst":
        params = SearchParams(params.k, params.ef, params.rerank_percent, params.batch_size,
                              "exact_bestfirst", params.cache_percent)
    return run_search(graph, q, params, source, metric, None, None, cache)
