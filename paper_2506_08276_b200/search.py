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

    def fetch(self, ids, report=None) -> np.ndarray:
        """search.py:89-93 (host rows; the device path reads the matrix in HBM)."""
        m = self.matrix
        if hasattr(m, "data_ptr"):
            import torch
            return m[torch.as_tensor(list(ids), dtype=torch.int64, device=m.device)].cpu().numpy()
        return np.asarray(m)[list(ids)]


class ProviderSource:
    """Recompute source (search.py:96-110). With our
    :class:`paper_2506_08276_b200.encoder.EncoderProvider` the GPU encoder embeds
    the token rows of the requested nodes inside the device loop. Any other
    provider (e.g. the reference's own ``SyntheticProvider``) is a HOST provider:
    the device traversal calls :meth:`fetch` once per iteration with the new ids
    of every in-flight query (``LV_SOURCE_CALLBACK``)."""

    def __init__(self, provider, payload_of=None) -> None:
        self.provider = provider
        self.payload_of = payload_of

    def fetch(self, ids, report=None) -> np.ndarray:
        """search.py:103-110: payload fetch + ``embed_all`` of the provider."""
        if hasattr(self.provider, "embed_batch") and self.payload_of is not None:
            requests = [_EmbeddingRequest(int(i), self.payload_of(int(i))) for i in ids]
            mb = int(getattr(getattr(self.provider, "config", None), "max_batch", 0) or
                     len(requests) or 1)
            rows = [np.asarray(self.provider.embed_batch(requests[j:j + mb]), dtype=np.float32)
                    for j in range(0, len(requests), mb)]
            return np.concatenate(rows) if rows else np.empty((0, 0), np.float32)
        raise InvalidArgumentError("provider has no host embed path")


@dataclass(frozen=True)
class _EmbeddingRequest:
    """vectors.py:33-38 (item_id, content)."""

    item_id: int
    content: bytes


class EmbeddingCache:
    """Pinned exact vectors of the highest-degree nodes (search.py:113-142).

    Built from ids (the device encoder computes the pinned rows once) or, like
    the reference, from ``vectors: {id: row}``."""

    def __init__(self, ids=None, vectors: dict | None = None) -> None:
        if vectors is not None:
            ids = vectors.keys()
        self.ids = np.asarray(sorted(int(i) for i in ids), dtype=np.int64)
        self._set = set(self.ids.tolist())
        self.vectors = vectors

    def __len__(self) -> int:
        return len(self.ids)

    def __contains__(self, node_id: int) -> bool:
        return node_id in self._set


def _cache_ids(cache) -> np.ndarray:
    """Sorted ids of our cache or the reference's (``.vectors`` dict)."""
    if hasattr(cache, "ids"):
        return np.ascontiguousarray(cache.ids, dtype=np.int64)
    return np.asarray(sorted(int(i) for i in cache.vectors), dtype=np.int64)


def _cache_rows(cache, ids: np.ndarray):
    vec = getattr(cache, "vectors", None)
    if not vec:
        return None
    return np.ascontiguousarray(np.stack([np.asarray(vec[int(i)], dtype=np.float32)
                                          for i in ids]))


def _source_kind(source) -> str:
    """matrix | encoder | callback — duck-typed like the reference (search.py:78-110)."""
    prov = getattr(source, "provider", None)
    if prov is None and hasattr(source, "matrix"):
        return "matrix"
    if prov is not None and hasattr(prov, "attach"):
        return "encoder"
    if hasattr(source, "fetch"):
        return "callback"
    raise InvalidArgumentError(
        "source must be MatrixSource, ProviderSource or an object with fetch(ids, report)")


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


def device_query_norms(Q):
    """The same norms computed on the device in the OpenBLAS sdot order
    (lv_numerics.cuh ``sdot_openblas``): bit-identical to :func:`query_norms`
    on a SkylakeX-kernel BLAS host for dim % 32 == 0. CUDA tensor in -> out."""
    import torch
    Q = Q.contiguous()
    out = torch.empty(Q.shape[0], dtype=torch.float32, device=Q.device)
    _lib.check(_lib.lib().lv_query_norms(Q.data_ptr(), Q.shape[0], Q.shape[1], out.data_ptr(),
                                         _lib.LV_IO_DEVICE,
                                         torch.cuda.current_stream(Q.device).cuda_stream))
    return out


def as_pruned(graph):
    """The CSR the device loads: a PrunedGraph (ours or the reference's), or the
    reference's ``OverlayGraph`` (update.py:93-191, what ``Engine.search``
    passes, index.py:315) — its base when nothing is overridden, else a frozen
    snapshot (``OverlayGraph.freeze``) cached on the overlay by content."""
    if hasattr(graph, "level_offsets"):
        return graph
    if hasattr(graph, "overrides") and hasattr(graph, "base"):
        base = graph.base
        deleted = np.asarray(getattr(graph, "_deleted", base.deleted if base is not None else []),
                             dtype=bool)
        if base is not None and graph.n == base.n and not any(graph.overrides):
            return base   # mark_deleted keeps base.deleted in step (update.py:156-161)
        key = (graph.n, graph.entry_point,
               tuple((lvl, v, tuple(row)) for lvl, d in enumerate(graph.overrides)
                     for v, row in sorted(d.items())))
        snap = graph.__dict__.get("_lv_frozen")
        if snap is None or snap[0] != key:
            snap = (key, graph.freeze(graph.max_degree))
            graph.__dict__["_lv_frozen"] = snap
        snap[1].deleted = deleted
        return snap[1]
    raise InvalidArgumentError("graph must be a PrunedGraph or an OverlayGraph")


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
        self._matrix_ref = None
        self._cache_ref = None   # the cache object whose ids/rows are on the device
        self._cache_rows_set = False
        self._encoder = None
        self._fetch = None

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
        if matrix is self._matrix_ref:   # strong reference held: identity is safe
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
        self._matrix_ref = matrix

    def attach_encoder(self, provider) -> None:
        if self._encoder is provider:
            return
        provider.attach(self)
        self._encoder = provider
        self._cache_ref = None

    def set_cache(self, cache, source_kind: str = "encoder", source=None) -> None:
        """Device copy of an EmbeddingCache (ours or the reference's). The
        cache object is held, so identity comparison cannot alias a freed one.
        Pinned rows: the reference cache's ``vectors`` when present, else the
        attached encoder's (encoder source) or ``source.fetch`` (host provider)."""
        if cache is self._cache_ref and (cache is None or source_kind == "matrix"
                                         or self._cache_rows_set):
            return
        ids = None if cache is None else _cache_ids(cache)
        _lib.check(_lib.lib().lv_index_set_cache(
            self.handle, None if ids is None else ids.ctypes.data,
            0 if ids is None else ids.shape[0], 0))
        self._cache_ref = cache
        self._cache_rows_set = source_kind == "encoder" and self._encoder is not None
        if cache is None or source_kind == "matrix" or not len(ids):
            return
        rows = _cache_rows(cache, ids)
        if rows is None and source_kind == "callback":
            rows = np.ascontiguousarray(source.fetch(ids.tolist(), SearchReport()),
                                        dtype=np.float32)
        if rows is not None:
            if rows.shape != (ids.shape[0], self.dim):
                raise InvalidArgumentError("cache vectors do not match the index dim")
            _lib.check(_lib.lib().lv_index_set_cache_rows(self.handle, rows.ctypes.data, 0))
            self._cache_rows_set = True

    def _bind_source(self, source, p, dry_matrix=None) -> str:
        """Point the device at the source; returns its kind."""
        kind = _source_kind(source)
        if kind == "matrix":
            p.source = _lib.LV_SOURCE_MATRIX
            self.set_matrix(source.matrix)
        elif kind == "encoder":
            p.source = _lib.LV_SOURCE_ENCODER
            if dry_matrix is not None:
                p.flags |= _lib.LV_DRY_RECOMPUTE
                self.set_matrix(dry_matrix)
            else:
                self.attach_encoder(source.provider)
        else:
            p.source = _lib.LV_SOURCE_CALLBACK
        return kind

    def _install_fetch(self, source, report: "SearchReport", errors: list):
        """ctypes trampoline: lv_fetch_fn -> source.fetch(ids, report)."""
        dim = self.dim

        def fn(_user, ids_p, n, rows_p):
            try:
                ids = np.ctypeslib.as_array(ids_p, shape=(n,)).tolist()
                rows = np.asarray(source.fetch(ids, report), dtype=np.float32)
                if rows.shape != (n, dim):
                    raise InvalidArgumentError(
                        f"provider returned {rows.shape}, expected ({n}, {dim})")
                np.ctypeslib.as_array(rows_p, shape=(n, dim))[...] = rows
                return 0
            except BaseException as exc:   # surfaced after the call (LV_ERR_PROVIDER)
                errors.append(exc)
                return 1

        cfn = _lib.FETCH_FN(fn)
        _lib.check(_lib.lib().lv_index_set_fetch(self.handle, cfn, None))
        self._fetch = cfn   # keep the trampoline alive
        return cfn

    def _run(self, call, kind, source, report):
        """Run lv_search_batch; a host-provider failure becomes SearchError
        with the partial report (search.py:169-172)."""
        errors: list = []
        if kind == "callback":
            self._install_fetch(source, report, errors)
        try:
            rc = call()
        finally:
            if kind == "callback":
                _lib.lib().lv_index_set_fetch(self.handle, _lib.FETCH_FN(0), None)
                self._fetch = None
        if rc != 0 and errors:
            from .errors import ProviderError, SearchError
            exc = errors[0]
            if isinstance(exc, ProviderError) or type(exc).__name__ == "ProviderError":
                raise SearchError(str(exc), partial_report=report) from exc
            raise exc
        _lib.check(rc)

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
        kind = self._bind_source(source, p)
        self.set_cache(cache, kind, source)
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
        scratch = SearchReport()
        self._run(lambda: _lib.lib().lv_search_batch(self.handle, Q.ctypes.data, qn.ctypes.data,
                                                      B, C.byref(p), C.byref(o), stream),
                  kind, source, scratch)
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
                      dry_matrix=None, smem_lut: bool = False, hash_visited: bool = False):
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
        p.flags = (_lib.LV_IO_DEVICE | (0 if shared_recompute else _lib.LV_NO_SHARED_RECOMPUTE)
                   | (_lib.LV_SMEM_LUT if smem_lut else 0)
                   | (_lib.LV_HASH_VISITED if hash_visited else 0))
        kind = self._bind_source(source, p, dry_matrix)
        self.set_cache(cache, kind, source)
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
        self._run(lambda: _lib.lib().lv_search_batch(self.handle, Q.data_ptr(), qp, B,
                                                      C.byref(p), C.byref(o), st),
                  kind, source, SearchReport())
        return out

    def last_stats(self) -> dict:
        st = _lib.SearchStats()
        _lib.check(_lib.lib().lv_last_search_stats(self.handle, C.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}


def device_index_for(graph, pq_model=None, pq_codes=None, metric=None,
                     dim=None) -> DeviceIndex:
    """Per-(graph, PQ) cached DeviceIndex (the index is immutable, graph.py:32).
    Entries hold the PQ objects they were built from and match by identity, so
    a retrained model can never reuse a freed object's device copy."""
    graph = as_pruned(graph)
    entries = graph.__dict__.setdefault("_lv_device", [])
    for e in entries:
        if e[0] is pq_model and e[1] is pq_codes and e[2] == metric and e[3] == dim:
            dev = e[4]
            break
    else:
        dev = DeviceIndex(graph, pq_model, pq_codes, metric, dim=dim)
        entries.append((pq_model, pq_codes, metric, dim, dev))
    dev.sync_deleted(graph.deleted)
    return dev


# --------------------------------------------------------------------------- reference API

def search_batch(graph, Q, params: SearchParams, source, metric: str, pq_model=None,
                 pq_codes=None, cache: EmbeddingCache | None = None, qn=None,
                 trace: bool = False) -> list[SearchReport]:
    """Batched ``run_search``: all queries traverse concurrently on the device."""
    if params.mode == "two_level" and (pq_model is None or pq_codes is None):
        raise InvalidArgumentError("two_level mode requires PQ artifacts")
    graph = as_pruned(graph)
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


def merge_pending(reports: list, Q, pending_ids, pending_vectors, metric: str, k: int,
                  qn=None) -> list:
    """``Engine.search``'s merge of the buffered (not yet inserted) items
    (index.py:320-327 over ``MutableIndex.buffer_scan``, update.py:483-488):
    distance() of each query to every pending vector (vectors.py:94-116, the
    np.dot order) on the device, merged with the graph results by (distance,
    id), first k kept. Updates and returns ``reports``."""
    _lib.require_device()
    pid = np.ascontiguousarray(pending_ids, dtype=np.int64).reshape(-1)
    if pid.size == 0 or not reports:
        return reports
    pv = np.ascontiguousarray(pending_vectors, dtype=np.float32).reshape(pid.shape[0], -1)
    Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(len(reports), -1)
    if Q.shape[1] != pv.shape[1]:
        raise InvalidArgumentError(f"dimension mismatch: {Q.shape[1]} vs {pv.shape[1]}")
    B = len(reports)
    ids = np.full((B, k), -1, np.int64)
    dist = np.zeros((B, k), np.float32)
    count = np.zeros(B, np.int32)
    for b, rep in enumerate(reports):
        res = rep.results[:k]
        count[b] = len(res)
        for j, (i, d) in enumerate(res):
            ids[b, j], dist[b, j] = i, d
    qn_p = None
    if qn is not None:
        qn = np.ascontiguousarray(qn, dtype=np.float32)
        qn_p = qn.ctypes.data
    _lib.check(_lib.lib().lv_merge_pending(
        _lib.LV_METRIC[metric], pv.ctypes.data, pid.ctypes.data, pid.shape[0], pv.shape[1],
        Q.ctypes.data, qn_p, B, k, ids.ctypes.data, dist.ctypes.data, count.ctypes.data, 0,
        None))
    for b, rep in enumerate(reports):
        rep.results = [(int(ids[b, j]), float(dist[b, j])) for j in range(int(count[b]))]
    return reports
