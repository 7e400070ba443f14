"""User-facing index API: ``build`` and ``LeannSearcher.search(query, top_k, complexity, recompute)``.

Mirrors the reference facade (``build_index_dir`` index.py:173-213 and
``Engine.search`` index.py:305-328, which embeds the query with the index's
provider, ``embed_query`` index.py:291-294, and calls ``run_search``
search.py:434-443) over a batch of queries at once:

* ``complexity`` is the search-list size ``ef`` (SearchParams.ef);
* ``recompute=True`` recomputes candidate embeddings with the GPU encoder from
  the token store (ProviderSource, search.py:96-110); ``recompute=False``
  scores against a resident embedding matrix (MatrixSource, search.py:78-93);
* a query is a token row (embedded with the index's encoder, like
  ``embed_query``) or an already-embedded float vector (the ndarray
  pass-through of Engine.search).

On-disk layout (same files the reference reads, so ``slimvec.Engine.open``
opens a directory written here): ``graph.bin`` (LGR1), ``pq.bin`` (LPQ1),
``deleted.bin`` (LDL1), ``items.dat``/``items.idx`` (token store), ``meta.txt``
(index.py:130-170 keys), ``mutations.log`` (empty journal).
"""
from __future__ import annotations

import ctypes as C
import hashlib
from pathlib import Path

import numpy as np

from . import _lib
from .builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
from .encoder import EncoderProvider, GpuEncoder, TokenStore
from .errors import FormatError, InvalidArgumentError
from .graph import load_graph, save_deleted, save_graph
from .pq import load_pq, save_pq
from .search import (MatrixSource, ProviderSource, SearchParams, build_embedding_cache,
                     device_index_for)

META_VERSION = "1"   # index.py:64


def provider_hash(kind: str, dim: int, seed: int = 0) -> str:
    """vectors.py:68-79: blake2b-64 of the value-determining provider fields."""
    key = f"synthetic:{dim}:{seed}" if kind == "synthetic" else f"external:{dim}"
    return hashlib.blake2b(key.encode(), digest_size=8).hexdigest()


def write_meta(path, mapping: dict) -> None:
    """index.py:130-132: sorted ``key=value`` lines."""
    Path(path).write_text("".join(f"{k}={mapping[k]}\n" for k in sorted(mapping)))


def read_meta(path) -> dict:
    """index.py:135-148."""
    try:
        text = Path(path).read_text()
    except FileNotFoundError:
        raise FormatError("meta", f"missing {path}")
    out = {}
    for line in text.splitlines():
        if not line.strip():
            continue
        if "=" not in line:
            raise FormatError("meta", f"malformed line: {line!r}")
        key, _, value = line.partition("=")
        out[key] = value
    return out


def meta_for(params: GpuBuildParams, n: int, dim: int) -> dict:
    """index.py:151-170 keys. The GPU encoder is an external-kind provider to
    the reference (``provider_hash`` of ``external:{dim}``), so
    ``slimvec.Engine.open`` accepts the directory; ``provider_model`` (extra
    key, ignored by the reference) names the encoder."""
    return {"format_version": META_VERSION, "n": n, "dim": dim, "metric": params.metric,
            "provider_kind": "external", "provider_seed": 0, "provider_max_batch": 64,
            "provider_hash": provider_hash("external", dim),
            "ef_construction": params.candidates, "max_degree": params.max_degree,
            "low_degree": params.low_degree, "hub_percent": params.hub_percent,
            "budget_bytes": "", "pq_subspaces": params.pq_subspaces or "",
            "seed": params.seed, "k_shards": 1}


def build(tokens, encoder: GpuEncoder, out_dir=None, params: GpuBuildParams | None = None,
          return_embeddings: bool = False):
    """Embed every passage with ``encoder``, build the pruned graph and PQ codes,
    and (optionally) write the index directory. Returns (graph, pq_model,
    pq_codes[, embeddings])."""
    import torch
    params = params or GpuBuildParams()
    if hasattr(tokens, "data_ptr"):
        tok_dev = tokens
    else:
        t = np.ascontiguousarray(tokens)
        tok_dev = torch.from_numpy(t.view(np.int16) if t.dtype == np.uint16 else
                                   t.view(np.int32)).cuda()
    E = encoder.encode(tok_dev)
    graph = build_graph_gpu(E, params)
    model, codes = train_pq_gpu(E, params.pq_subspaces, params.metric, params.pq_iters,
                                params.seed)
    if out_dir is not None:
        d = Path(out_dir)
        d.mkdir(parents=True, exist_ok=True)
        save_graph(graph, d / "graph.bin")
        save_pq(model, codes, d / "pq.bin")
        save_deleted(graph.deleted, d / "deleted.bin")
        if not hasattr(tokens, "data_ptr"):
            TokenStore(np.asarray(tokens)).save(d)
        meta = meta_for(params, graph.n, int(E.shape[1]))
        meta["provider_model"] = encoder.cfg.name
        write_meta(d / "meta.txt", meta)
        (d / "mutations.log").write_bytes(b"")
    out = (graph, model, codes)
    return out + (E,) if return_embeddings else out


class LeannSearcher:
    """A resident index (graph + PQ + token store + encoder) on one GPU."""

    def __init__(self, graph, pq_model, pq_codes, encoder: GpuEncoder, tokens,
                 matrix=None, rerank_percent: float = 30.0, batch_size: int = 64,
                 cache_percent: float | None = None) -> None:
        self.graph = graph
        self.pq_model = pq_model
        self.pq_codes = pq_codes
        self.encoder = encoder
        self.provider = EncoderProvider(encoder, tokens if hasattr(tokens, "data_ptr")
                                        else TokenStore(tokens))
        self.matrix = matrix
        self.rerank_percent = rerank_percent
        self.batch_size = batch_size
        self.device_index = device_index_for(graph, pq_model, pq_codes)
        self.metric = pq_model.metric
        self._out = None
        # buffered adds not yet inserted into the graph (MutableIndex.buffer,
        # update.py:459-515): ids + exact vectors, merged into every result
        self._pending_ids = np.empty(0, np.int64)
        self._pending_vecs = np.empty((0, pq_model.dim), np.float32)
        self._pending_dev = None
        # hub-node embedding cache (build_embedding_cache, search.py:130-142):
        # pinned exact vectors, results-transparent, computed once at open time
        self.cache = (build_embedding_cache(graph, cache_percent)
                      if cache_percent else None)

    @classmethod
    def open(cls, index_dir, encoder: GpuEncoder, token_bytes: int = 2, **kw) -> "LeannSearcher":
        d = Path(index_dir)
        g = load_graph(d / "graph.bin")
        model, codes = load_pq(d / "pq.bin")
        store = TokenStore.load(d, token_bytes)
        return cls(g, model, codes, encoder, store.tokens, **kw)

    def _params(self, top_k: int, complexity: int) -> SearchParams:
        return SearchParams(k=top_k, ef=max(complexity, top_k),
                            rerank_percent=self.rerank_percent, batch_size=self.batch_size)

    def embed_queries(self, queries):
        """Token rows -> unit query vectors on the device (embed_query, index.py:291-294)."""
        import torch
        if hasattr(queries, "data_ptr"):
            if queries.dtype == torch.float32:
                return queries
            return self.encoder.encode(queries)
        q = np.asarray(queries)
        if q.dtype == np.float32:
            return torch.from_numpy(np.ascontiguousarray(q.reshape(-1, q.shape[-1]))).cuda()
        q = np.ascontiguousarray(q.reshape(-1, q.shape[-1]))
        dev = torch.from_numpy(q.view(np.int16) if q.dtype == np.uint16 else
                               q.astype(np.int32)).cuda(non_blocking=True)
        return self.encoder.encode(dev)

    # -- buffered adds (MutableIndex.buffered_add / buffer_scan, update.py:459-488)
    def add_pending(self, ids, vectors) -> None:
        """Hold already-embedded items (ids >= n, not yet in the graph): every
        search merges them exactly, like ``Engine.search`` (index.py:320-327)."""
        ids = np.asarray(ids, dtype=np.int64).reshape(-1)
        vecs = np.ascontiguousarray(vectors, dtype=np.float32).reshape(ids.shape[0], -1)
        if vecs.shape[1] != self._pending_vecs.shape[1]:
            raise InvalidArgumentError("pending vectors do not match the index dim")
        if ids.size and (ids.min() < self.graph.n or
                         np.intersect1d(ids, self._pending_ids).size or
                         np.unique(ids).size != ids.size):
            raise InvalidArgumentError("pending ids must be new (>= n) and distinct")
        self._pending_ids = np.concatenate([self._pending_ids, ids])
        self._pending_vecs = np.concatenate([self._pending_vecs, vecs])
        self._pending_dev = None

    def clear_pending(self) -> None:
        self._pending_ids = self._pending_ids[:0]
        self._pending_vecs = self._pending_vecs[:0]
        self._pending_dev = None

    def _merge_pending(self, Q, out, B: int, k: int) -> None:
        """Device buffer_scan + (distance, id) merge of the first k (lv_merge_pending)."""
        import torch
        if not len(self._pending_ids):
            return
        if self._pending_dev is None:
            self._pending_dev = (torch.from_numpy(self._pending_vecs).to(Q.device),
                                 torch.from_numpy(self._pending_ids).to(Q.device))
        pv, pi = self._pending_dev
        st = torch.cuda.current_stream(Q.device).cuda_stream
        _lib.check(_lib.lib().lv_merge_pending(
            _lib.LV_METRIC[self.metric], pv.data_ptr(), pi.data_ptr(), pv.shape[0], pv.shape[1],
            Q.data_ptr(), None, B, k, out["ids"].data_ptr(), out["dist"].data_ptr(),
            out["count"].data_ptr(), _lib.LV_IO_DEVICE, C.c_void_p(st)))

    def search(self, queries, top_k: int = 3, complexity: int = 64, recompute: bool = True,
               max_inflight: int = 0):
        """Batched search. Host input -> host numpy (ids [B, k], dists [B, k],
        counters [B, 4]); CUDA input -> fresh CUDA tensors (no host
        synchronisation; later calls never overwrite them). The query norm is
        computed on the device in numpy's np.dot order (lv_query_norms)."""
        import torch
        on_device = hasattr(queries, "data_ptr")
        Q = self.embed_queries(queries)
        params = self._params(top_k, complexity)
        if recompute:
            source = ProviderSource(self.provider)
        else:
            if self.matrix is None:
                raise InvalidArgumentError("recompute=False needs a resident embedding matrix")
            source = MatrixSource(self.matrix)
        out = self.device_index.search_device(Q, params, source, qn=None, cache=self.cache,
                                              max_inflight=max_inflight, out=self._out)
        self._out = out
        B = Q.shape[0]
        self._merge_pending(Q, out, B, top_k)
        if on_device:
            return out["ids"][:B].clone(), out["dist"][:B].clone(), out["counters"][:B].clone()
        ids = out["ids"][:B].cpu().numpy()
        dist = out["dist"][:B].cpu().numpy()
        counters = out["counters"][:B].cpu().numpy()
        torch.cuda.synchronize()
        return ids, dist, counters
