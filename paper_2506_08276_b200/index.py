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

On-disk layout (same files the reference reads): ``graph.bin`` (LGR1),
``pq.bin`` (LPQ1), ``items.dat``/``items.idx`` (token store), ``meta.txt``.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

from .builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
from .encoder import EncoderProvider, GpuEncoder, TokenStore
from .errors import InvalidArgumentError
from .graph import load_graph, save_graph
from .pq import load_pq, save_pq
from .search import (MatrixSource, ProviderSource, SearchParams, build_embedding_cache,
                     device_index_for)


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
        if not hasattr(tokens, "data_ptr"):
            TokenStore(np.asarray(tokens)).save(d)
        (d / "meta.txt").write_text(
            f"n={graph.n}\ndim={E.shape[1]}\nmetric={params.metric}\n"
            f"provider=lv-encoder:{encoder.cfg.name}\n")
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
        self._out = None
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

    def search(self, queries, top_k: int = 3, complexity: int = 64, recompute: bool = True,
               max_inflight: int = 0):
        """Batched search. Host input -> host numpy (ids [B, k], dists [B, k],
        counters [B, 4]); CUDA input -> CUDA tensors (no host synchronisation)."""
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
        if on_device:
            return out["ids"][:B], out["dist"][:B], out["counters"][:B]
        ids = out["ids"][:B].cpu().numpy()
        dist = out["dist"][:B].cpu().numpy()
        counters = out["counters"][:B].cpu().numpy()
        torch.cuda.synchronize()
        return ids, dist, counters
