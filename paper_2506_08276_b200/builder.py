"""GPU index construction: LGR1 pruned graph + LPQ1 PQ artefacts from an embedding matrix.

Measurement infrastructure for the search hot path: the
reference builder (builder.py:499-548) inserts nodes one at a time in Python
and needs ~3.8 h at 1M nodes, so configs 2-5 cannot use it. This builder keeps
its structure and rules, batched on the GPU with PyTorch:

* levels: the reference's keyed geometric draw ``assign_level`` (builder.py:83-96);
  entry point = lowest id at the top level (the first such node the
  reference inserts);
* per level: the exact k nearest among that level's nodes with a SMALLER id
  (bf16 GEMM tiles, exact fp32 re-rank) in place of the HNSW
  ``_search_layer`` beam over the nodes inserted before (insertion is in id
  order, builder.py:404-422): early nodes get the long-range links that make
  the graph navigable. On the reference's standard fixture this graph
  searches like the reference's (recall@3 0.91 / 0.733 at 325 / 184
  recomputations per query at ef 120 / 50 against the reference graph's
  0.90 / 0.74 at 322 / 184; tests/test_gpu_builder_parity.py). Without the
  id-prefix restriction (all-pairs k-NN) recall fell to 0.82 / 0.66. Above
  ``exact_knn_max`` nodes the candidates come from an IVF search instead;
* relative-neighbourhood selection (``rng_shrink``, builder.py:99-118) of the
  candidates, then backlinks with shrink-to-M (``_Inserter.insert``,
  builder.py:367-402);
* two passes with hub preservation: pass 1 at the uniform cap M gives the
  degrees, ``select_hubs`` (builder.py:121-127) picks the top beta%, pass 2
  inserts hubs at cap M and everyone else at m = M // 5 (builder.py:499-548);
* PQ: per-subspace k-means++ (PCG64 seed + s) and fixed iterations on the
  first-100k sample, nearest-centroid codes (pq.py:79-136, cluster.py:15-64).

Search parity does not depend on this builder: both the reference search and
the device search read the same files it writes.
"""
from __future__ import annotations

import hashlib
import math
import struct
from dataclasses import dataclass

import numpy as np

from .graph import PrunedGraph
from .pq import PQCodes, PQModel, default_m_pq

_MAX_LEVEL = 24           # builder.py:36
_PQ_SAMPLE_CAP = 100_000  # builder.py:38


@dataclass
class GpuBuildParams:
    """builder.py:42-69 knobs used by the batched builder."""

    max_degree: int = 32
    low_degree: int | None = None
    hub_percent: float = 2.0
    metric: str = "cosine"
    seed: int = 0
    pq_subspaces: int | None = None
    pq_iters: int = 10
    candidates: int = 64      # k-NN pool per node (plays ef_construction's role)
    insertion_order: bool = True  # candidates among smaller ids only (HNSW insertion in id order)
    exact_knn_max: int = 2_000_000  # above: IVF approximate k-NN (_knn_ivf)

    def __post_init__(self) -> None:
        if self.low_degree is None:
            self.low_degree = max(1, self.max_degree // 5)


def assign_level(node_id: int, seed: int, max_degree: int) -> int:
    """Keyed geometric level draw, ratio 1/ln(M) (builder.py:83-96)."""
    key = struct.pack("<Q", seed & 0xFFFFFFFFFFFFFFFF)
    digest = hashlib.blake2b(b"level:%d" % node_id, digest_size=8, key=key).digest()
    (word,) = struct.unpack("<Q", digest)
    u = ((word >> 11) + 1) / float(2 ** 53)
    return min(int(-math.log(u) / math.log(max_degree)), _MAX_LEVEL)


def select_hubs(degrees: np.ndarray, hub_percent: float, n: int) -> np.ndarray:
    """Top ceil(beta*n/100) ids by (degree desc, id asc) (builder.py:121-127)."""
    count = min(n, math.ceil(hub_percent / 100.0 * n))
    order = np.lexsort((np.arange(n), -np.asarray(degrees, dtype=np.int64)))
    return np.sort(order[:count])


def _prep(x, metric):
    import torch
    x = x.float()
    if metric == "cosine":
        x = x / x.norm(dim=1, keepdim=True).clamp_min(1e-30)
    return x


def _pair_dist(a, b, metric):
    """Distances between matching rows (a, b: [..., d])."""
    if metric == "l2":
        d = a - b
        return (d * d).sum(-1)
    return -(a * b).sum(-1)


def _knn(x, k: int, metric: str, chunk: int = 0, prefix: bool = False):
    """Exact k nearest (excluding self) of every row of x among x: bf16 GEMM
    candidates (k + 16 of them), re-ranked with fp32 distances.

    Random-init encoders over uniform tokens give very concentrated embeddings
    (BERT-base: pairwise cosine 0.982 +- 0.002), far below bf16 resolution at
    |x.y| ~ 1. For cosine (unit rows) and l2 the candidates are therefore
    scored as L2 distances of mean-centred rows, which is translation
    invariant and keeps bf16's relative precision on the small residuals; ip
    is not translation invariant and is scored in fp32.

    prefix=True: the k nearest among the rows with a SMALLER id only (-1 /
    +inf padded) — the candidate set an HNSW-style insertion in id order
    (builder.py:404-422, exact search in place of ef_construction's beam)
    sees, which gives early nodes the long-range links that make the graph
    navigable."""
    import torch
    n = x.shape[0]
    kk = min(n - 1, k)
    extra = min(n - 1, kk + 16)
    if metric in ("cosine", "l2"):
        xc = x - x.mean(0, keepdim=True)
        xb = xc.to(torch.bfloat16)
        sq = (xb.float() ** 2).sum(1)
    else:
        xb, sq = x, None
    ids = torch.empty((n, kk), dtype=torch.int64, device=x.device)
    dist = torch.empty((n, kk), dtype=torch.float32, device=x.device)
    ar = torch.arange(n, device=x.device)
    chunk = chunk or max(256, min(2048, (1 << 31) // max(1, n)))  # <= 8 GB of scores
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        cols = e if prefix else n              # prefix: only ids below the chunk's end
        sc = (xb[s:e] @ xb[:cols].T).float()
        if sq is not None:
            sc = 2 * sc - sq[None, :cols]      # larger = closer
        sc[torch.arange(e - s, device=x.device), ar[s:e]] = -float("inf")
        if prefix:                             # ids >= the row's own id
            sc[:, s:e].masked_fill_(ar[None, s:e] >= ar[s:e, None], -float("inf"))
        cand = sc.topk(min(extra, cols), dim=1).indices
        if cand.shape[1] < extra:
            cand = torch.cat([cand, ar[s:e, None].expand(-1, extra - cand.shape[1])], 1)
        dd = _pair_dist(x[s:e, None, :], x[cand], metric)
        bad = cand == ar[s:e, None]
        if prefix:
            bad |= cand > ar[s:e, None]
        dd = torch.where(bad, torch.full_like(dd, float("inf")), dd)
        cand = torch.where(bad, torch.full_like(cand, -1), cand)
        # (distance, id) ascending
        order = torch.argsort(torch.where(cand < 0, n, cand), dim=1)
        cand = cand.gather(1, order)
        dd = dd.gather(1, order)
        order = torch.argsort(dd, dim=1, stable=True)
        ids[s:e] = cand.gather(1, order)[:, :kk]
        dist[s:e] = dd.gather(1, order)[:, :kk]
    return ids, dist


def _rerank(x, rows, cand, kk, metric):
    """Exact fp32 distances of candidate ids ``cand`` [b, c] to rows ``rows``
    [b] (self excluded), sorted by (distance, id); the first kk kept."""
    import torch
    dd = _pair_dist(x[rows][:, None, :], x[cand], metric)
    dd = torch.where(cand == rows[:, None], torch.full_like(dd, float("inf")), dd)
    order = torch.argsort(cand, dim=1)
    cand = cand.gather(1, order)
    dd = dd.gather(1, order)
    order = torch.argsort(dd, dim=1, stable=True)
    return cand.gather(1, order)[:, :kk], dd.gather(1, order)[:, :kk]


def _knn_ivf(x, k: int, metric: str, nlist: int = 0, nprobe: int = 8, sample: int = 262144,
             iters: int = 8, seed: int = 0):
    """Approximate k nearest of every row among x for corpora too large for the
    exact O(n^2) scan (config-3: 10M): k-means (nlist ~ sqrt(n) centroids, on
    a sample) over the mean-centred rows; every cluster's members search the
    members of the cluster's nprobe nearest centroids (bf16 GEMM candidates,
    exact fp32 re-rank as in _knn). Plays the role of the reference's
    approximate HNSW candidate search (builder.py:285-366)."""
    import torch
    n, dim = x.shape
    dev = x.device
    kk = min(n - 1, k)
    extra = kk + 16
    nlist = nlist or 1 << max(4, int(round(math.log2(math.sqrt(n)))))
    xc = x - x.mean(0, keepdim=True) if metric in ("cosine", "l2") else x
    xb = xc.to(torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(seed)
    samp = xc[torch.randperm(n, generator=g, device=dev)[:min(n, sample)]]
    cent = samp[:nlist].clone()

    def nearest(v, c, chunk=65536):
        cn = (c * c).sum(1)
        out = torch.empty(v.shape[0], dtype=torch.int64, device=dev)
        for s0 in range(0, v.shape[0], chunk):
            out[s0:s0 + chunk] = (cn[None, :] - 2.0 * (v[s0:s0 + chunk].float() @ c.T)).argmin(1)
        return out

    for _ in range(iters):
        a = nearest(samp, cent)
        sums = torch.zeros_like(cent).index_add_(0, a, samp)
        cnt = torch.bincount(a, minlength=nlist).float()
        cent = torch.where(cnt[:, None] > 0, sums / cnt.clamp_min(1)[:, None], cent)
    assign = nearest(xc, cent)
    order = torch.argsort(assign)
    counts = torch.bincount(assign, minlength=nlist)
    starts = torch.cumsum(counts, 0) - counts
    cc = (cent * cent).sum(1)
    probe = (cc[None, :] - 2.0 * cent @ cent.T).topk(min(nprobe, nlist), dim=1,
                                                     largest=False).indices
    sq = (xb.float() ** 2).sum(1) if metric in ("cosine", "l2") else None
    ids = torch.empty((n, kk), dtype=torch.int64, device=dev)
    dist = torch.empty((n, kk), dtype=torch.float32, device=dev)
    counts_h, starts_h, probe_h = counts.tolist(), starts.tolist(), probe.cpu().tolist()
    for c in range(nlist):
        if counts_h[c] == 0:
            continue
        q = order[starts_h[c]:starts_h[c] + counts_h[c]]
        cand = torch.cat([order[starts_h[p]:starts_h[p] + counts_h[p]] for p in probe_h[c]])
        for s0 in range(0, q.shape[0], 4096):
            qq = q[s0:s0 + 4096]
            sc = (xb[qq] @ xb[cand].T).float()
            if sq is not None:
                sc = 2 * sc - sq[cand][None, :]
            sc[cand[None, :] == qq[:, None]] = -float("inf")
            top = cand[sc.topk(min(extra, cand.shape[0]), dim=1).indices]
            if top.shape[1] < kk:  # tiny neighbourhood: pad with self (rejected later)
                top = torch.cat([top, qq[:, None].expand(-1, kk - top.shape[1])], 1)
            ii, dd = _rerank(x, qq, top, kk, metric)
            ids[qq], dist[qq] = ii, dd
    return ids, dist


def _rng_select(x, cand, cdist, caps, metric, chunk: int = 8192):
    """Relative-neighbourhood selection (rng_shrink, builder.py:99-118), batched:
    candidates per owner sorted ascending by (distance, id), -1 padded; keep c
    iff no kept k has dist(c, k) < dist(c, owner); stop at the owner's cap."""
    import torch
    B, R = cand.shape
    keep = torch.zeros((B, R), dtype=torch.bool, device=x.device)
    for s in range(0, B, chunk):
        e = min(B, s + chunk)
        c = cand[s:e]
        valid = c >= 0
        v = x[c.clamp_min(0)]                                  # [b, R, d]
        if metric == "l2":
            sq = (v * v).sum(-1)
            pair = sq[:, :, None] + sq[:, None, :] - 2 * torch.bmm(v, v.transpose(1, 2))
        else:
            pair = -torch.bmm(v, v.transpose(1, 2))
        d = cdist[s:e]
        cap = caps[s:e]
        kept = torch.zeros_like(valid)
        cnt = torch.zeros(e - s, dtype=torch.int32, device=x.device)
        for j in range(R):
            blocked = (kept & (pair[:, j, :] < d[:, j:j + 1])).any(1)
            take = valid[:, j] & ~blocked & (cnt < cap)
            kept[:, j] = take
            cnt += take.int()
        keep[s:e] = kept
    return keep


def _level_graph(x_all, members, caps_all, M, metric, k, knn=None, prefix=False):
    """One level: candidates -> RNG forward selection -> backlinks + shrink to M.
    Returns (offsets u64[n+1], neighbours u32[nnz]) over all n nodes."""
    import torch
    n = x_all.shape[0]
    dev = x_all.device
    nm = members.shape[0]
    if nm <= 1:
        return np.zeros(n + 1, dtype=np.uint64), np.zeros(0, dtype=np.uint32)
    x = x_all[members]
    lid, ldist = knn if knn is not None else _knn(x, k, metric, prefix=prefix)
    caps = caps_all[members]
    keep = _rng_select(x, lid, ldist, caps, metric)
    # forward edges (local ids) + backlinks
    own = torch.arange(nm, device=dev)[:, None].expand_as(lid)
    src = own[keep]
    dst = lid[keep]
    d = ldist[keep]
    osrc = torch.cat([src, dst])
    odst = torch.cat([dst, src])
    od = torch.cat([d, d])
    key = osrc * nm + odst
    key, inv = torch.unique(key, return_inverse=True)
    first = torch.full((key.shape[0],), -1, dtype=torch.int64, device=dev)
    first.scatter_reduce_(0, inv, torch.arange(inv.shape[0], device=dev), reduce="amin",
                          include_self=False)
    osrc, odst, od = osrc[first], odst[first], od[first]
    # sort by (owner, distance, id)
    order = torch.argsort(odst, stable=True)
    osrc, odst, od = osrc[order], odst[order], od[order]
    order = torch.argsort(od, stable=True)
    osrc, odst, od = osrc[order], odst[order], od[order]
    order = torch.argsort(osrc, stable=True)
    osrc, odst, od = osrc[order], odst[order], od[order]
    counts = torch.bincount(osrc, minlength=nm)
    starts = torch.cumsum(counts, 0) - counts
    rank = torch.arange(osrc.shape[0], device=dev) - starts[osrc]
    Rmax = 3 * M
    sel = rank < Rmax
    mat = torch.full((nm, Rmax), -1, dtype=torch.int64, device=dev)
    mdist = torch.full((nm, Rmax), float("inf"), device=dev)
    mat[osrc[sel], rank[sel]] = odst[sel]
    mdist[osrc[sel], rank[sel]] = od[sel]
    over = counts > M
    final = mat >= 0
    if bool(over.any()):
        rows = torch.nonzero(over).squeeze(1)
        kk = _rng_select(x, mat[rows], mdist[rows],
                         torch.full((rows.shape[0],), M, dtype=torch.int32, device=dev), metric)
        final[rows] = kk
    deg = final.sum(1)
    nb_local = mat[final]                      # row-major: grouped by owner, ascending distance
    nb = members[nb_local]
    deg_all = torch.zeros(n, dtype=torch.int64, device=dev)
    deg_all[members] = deg
    offs = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    offs[1:] = torch.cumsum(deg_all, 0)
    # owners in member order == ascending global id (members is sorted)
    return offs.cpu().numpy().astype(np.uint64), nb.cpu().numpy().astype(np.uint32)


def build_graph_gpu(matrix, params: GpuBuildParams) -> PrunedGraph:
    """Two-pass hub-preserving pruned graph over ``matrix`` (CUDA tensor [n, d])."""
    import torch
    n = matrix.shape[0]
    dev = matrix.device
    x = _prep(matrix, params.metric)
    M, m = params.max_degree, params.low_degree
    levels = np.array([assign_level(v, params.seed, M) for v in range(n)], dtype=np.uint16)
    top = int(levels.max())
    entry = int(np.flatnonzero(levels == top)[0])
    base = torch.arange(n, device=dev)
    full_caps = torch.full((n,), M, dtype=torch.int32, device=dev)
    # pass 1 (uniform cap) -> degrees -> hubs
    pre = params.insertion_order
    knn0 = (_knn(x, params.candidates, params.metric, prefix=pre) if n <= params.exact_knn_max
            else _knn_ivf(x, params.candidates, params.metric, seed=params.seed))
    offs1, _ = _level_graph(x, base, full_caps, M, params.metric, params.candidates, knn0)
    degrees = np.diff(offs1.astype(np.int64))
    hubs = select_hubs(degrees, params.hub_percent, n)
    caps = torch.full((n,), m, dtype=torch.int32, device=dev)
    caps[torch.from_numpy(hubs).to(dev)] = M
    offsets, neighbors = [], []
    for lvl in range(top + 1):
        if lvl == 0:
            o, nb = _level_graph(x, base, caps, M, params.metric, params.candidates, knn0)
        else:
            mem = torch.from_numpy(np.flatnonzero(levels >= lvl)).to(dev)
            o, nb = _level_graph(x, mem, full_caps, M, params.metric, params.candidates,
                                 prefix=pre)
        offsets.append(o)
        neighbors.append(nb)
    return PrunedGraph(n=n, max_degree=M, entry_point=entry, levels=levels,
                       level_offsets=offsets, level_neighbors=neighbors)


def _kmeanspp_init(x, k: int, seed: int):
    """cluster.py:48-64 on the GPU (one subspace)."""
    import torch
    rng = np.random.Generator(np.random.PCG64(seed))
    n = x.shape[0]
    cent = torch.empty((k, x.shape[1]), dtype=torch.float32, device=x.device)
    first = int(rng.integers(0, n))
    cent[0] = x[first]
    min_sq = ((x - cent[0]) ** 2).sum(1).double()
    for c in range(1, k):
        total = float(min_sq.sum())
        if total <= 0.0:
            cent[c:] = cent[c - 1]
            break
        target = rng.random() * total
        idx = int(torch.searchsorted(torch.cumsum(min_sq, 0), torch.tensor(
            [target], dtype=torch.float64, device=x.device)).item())
        idx = min(idx, n - 1)
        cent[c] = x[idx]
        torch.minimum(min_sq, ((x - cent[c]) ** 2).sum(1).double(), out=min_sq)
    return cent


def train_pq_gpu(matrix, m_pq: int | None, metric: str, iters: int = 10, seed: int = 0,
                 sample_cap: int = _PQ_SAMPLE_CAP):
    """pq_train + pq_encode (pq.py:79-136) batched over subspaces on the GPU."""
    import torch
    n, dim = matrix.shape
    m_pq = m_pq or default_m_pq(dim)
    padded = dim if dim % m_pq == 0 else dim + (m_pq - dim % m_pq)
    sub = padded // m_pq
    x = torch.zeros((n, padded), dtype=torch.float32, device=matrix.device)
    x[:, :dim] = matrix.float()
    sample = x[:min(n, sample_cap)]
    if sample.shape[0] < 256:
        reps = -(-256 // sample.shape[0])
        sample = sample.repeat(reps, 1)[:256]
    xs = sample.view(sample.shape[0], m_pq, sub).transpose(0, 1).contiguous()  # [m, Ns, sub]
    cbs = torch.stack([_kmeanspp_init(xs[s], 256, seed + s) for s in range(m_pq)])
    for _ in range(iters):
        cn = (cbs * cbs).sum(-1)                                   # [m, 256]
        assign = torch.argmin(cn[:, None, :] - 2.0 * torch.bmm(xs, cbs.transpose(1, 2)), dim=2)
        sums = torch.zeros_like(cbs, dtype=torch.float64)
        cnt = torch.zeros(cbs.shape[:2], dtype=torch.float64, device=x.device)
        sums.scatter_add_(1, assign[:, :, None].expand(-1, -1, sub), xs.double())
        cnt.scatter_add_(1, assign, torch.ones_like(assign, dtype=torch.float64))
        upd = (sums / cnt.clamp_min(1)[:, :, None]).float()
        cbs = torch.where(cnt[:, :, None] > 0, upd, cbs)
    model = PQModel(dim=dim, padded_dim=padded, m_pq=m_pq, metric=metric,
                    codebooks=cbs.cpu().numpy().astype(np.float32))
    return model, encode_pq_gpu(model, matrix)


def encode_pq_gpu(model: PQModel, matrix) -> PQCodes:
    """pq_encode (pq.py:114-136) on the GPU: per subspace the centroid minimising
    ||c||^2 - 2 x.c (fp32, tf32 off), lowest index on ties (argmin). The
    reference computes x.c with a BLAS sgemm whose summation order is the
    host's; codes agree except where two centroids tie to ~1e-6
    (tests/test_gpu_builder_parity.py)."""
    import torch
    x_in = matrix if hasattr(matrix, "data_ptr") else torch.from_numpy(
        np.ascontiguousarray(matrix, dtype=np.float32)).cuda()
    n, dim = x_in.shape
    m_pq, padded = model.m_pq, model.padded_dim
    sub = padded // m_pq
    cbs = torch.from_numpy(np.ascontiguousarray(model.codebooks, dtype=np.float32)).to(x_in.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        codes = torch.empty((n, m_pq), dtype=torch.uint8, device=x_in.device)
        cn = (cbs * cbs).sum(-1)
        for s0 in range(0, n, 65536):
            blk = torch.zeros((min(65536, n - s0), padded), dtype=torch.float32,
                              device=x_in.device)
            blk[:, :dim] = x_in[s0:s0 + 65536].float()
            blk = blk.view(-1, m_pq, sub).transpose(0, 1)
            d = cn[:, None, :] - 2.0 * torch.bmm(blk, cbs.transpose(1, 2))
            codes[s0:s0 + 65536] = torch.argmin(d, dim=2).transpose(0, 1).to(torch.uint8)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return PQCodes(codes=codes.cpu().numpy())


def brute_force_topk(matrix, queries, k: int, metric: str, deleted=None, chunk: int = 0):
    """evaluation.py:82-95 (exact reference order): see evaluation.brute_force_topk."""
    from .evaluation import brute_force_topk as bf
    active = None if deleted is None else ~np.asarray(deleted, dtype=bool)
    return bf(matrix, queries, k, metric, active=active, chunk=chunk)


def mean_recall(results, truth) -> float:
    """evaluation.py:108-118: |found ∩ truth| / k averaged over queries."""
    tot = 0.0
    for got, gt in zip(results, truth):
        tot += len(set(int(i) for i in got) & set(int(i) for i in gt)) / len(gt)
    return tot / len(truth)
