"""Recall oracle and ef tuning (reference ``evaluation.py:82-161``) on the device.

* :func:`brute_force_topk` / :func:`ground_truth` (evaluation.py:82-105): the k
  smallest ``(distance, id)`` over the active rows, with the distance bits of
  the reference's ``distance_many`` (numpy einsum order, ``lv_distance_gather``)
  and the ``np.lexsort((ids, d))`` tie order. An fp32 GEMM (tf32 off) nominates
  the ``k + candidates`` nearest rows per query; the exact re-rank then orders
  them bit-exactly. The only assumption is that the GEMM's rounding (~1e-6
  relative) never moves a true top-k row behind ``k + candidates`` others.
* :func:`recall_at_k`, :func:`mean_recall` (evaluation.py:108-118).
* :func:`tune_ef` (evaluation.py:132-161): the same memoised binary search,
  infeasible result and non-monotone warning; ``n`` is the caller's upper
  bound exactly as in the reference (its harness passes ``graph.n``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidArgumentError


def brute_force_topk(matrix, queries, k: int, metric: str = "cosine", active=None,
                     candidates: int = 32, chunk: int = 0) -> np.ndarray:
    """[B, k] int64 ids (-1 padded when fewer than k active rows), evaluation.py:82-95."""
    import torch
    _lib.require_device()
    E = matrix if hasattr(matrix, "data_ptr") else torch.from_numpy(
        np.ascontiguousarray(matrix, dtype=np.float32)).cuda()
    E = E.float().contiguous()
    Q = torch.as_tensor(queries, dtype=torch.float32, device=E.device).contiguous()
    if Q.ndim == 1:
        Q = Q.reshape(1, -1)
    n, dim = E.shape
    if Q.shape[1] != dim:
        raise InvalidArgumentError(f"dimension mismatch: {Q.shape[1]} vs {dim}")
    c = min(n, k + candidates)
    act = None if active is None else torch.as_tensor(np.asarray(active, dtype=bool),
                                                      device=E.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    out = np.full((Q.shape[0], k), -1, dtype=np.int64)
    chunk = chunk or max(16, min(1024, (1 << 31) // max(1, n)))   # <= 8 GB of scores
    st = torch.cuda.current_stream(E.device).cuda_stream
    try:
        rn = E.norm(dim=1) if metric == "cosine" else None
        sq = (E * E).sum(1) if metric == "l2" else None
        for s in range(0, Q.shape[0], chunk):
            q = Q[s:s + chunk]
            dots = q @ E.T
            if metric == "cosine":
                d = -(dots / (rn[None, :] * q.norm(dim=1, keepdim=True)))
            elif metric == "ip":
                d = -dots
            else:
                d = (q * q).sum(1, keepdim=True) + sq[None, :] - 2 * dots
            if act is not None:
                d[:, ~act] = float("inf")
            cand = d.topk(c, dim=1, largest=False).indices.contiguous()
            if act is not None:
                cand = torch.where(act[cand], cand, torch.full_like(cand, -1))
            exact = torch.empty(cand.shape, dtype=torch.float32, device=E.device)
            _lib.check(_lib.lib().lv_distance_gather(
                _lib.LV_METRIC[metric], E.data_ptr(), dim, cand.data_ptr(), q.shape[0], c,
                q.data_ptr(), None, exact.data_ptr(), st))
            ids = cand.cpu().numpy()
            ds = exact.cpu().numpy().astype(np.float64)
            for r in range(ids.shape[0]):
                order = np.lexsort((ids[r], ds[r]))[:k]
                keep = [int(ids[r, i]) for i in order if ids[r, i] >= 0]
                out[s + r, :len(keep)] = keep
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def ground_truth(matrix, queries, k: int, metric: str = "cosine", active=None) -> list:
    """evaluation.py:98-105 (ids per query; inactive rows excluded)."""
    return [[int(i) for i in row if i >= 0]
            for row in brute_force_topk(matrix, queries, k, metric, active)]


def recall_at_k(returned, truth) -> float:
    """evaluation.py:108-112: |returned ∩ truth| / k."""
    truth = [int(i) for i in truth]
    if not truth:
        raise InvalidArgumentError("recall undefined for k == 0")
    return len(set(int(i) for i in returned) & set(truth)) / len(truth)


def mean_recall(results, truth) -> float:
    """evaluation.py:115-118."""
    truth = getattr(truth, "ids", truth)
    return float(np.mean([recall_at_k(r, t) for r, t in zip(results, truth)]))


@dataclass
class TuneResult:
    """evaluation.py:124-129."""

    ef: int
    recall: float
    feasible: bool
    warning: str | None = None


def tune_ef(evaluate, k: int, n: int, target_recall: float) -> TuneResult:
    """Minimal ef whose mean recall meets the target (evaluation.py:132-161):
    memoised, infeasible at n, found endpoint re-checked one step below."""
    memo: dict[int, float] = {}

    def rec(ef: int) -> float:
        if ef not in memo:
            memo[ef] = evaluate(ef)
        return memo[ef]

    if rec(n) < target_recall:
        return TuneResult(ef=n, recall=rec(n), feasible=False)
    lo, hi = k, n
    while lo < hi:
        mid = (lo + hi) // 2
        if rec(mid) >= target_recall:
            hi = mid
        else:
            lo = mid + 1
    warning = None
    if lo > k and rec(lo - 1) >= target_recall:
        warning = (f"non-monotone recall near ef={lo}: ef-1 also meets the target;"
                   " widened by one step")
    return TuneResult(ef=lo, recall=rec(lo), feasible=True, warning=warning)
