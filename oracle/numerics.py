"""TEST INFRASTRUCTURE ONLY. Bit-level restatement of the reference's float math.

The reference computes every distance with ``np.einsum`` in float32
(``vectors.py:120-140``, ``pq.py:175-177``) and every ADC sum with
``ndarray.sum(axis=1, dtype=np.float64)`` (``pq.py:186-189``). Neither is a
correctly rounded operation; both have a fixed evaluation order on numpy 2.3.5,
restated here so the CUDA kernels have an exact, platform-independent target:

* ``einsum_dot``: 4 float32 lanes; 16-element blocks accumulate the four
  4-wide sub-blocks in REVERSE order (12..15, 8..11, 4..7, 0..3); a tail of
  zero-padded 4-wide steps; final ``0 + ((l0 + l1) + (l2 + l3))``. No FMA.
  (re-pinned by ``tests/test_oracle_numerics.py``.)
* ``pairwise_sum64``: numpy's pairwise summation for n <= 128 — 8 strided
  float64 accumulators, ``((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7))``, then the
  remainder sequentially; n < 8 is a plain sequential sum from 0.0.
"""

from __future__ import annotations

import numpy as np

METRICS = ("l2", "ip", "cosine")  # vectors.py:19 (tag order = LPQ1 metric byte)


def einsum_dot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise dot in numpy-einsum order: ``einsum('ij,j->i')`` / ``('ij,ij->i')``."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    n, d = a.shape
    b = np.broadcast_to(np.asarray(b, dtype=np.float32), a.shape)
    acc = np.zeros((n, 4), dtype=np.float32)
    j = 0
    while d - j >= 16:
        for k in (3, 2, 1, 0):
            acc = acc + a[:, j + 4 * k:j + 4 * k + 4] * b[:, j + 4 * k:j + 4 * k + 4]
        j += 16
    while j < d:
        w = min(4, d - j)
        ta = np.zeros((n, 4), dtype=np.float32)
        tb = np.zeros((n, 4), dtype=np.float32)
        ta[:, :w] = a[:, j:j + w]
        tb[:, :w] = b[:, j:j + w]
        acc = acc + ta * tb
        j += 4
    return np.float32(0.0) + ((acc[:, 0] + acc[:, 1]) + (acc[:, 2] + acc[:, 3]))


def pairwise_sum64(x: np.ndarray) -> np.ndarray:
    """Row sums of a float64 (n, m) array in numpy's pairwise order (m <= 128)."""
    x = np.asarray(x, dtype=np.float64)
    n, m = x.shape
    if m < 8:
        res = np.zeros(n, dtype=np.float64)
        for i in range(m):
            res = res + x[:, i]
        return res
    if m > 128:
        half = (m // 2) - ((m // 2) % 8)
        return pairwise_sum64(x[:, :half]) + pairwise_sum64(x[:, half:])
    r = [x[:, i].copy() for i in range(8)]
    i = 8
    while i < m - (m % 8):
        for k in range(8):
            r[k] = r[k] + x[:, i + k]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < m:
        res = res + x[:, i]
        i += 1
    return res


def query_norm(q: np.ndarray) -> np.float32:
    """``np.float32(np.sqrt(np.dot(q, q)))`` exactly as ``vectors.py:138``/``pq.py:163``.

    This is a host BLAS ``sdot``; its order is CPU-dependent, so the B200 path
    takes this value from the host instead of recomputing it on the device.
    """
    q = np.asarray(q, dtype=np.float32)
    return np.float32(np.sqrt(np.dot(q, q)))


def distance_many(rows: np.ndarray, q: np.ndarray, metric: str = "cosine",
                  qn: np.float32 | None = None) -> np.ndarray:
    """Restates ``distance_many`` (vectors.py:120-140) with the pinned einsum order."""
    rows = np.asarray(rows, dtype=np.float32)
    q = np.asarray(q, dtype=np.float32)
    if rows.shape[1] != q.shape[0]:
        raise ValueError(f"dimension mismatch: {rows.shape[1]} vs {q.shape[0]}")
    if metric == "l2":
        d = rows - q
        return einsum_dot(d, d)
    if metric == "ip":
        return -einsum_dot(rows, q)
    if metric == "cosine":
        dots = einsum_dot(rows, q)
        row_norms = np.sqrt(einsum_dot(rows, rows))
        if qn is None:
            qn = query_norm(q)
        return -(dots / (row_norms * np.float32(qn)))
    raise ValueError(f"unknown metric: {metric!r}")


def adc_build(codebooks: np.ndarray, dim: int, metric: str, q: np.ndarray,
              qn: np.float32 | None = None) -> np.ndarray:
    """Restates ``adc_build`` (pq.py:153-178): (m, 256) float32 LUT."""
    m, kc, sub = codebooks.shape
    q = np.asarray(q, dtype=np.float32)
    if q.shape[0] != dim:
        raise ValueError(f"expected dim {dim}, got {q.shape[0]}")
    if metric == "cosine":
        norm = float(query_norm(q) if qn is None else qn)
        if norm == 0.0:
            raise ValueError("cosine ADC undefined for zero query")
        q = q / np.float32(norm)
    qp = np.zeros(m * sub, dtype=np.float32)
    qp[:dim] = q
    table = np.empty((m, kc), dtype=np.float32)
    for s in range(m):
        qs = qp[s * sub:(s + 1) * sub]
        cb = codebooks[s]
        if metric == "l2":
            d = cb - qs
            table[s] = einsum_dot(d, d)
        else:
            table[s] = -einsum_dot(cb, qs)
    return table


def approx_distance_many(table: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Restates ``approx_distance_many`` (pq.py:186-189): fp64 pairwise sum -> f32."""
    codes = np.asarray(codes, dtype=np.uint8)
    if codes.ndim == 1:
        codes = codes.reshape(1, -1)
    rows = np.arange(table.shape[0])
    gathered = table[rows[None, :], codes].astype(np.float64)
    return pairwise_sum64(gathered).astype(np.float32)
