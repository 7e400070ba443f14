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

    This is a host BLAS ``sdot``; its order depends on the BLAS kernel the
    host selects. On this image's hosts (OpenBLAS SkylakeX kernel) it equals
    :func:`sdot_openblas`, which the device reproduces (``lv_query_norms``).
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


def _fma32(a, b, c):
    """float32 fused multiply-add, emulated in float64 (a*b is exact there; the
    one float64 rounding before the float32 one can only matter at an exact
    float32 midpoint, which the pinning test below never hit)."""
    return (np.float64(a) * np.float64(b) + np.float64(c)).astype(np.float32) \
        if np.ndim(a) == 0 else (a.astype(np.float64) * b.astype(np.float64)
                                 + c.astype(np.float64)).astype(np.float32)


def sdot_openblas(x: np.ndarray, y: np.ndarray) -> np.float32:
    """``np.dot`` of two float32 vectors as scipy-openblas 0.3.30's SkylakeX
    ``sdot`` kernel evaluates it (numpy hands 1-D float32 dots to cblas_sdot):
    n1 = n & -32; four 16-lane FMA accumulators over the n1 & -64 prefix, each
    folded to 8 lanes (lo + hi); four 8-lane FMA accumulators over the last
    32-block; ((a0 + a1) + a2) + a3; lanes l + l+4; (h0 + h1) + (h2 + h3); then
    the scalar tail ``dot += y[i] * x[i]`` (separately rounded). Pinned against
    np.dot for every n % 32 == 0 (tests/test_oracle_golden.py::test_sdot_order).
    This is what ``distance()`` (vectors.py:94-116) and every ``qn``
    (vectors.py:138, pq.py:163) compute on this image's hosts."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    n = x.shape[0]
    n1 = n & ~31
    dot = np.float32(0.0)
    i = 0
    if n1:
        n64 = n1 & ~63
        a5 = np.zeros((4, 16), np.float32)
        while i < n64:
            a5 = _fma32(x[i:i + 64].reshape(4, 16), y[i:i + 64].reshape(4, 16), a5)
            i += 64
        acc = (a5[:, :8] + a5[:, 8:]).astype(np.float32)
        while i < n1:
            acc = _fma32(x[i:i + 32].reshape(4, 8), y[i:i + 32].reshape(4, 8), acc)
            i += 32
        a = ((acc[0] + acc[1]) + acc[2]) + acc[3]
        h = (a[:4] + a[4:]).astype(np.float32)
        dot = np.float32(np.float32(h[0] + h[1]) + np.float32(h[2] + h[3]))
    while i < n:
        dot = np.float32(dot + np.float32(y[i] * x[i]))
        i += 1
    return dot


def distance(a: np.ndarray, b: np.ndarray, metric: str = "cosine") -> float:
    """vectors.py:94-116 with np.dot as :func:`sdot_openblas`."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    if metric == "l2":
        d = (a - b).astype(np.float32)
        return float(sdot_openblas(d, d))
    if metric == "ip":
        return float(-sdot_openblas(a, b))
    denom = float(np.sqrt(sdot_openblas(a, a))) * float(np.sqrt(sdot_openblas(b, b)))
    if denom == 0.0:
        raise ValueError("cosine distance undefined for zero vector")
    return float(np.float32(-sdot_openblas(a, b)) / np.float32(denom))
