"""Config-2-shaped embeddings for the search-parity fixture (shared by the
GPU index tool, the golden generator and the GPU test).

Search parity is stated "given identical embeddings" (BASELINE.json
north_star), so the C2-shape fixture regenerates its 100k x 768 float32
matrix from a seed on every machine instead of shipping 300 MB: PCG64
normals combined with element-wise float64 arithmetic only (no BLAS), then
one rounding to float32 — bit-identical on any host with this numpy. The
structure is a two-level topic mixture (64 topics, 4096 sub-topics, isotropic
noise) so the graph has neighbourhoods to find.
"""
from __future__ import annotations

import numpy as np

N, DIM, NQ, SEED = 100_000, 768, 512, 2506


def _mix(rng, n, topics, subs, sub_topic):
    s = rng.integers(0, subs.shape[0], n)
    noise = rng.standard_normal((n, DIM))
    x = topics[sub_topic[s]] + 0.8 * subs[s] + 0.55 * noise
    return x.astype(np.float32)


def make(n: int = N, nq: int = NQ, seed: int = SEED):
    """(E [n, 768] float32, Q [nq, 768] float32)."""
    rng = np.random.default_rng(seed)
    topics = rng.standard_normal((64, DIM))
    subs = rng.standard_normal((4096, DIM))
    sub_topic = rng.integers(0, 64, 4096)
    E = np.concatenate([_mix(rng, min(20_000, n - i), topics, subs, sub_topic)
                        for i in range(0, n, 20_000)])
    Q = _mix(np.random.default_rng(seed + 1), nq, topics, subs, sub_topic)
    return E, Q
