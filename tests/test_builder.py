"""CPU checks of the measurement-infrastructure builder."""
from __future__ import annotations

import numpy as np


def test_ivf_knn_matches_exact_knn_on_clustered_data():
    """The approximate k-NN used above GpuBuildParams.exact_knn_max (config-3,
    10M passages) finds the exact neighbours on clustered data."""
    import torch
    from paper_2506_08276_b200.builder import _knn, _knn_ivf, _prep
    g = torch.Generator().manual_seed(0)
    n, d = 6000, 48
    centers = torch.randn(30, d, generator=g)
    x = centers[torch.randint(0, 30, (n,), generator=g)] + 0.3 * torch.randn(n, d, generator=g)
    x = _prep(x, "cosine")
    exact, _ = _knn(x, 12, "cosine")
    approx, dist = _knn_ivf(x, 12, "cosine", nlist=32, nprobe=6, sample=3000)
    recall = np.mean([len(set(a.tolist()) & set(b.tolist())) / 12 for a, b in zip(approx, exact)])
    assert recall > 0.95, recall
    assert bool((approx != torch.arange(n)[:, None]).all())       # never self
    assert bool((dist[:, 1:] >= dist[:, :-1]).all())               # ascending distance
