"""Engine.search with a pending (buffered-add) buffer on the device, against
the UNMODIFIED reference Engine (fixture tests/golden/make_engine_golden.py):
two-level / best-first search in matrix mode, then lv_merge_pending —
ids and distance bits identical to the reference's merged reports
(index.py:320-327, update.py:483-488, vectors.py:94-116). Also the device
query norm (lv_query_norms, OpenBLAS sdot order) against host np.dot."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
FIX = GOLDEN / "engine_pending"


@pytest.fixture(scope="module")
def lv():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    return lv


@pytest.mark.parametrize("device_qn", [False, True])
def test_pending_merge_matches_reference_engine(lv, device_qn):
    meta = json.loads((FIX / "cases.json").read_text())
    g = lv.load_graph(FIX / "graph.bin")
    g.deleted = lv.load_deleted(FIX / "deleted.bin", g.n)
    model, codes = lv.load_pq(FIX / "pq.bin")
    E = np.load(FIX / "matrix.npy")
    Q = np.load(FIX / "queries.npy")
    pids, pvec = np.load(FIX / "pending_ids.npy"), np.load(FIX / "pending_vecs.npy")
    qn = lv.search.query_norms(Q)
    n_pending_hits = 0
    for case in meta["cases"]:
        p = lv.SearchParams(**case["params"])
        reps = lv.search_batch(g, Q, p, lv.MatrixSource(E), "cosine", model, codes, qn=qn)
        lv.merge_pending(reps, Q, pids, pvec, "cosine", p.k, qn=None if device_qn else qn)
        for rep, exp in zip(reps, case["reports"]):
            assert [i for i, _ in rep.results] == exp["ids"]
            assert [int(np.float32(d).view(np.uint32)) for _, d in rep.results] == exp["dist"]
            assert rep.recomputations == exp["recomputations"]
            n_pending_hits += any(i >= meta["n"] for i in exp["ids"])
    assert n_pending_hits > 20


def test_pending_merge_rejects_zero_cosine(lv):
    from paper_2506_08276_b200.errors import InvalidArgumentError
    reps = [lv.SearchReport(results=[(0, -0.5)])]
    with pytest.raises(InvalidArgumentError):
        lv.merge_pending(reps, np.ones((1, 32), np.float32), [7], np.zeros((1, 32), np.float32),
                         "cosine", 3)


@pytest.mark.parametrize("dim", [32, 256, 768, 1024])
def test_device_query_norms_match_host_np_dot(lv, dim):
    import torch
    rng = np.random.default_rng(dim)
    Q = rng.standard_normal((512, dim)).astype(np.float32)
    dev = lv.device_query_norms(torch.from_numpy(Q).cuda()).cpu().numpy()
    host = lv.search.query_norms(Q)
    assert (dev.view(np.uint32) == host.view(np.uint32)).all(), \
        f"{(dev != host).sum()} of 512 differ: the host BLAS is not the SkylakeX sdot kernel"
