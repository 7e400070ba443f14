"""GPU builder and PQ encoder against the reference,
on the reference's standard fixture (evaluation.py:30-44: 10k x 32, M=16,
low 5, hub 8%, PQ m=8; tests/golden/standard, built by the unmodified
reference builder):

* build_graph_gpu on the same embeddings, searched with the reference's PQ
  at its published operating points (ef 120 / 50, rerank 30%): recall@3
  within 0.01 of the reference graph's and recomputations/query within 10%;
* the GPU file is a valid LGR1 (our validate mirrors graph.py:100-135; the
  reference's own load_graph/validate accepted the GPU-built config-2-shape
  graph when tests/golden/make_c2shape_golden.py ran);
* encode_pq_gpu with the reference's codebooks == pq_encode's codes
  (pq.py:114-136) except at near-ties (both centroid distances within 1e-5).
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
FIX = GOLDEN / "standard"


@pytest.fixture(scope="module")
def fx():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.evaluation import ground_truth
    E, Q = np.load(FIX / "matrix.npy"), np.load(FIX / "queries.npy")
    cases = json.loads((GOLDEN / "standard_cases.json").read_text())
    return dict(lv=lv, E=E, Q=Q, qn=np.load(FIX / "qn.npy"), cases=cases,
                g_ref=lv.load_graph(FIX / "graph.bin"), pq=lv.load_pq(FIX / "pq.bin"),
                gt=ground_truth(E, Q, 3, "cosine"))


def _recall(reps, gt):
    return float(np.mean([len({i for i, _ in r.results} & set(t)) / 3 for r, t in zip(reps, gt)]))


def test_gpu_graph_matches_reference_graph_quality(fx):
    import torch
    lv = fx["lv"]
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu
    g = build_graph_gpu(torch.from_numpy(fx["E"]).cuda(),
                        GpuBuildParams(max_degree=16, low_degree=5, hub_percent=8.0,
                                       metric="cosine", seed=42, candidates=64))
    lv.validate(g)
    model, codes = fx["pq"]
    for case in fx["cases"]:
        p = lv.SearchParams(**case["params"])
        ref_recall = float(np.mean([len(set(r["ids"]) & set(t)) / 3
                                    for r, t in zip(case["reports"], fx["gt"])]))
        ref_rec = float(np.mean([r["recomputations"] for r in case["reports"]]))
        reps = lv.search_batch(g, fx["Q"], p, lv.MatrixSource(fx["E"]), "cosine", model, codes,
                               qn=fx["qn"])
        got_recall = _recall(reps, fx["gt"])
        got_rec = float(np.mean([r.recomputations for r in reps]))
        print(f"{case['params']}: GPU graph recall@3 {got_recall:.3f} recomputes/q {got_rec:.1f}"
              f" | reference graph {ref_recall:.3f} / {ref_rec:.1f}")
        assert got_recall >= ref_recall - 0.01, (got_recall, ref_recall)
        assert abs(got_rec - ref_rec) <= 0.10 * ref_rec, (got_rec, ref_rec)


def test_encode_pq_gpu_matches_reference_codes(fx):
    from paper_2506_08276_b200.builder import encode_pq_gpu
    model, codes = fx["pq"]
    got = encode_pq_gpu(model, fx["E"]).codes
    ref = codes.codes
    bad = np.argwhere(got != ref)
    sub = model.padded_dim // model.m_pq
    x = np.zeros((fx["E"].shape[0], model.padded_dim), np.float64)
    x[:, :model.dim] = fx["E"]
    for r, s in bad:
        blk = x[r, s * sub:(s + 1) * sub]
        cb = model.codebooks[s].astype(np.float64)
        d = (cb * cb).sum(1) - 2.0 * cb @ blk
        a, b = d[got[r, s]], d[ref[r, s]]
        assert abs(a - b) <= 1e-5 * max(1.0, abs(b)), (r, s, a, b)
    print(f"{len(bad)} of {ref.size} codes differ, all near-ties")
    assert len(bad) <= 1e-3 * ref.size
