"""North-star parity at BASELINE.json configs[0] (config-1, full size) against
the UNMODIFIED reference (tests/golden/make_c1_golden.py: 10k passages x 128
uniform tokens, 4-layer d=256 encoder, reference builder M=32, PQ m=32, the
reference's run_search over the torch-fp32 embeddings, 1000 queries, 3
parameter cases):

* matrix mode on the reference's embeddings: ids, distance bits and counters
  identical on every query — with host np.dot query norms and with the device
  norms (lv_query_norms);
* fp32 encoder mode (every candidate re-embedded by the GPU fp32 encoder from
  its token row inside the search): top-k id sets identical on >= 99% of
  queries, every returned id's distance within 1e-5 relative of the
  reference's distance for that id;
* bf16 encoder mode (tcgen05 encoder): recall@3 against the reference's
  brute-force ground truth within 0.5 points of the reference's recall.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
FIX = GOLDEN / "c1"


@pytest.fixture(scope="module")
def fx():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.encoder import EncoderConfig
    meta = json.loads((FIX / "reference_results.json").read_text())
    return dict(lv=lv, meta=meta, cfg=EncoderConfig(**meta["encoder"]),
                g=lv.load_graph(FIX / "graph.bin"), pq=lv.load_pq(FIX / "pq.bin"),
                tok=np.load(FIX / "tokens.npy"), qtok=np.load(FIX / "qtokens.npy"),
                E=np.load(FIX / "embeddings_ref.npy"), Q=np.load(FIX / "queries_ref.npy"))


def _bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def _recall(results, gt):
    return float(np.mean([len(set(r) & set(t)) / len(t) for r, t in zip(results, gt)]))


def test_c1_matrix_mode_bit_exact(fx):
    lv = fx["lv"]
    model, codes = fx["pq"]
    qn = lv.search.query_norms(fx["Q"])
    for case in fx["meta"]["cases"]:
        reps = lv.search_batch(fx["g"], fx["Q"], lv.SearchParams(**case["params"]),
                               lv.MatrixSource(fx["E"]), "cosine", model, codes, qn=qn)
        for rep, exp in zip(reps, case["reports"]):
            assert [i for i, _ in rep.results] == exp["ids"]
            assert list(_bits([d for _, d in rep.results])) == list(_bits(exp["dist"]))
            assert rep.recomputations == exp["recomputations"]
            assert rep.approx_lookups == exp["approx_lookups"]


def test_c1_matrix_mode_device_norms_bit_exact(fx):
    import torch
    lv = fx["lv"]
    model, codes = fx["pq"]
    dev = lv.search.device_index_for(fx["g"], model, codes)
    Et = torch.from_numpy(fx["E"]).cuda()
    for case in fx["meta"]["cases"]:
        out = dev.search_device(torch.from_numpy(fx["Q"]).cuda(), lv.SearchParams(**case["params"]),
                                lv.MatrixSource(Et), qn=None)
        ids = out["ids"].cpu().numpy()
        dist = out["dist"].cpu().numpy()
        cnt = out["counters"].cpu().numpy()
        for b, exp in enumerate(case["reports"]):
            assert list(ids[b]) == exp["ids"]
            assert list(_bits(dist[b])) == list(_bits(exp["dist"]))
            assert cnt[b, 0] == exp["recomputations"] and cnt[b, 1] == exp["approx_lookups"]


def _encoder_runs(fx, precision):
    lv = fx["lv"]
    from paper_2506_08276_b200.encoder import (EncoderProvider, GpuEncoder, TokenStore,
                                               init_weights)
    enc = GpuEncoder(fx["cfg"], init_weights(fx["cfg"], seed=fx["meta"]["weight_seed"]),
                     precision=precision)
    Qg = enc.encode(fx["qtok"])
    src = lv.ProviderSource(EncoderProvider(enc, TokenStore(fx["tok"])))
    model, codes = fx["pq"]
    out = []
    for case in fx["meta"]["cases"]:
        reps = lv.search_batch(fx["g"], Qg, lv.SearchParams(**case["params"]), src, "cosine",
                               model, codes)
        out.append((case, reps))
    return out


def test_c1_fp32_encoder_mode_matches_reference(fx):
    for case, reps in _encoder_runs(fx, "fp32"):
        same = 0
        for rep, exp in zip(reps, case["reports"]):
            got = dict(rep.results)
            same += set(got) == set(exp["ids"])
            for i, d in zip(exp["ids"], exp["dist"]):   # every shared id, any order
                if i in got:
                    assert abs(got[i] - d) <= 1e-5 * abs(d), (case["params"], i, got[i], d)
        frac = same / len(reps)
        print(f"fp32 {case['params']}: identical top-k sets on {frac:.4f} of queries")
        assert frac >= 0.99, (case["params"], frac)


def test_c1_bf16_encoder_mode_recall_within_half_point(fx):
    gt = fx["meta"]["ground_truth"]
    for case, reps in _encoder_runs(fx, "bf16"):
        got = _recall([[i for i, _ in r.results] for r in reps], gt)
        print(f"bf16 {case['params']}: recall@3 {got:.4f} vs reference {case['recall']:.4f}")
        assert abs(got - case["recall"]) <= 0.005, (case["params"], got, case["recall"])


def test_c1_ground_truth_matches_reference(fx):
    """brute_force_topk / ground_truth (evaluation.py:82-105) on the device ==
    the reference's ids for all 1000 queries (einsum-order distances + lexsort)."""
    from paper_2506_08276_b200.evaluation import ground_truth
    assert ground_truth(fx["E"], fx["Q"], 3, "cosine") == fx["meta"]["ground_truth"]
