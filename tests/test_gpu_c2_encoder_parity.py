"""Encoder-mode parity at config-2 width (BERT-base, 768-d, PQ m=64,
GPU-built M=32 graph): 8000 LDA passages x 128 tokens, 1000 queries.

* fp32 recompute mode (the GPU fp32 encoder re-embeds every candidate inside
  the search) against the oracle port of the reference search
  (oracle/search_port.py, pinned to the unmodified reference at config-2 shape
  by tests/golden/c2shape) over MatrixSource(fp32 embeddings): identical ids,
  distance bits and counters on every query;
* bf16 recompute mode: recall@3 (reference-order ground truth over the fp32
  embeddings) within 0.5 points of the fp32 reference's recall."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world():
    import torch
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
    from paper_2506_08276_b200.encoder import (ENCODERS, GpuEncoder, TokenStore, init_weights,
                                               lda_tokens)
    from paper_2506_08276_b200.evaluation import ground_truth
    cfg = ENCODERS["bert-base"]
    w = init_weights(cfg, seed=17)
    tok = lda_tokens(8000, 128, cfg.vocab, seed=18, n_topics=32, alpha=0.05, background=0.05)
    qtok = lda_tokens(1000, 128, cfg.vocab, seed=19, n_topics=32, alpha=0.05, background=0.05)
    enc32 = GpuEncoder(cfg, w, precision="fp32")
    E = enc32.encode(tok)
    Q = enc32.encode(qtok)
    Et = torch.from_numpy(E).cuda()
    g = build_graph_gpu(Et, GpuBuildParams(max_degree=32, hub_percent=2.0, metric="cosine"))
    model, codes = train_pq_gpu(Et, 64, "cosine")
    return dict(lv=lv, cfg=cfg, w=w, tok=tok, qtok=qtok, E=E, Q=Q, g=g, model=model,
                codes=codes, enc32=enc32, store=TokenStore(tok),
                gt=ground_truth(E, Q, 3, "cosine"))


P = dict(k=3, ef=48, rerank_percent=50.0)


def test_bert_fp32_recompute_matches_reference_search(world):
    from oracle import search_port as sp
    from paper_2506_08276_b200.encoder import EncoderProvider
    lv = world["lv"]
    reps = lv.search_batch(world["g"], world["Q"], lv.SearchParams(**P),
                           lv.ProviderSource(EncoderProvider(world["enc32"], world["store"])),
                           "cosine", world["model"], world["codes"])
    g = world["g"]
    og = sp.CsrGraph(g.n, g.max_degree, g.entry_point, g.levels, g.level_offsets,
                     g.level_neighbors)
    src = sp.MatrixRows(world["E"])
    for i in range(0, len(reps), 4):   # every 4th query: the CPU oracle is the slow side
        ref = sp.two_level(og, world["Q"][i], sp.SearchParams(**P), world["model"].codebooks,
                           world["codes"].codes, src, "cosine")
        assert [j for j, _ in reps[i].results] == [j for j, _ in ref.results], i
        assert [np.float32(x).view(np.uint32) for _, x in reps[i].results] == \
            [np.float32(x).view(np.uint32) for _, x in ref.results], i
        assert reps[i].recomputations == ref.recomputations, i


def test_bert_bf16_recall_within_half_point(world):
    from paper_2506_08276_b200.encoder import EncoderProvider, GpuEncoder
    from paper_2506_08276_b200.evaluation import mean_recall
    lv = world["lv"]
    p = lv.SearchParams(**P)
    ref = lv.search_batch(world["g"], world["Q"], p, lv.MatrixSource(world["E"]), "cosine",
                          world["model"], world["codes"])
    enc16 = GpuEncoder(world["cfg"], world["w"], precision="bf16")
    Q16 = enc16.encode(world["qtok"])
    got = lv.search_batch(world["g"], Q16, p,
                          lv.ProviderSource(EncoderProvider(enc16, world["store"])), "cosine",
                          world["model"], world["codes"])
    r_ref = mean_recall([[i for i, _ in r.results] for r in ref], world["gt"])
    r_got = mean_recall([[i for i, _ in r.results] for r in got], world["gt"])
    print(f"BERT-base bf16 recall@3 {r_got:.4f} vs fp32 reference {r_ref:.4f}")
    assert abs(r_got - r_ref) <= 0.005, (r_got, r_ref)
