"""Golden fixture for the fp32-encoder parity criterion (run in the build container).

Usage: python tests/golden/make_encoder_golden.py

1. Synthetic passages/queries (encoder.lda_tokens) and a seeded random-init
   4-layer d=256 encoder (encoder.init_weights).
2. Embeddings from the torch fp32 encoder oracle (oracle/encoder_ref.py).
3. Index built by the UNMODIFIED reference builder from those embeddings
   (the steps of build_index, builder.py:499-548, minus embed_items).
4. The reference's own run_search (search.py:434-443) with
   MatrixSource(embeddings) for every query; results and counters saved, with
   the reference's ground truth and recall (evaluation.py:82-118).

The GPU test (tests/test_gpu_encoder_parity.py) re-embeds the same token rows
with the GPU fp32 encoder inside the recompute path and must return the same
top-k id sets on >= 99% of queries with distances within 1e-5 relative
(BASELINE.json north_star, fp32 encoder mode). Nothing here runs on the GPU box.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from slimvec.builder import (BuildParams, assign_level, build_graph,  # noqa: E402
                             select_hubs, train_and_encode_pq)
from slimvec.graph import save_graph  # noqa: E402
from slimvec.pq import save_pq  # noqa: E402
from slimvec.evaluation import ground_truth, mean_recall  # noqa: E402
from slimvec.search import MatrixSource, SearchParams, run_search  # noqa: E402

from oracle.encoder_ref import RefEncoder  # noqa: E402
from paper_2506_08276_b200.encoder import EncoderConfig, init_weights, lda_tokens  # noqa: E402

OUT = Path(__file__).resolve().parent / "enc_fp32"
CFG = EncoderConfig("golden-4l-d256", 4, 256, 4, 1024, 30522, 128)
N, NQ, S, SEED = 2000, 1000, 64, 11
PARAMS = [dict(k=3, ef=32, rerank_percent=30.0), dict(k=3, ef=64, rerank_percent=100.0)]


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    tok = lda_tokens(N, S, CFG.vocab, seed=SEED, n_topics=16, alpha=0.1)
    qtok = lda_tokens(NQ, S, CFG.vocab, seed=SEED + 1, n_topics=16, alpha=0.1)
    ref = RefEncoder(CFG, init_weights(CFG, seed=SEED))
    E = ref.encode(tok)
    Q = ref.encode(qtok)
    bp = BuildParams(max_degree=32, metric="cosine", seed=0, pq_subspaces=16, ef_construction=64)
    level_of = lambda v: assign_level(v, bp.seed, bp.max_degree)  # noqa: E731
    pass1 = build_graph(E, bp, None, level_of)
    degrees = np.array([len(r) if r else 0 for r in pass1.base], dtype=np.int64)
    hub_mask = np.zeros(N, dtype=bool)
    hub_mask[select_hubs(degrees, bp.hub_percent, N)] = True
    graph = build_graph(E, bp, hub_mask, level_of).freeze()
    model, codes = train_and_encode_pq(E, bp)
    save_graph(graph, OUT / "graph.bin")
    save_pq(model, codes, OUT / "pq.bin")
    np.save(OUT / "tokens.npy", tok)
    np.save(OUT / "qtokens.npy", qtok)
    np.save(OUT / "embeddings_ref.npy", E)
    np.save(OUT / "queries_ref.npy", Q)
    gt = ground_truth(E, Q, 3, "cosine")   # evaluation.py:98-105
    cases = []
    for p in PARAMS:
        reps = []
        for q in Q:
            r = run_search(graph, q, SearchParams(**p), MatrixSource(E), "cosine", model, codes)
            reps.append(dict(ids=[int(i) for i, _ in r.results],
                             dist=[float(d) for _, d in r.results],
                             recomputations=r.recomputations, approx_lookups=r.approx_lookups))
        cases.append(dict(params=p, recall=mean_recall([r["ids"] for r in reps], gt),
                          reports=reps))
    meta = dict(encoder=CFG.__dict__, n=N, n_queries=NQ, seq_len=S, seed=SEED,
                ground_truth=gt.ids, cases=cases)
    (OUT / "reference_results.json").write_text(json.dumps(meta))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
