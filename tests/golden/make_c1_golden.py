"""Config-1 golden fixture from the UNMODIFIED reference (run in the build container).

Usage: python tests/golden/make_c1_golden.py        (~5 min on 8 cores)

BASELINE.json configs[0] at full size: 10k passages x 128 uniform tokens
(SURVEY 8(d)), the 4-layer d=256 random-init encoder, degree-32 pruned graph
(M=32, hub 2%, efC=64), PQ m=32, top-3, 1000 queries.

1. Embeddings of every passage and query from the torch fp32 encoder oracle
   (oracle/encoder_ref.py) — the fp32-mode "identical embeddings".
2. Index built by the reference builder from those embeddings (the steps of
   build_index, builder.py:499-548, minus embed_items).
3. The reference's run_search (search.py:434-443) with MatrixSource(E) for
   every query at each parameter case; results, distances and counters saved.
4. The reference's ground truth (brute_force_topk, evaluation.py:82-95) and
   mean_recall (evaluation.py:108-118) per case.

tests/test_gpu_c1_parity.py checks the device path against this fixture:
matrix mode bit-exact, fp32 recompute mode ID-for-ID on >= 99% of queries with
distances within 1e-5 relative, bf16 recompute mode recall within 0.5 points
(BASELINE.json north_star). Nothing here runs on the GPU box.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from slimvec.builder import (BuildParams, assign_level, build_graph,  # noqa: E402
                             select_hubs, train_and_encode_pq)
from slimvec.evaluation import ground_truth, mean_recall  # noqa: E402
from slimvec.graph import save_graph  # noqa: E402
from slimvec.pq import save_pq  # noqa: E402
from slimvec.search import MatrixSource, SearchParams, run_search  # noqa: E402

from oracle.encoder_ref import RefEncoder  # noqa: E402
from paper_2506_08276_b200.encoder import ENCODERS, init_weights, synthetic_tokens  # noqa: E402

OUT = Path(__file__).resolve().parent / "c1"
CFG = ENCODERS["c1-4l-d256"]
N, NQ, S, SEED = 10_000, 1000, 128, 101
PARAMS = [dict(k=3, ef=128, rerank_percent=30.0), dict(k=3, ef=64, rerank_percent=30.0),
          dict(k=3, ef=48, rerank_percent=100.0)]


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    tok = synthetic_tokens(N, S, CFG.vocab, seed=SEED)
    qtok = synthetic_tokens(NQ, S, CFG.vocab, seed=SEED + 1)
    ref = RefEncoder(CFG, init_weights(CFG, seed=SEED + 2))
    E = np.concatenate([ref.encode(tok[i:i + 500]) for i in range(0, N, 500)])
    Q = ref.encode(qtok)
    print(f"embedded in {time.time() - t0:.0f}s", flush=True)
    bp = BuildParams(max_degree=32, metric="cosine", seed=0, pq_subspaces=32, ef_construction=64)
    level_of = lambda v: assign_level(v, bp.seed, bp.max_degree)  # noqa: E731
    pass1 = build_graph(E, bp, None, level_of)
    degrees = np.array([len(r) if r else 0 for r in pass1.base], dtype=np.int64)
    hub_mask = np.zeros(N, dtype=bool)
    hub_mask[select_hubs(degrees, bp.hub_percent, N)] = True
    graph = build_graph(E, bp, hub_mask, level_of).freeze()
    model, codes = train_and_encode_pq(E, bp)
    print(f"built in {time.time() - t0:.0f}s", flush=True)
    save_graph(graph, OUT / "graph.bin")
    save_pq(model, codes, OUT / "pq.bin")
    np.save(OUT / "tokens.npy", tok)
    np.save(OUT / "qtokens.npy", qtok)
    np.save(OUT / "embeddings_ref.npy", E)
    np.save(OUT / "queries_ref.npy", Q)
    gt = ground_truth(E, Q, 3, "cosine")
    cases = []
    for p in PARAMS:
        reps = []
        for q in Q:
            r = run_search(graph, q, SearchParams(**p), MatrixSource(E), "cosine", model, codes)
            reps.append(dict(ids=[int(i) for i, _ in r.results],
                             dist=[float(d) for _, d in r.results],
                             recomputations=r.recomputations, approx_lookups=r.approx_lookups))
        rec = mean_recall([r["ids"] for r in reps], gt)
        cases.append(dict(params=p, recall=rec, reports=reps))
        print(f"{p}: recall@3 {rec:.4f}, recomputes/q "
              f"{np.mean([r['recomputations'] for r in reps]):.1f} ({time.time() - t0:.0f}s)",
              flush=True)
    meta = dict(encoder=CFG.__dict__, weight_seed=SEED + 2, n=N, n_queries=NQ, seq_len=S,
                seed=SEED, ground_truth=gt.ids, cases=cases,
                note="tokens: synthetic_tokens(N, S, vocab, SEED) / (NQ, ..., SEED + 1)")
    (OUT / "reference_results.json").write_text(json.dumps(meta))
    print("wrote", OUT, f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
