"""Config-2-shaped search-parity golden from the UNMODIFIED reference (build container).

Usage: python tools/make_c2shape_index.py gpurun_out/c2shape   (on the B200 box)
       cp gpurun_out/c2shape/{graph,pq}.bin tests/golden/c2shape/
       python tests/golden/make_c2shape_golden.py                 (here, ~10 min)

* Embeddings: the seeded 100k x 768 matrix of tests/golden/c2shape.py
  (BERT-base width; regenerated bit-identically on any host).
* Index: built by the GPU builder (M=32, m=6, hub 2%, PQ m=64 — config-2's
  graph and PQ shape), loaded here by the reference's own load_graph /
  load_pq, whose validate() must accept the GPU files.
* The reference's run_search (search.py:434-443) with MatrixSource(E) for 256
  queries at two parameter cases; ids, distances, counters saved, with the
  reference's ground truth / recall (evaluation.py:82-118).
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import c2shape  # noqa: E402
from slimvec.evaluation import ground_truth, mean_recall  # noqa: E402
from slimvec.graph import load_graph  # noqa: E402
from slimvec.pq import load_pq  # noqa: E402
from slimvec.search import MatrixSource, SearchParams, run_search  # noqa: E402

OUT = HERE / "c2shape"
NQ = 256
PARAMS = [dict(k=3, ef=64, rerank_percent=30.0), dict(k=10, ef=96, rerank_percent=70.0)]


def main() -> None:
    t0 = time.time()
    E, Q = c2shape.make()
    Q = Q[:NQ]
    graph = load_graph(OUT / "graph.bin")       # runs the reference's validate()
    model, codes = load_pq(OUT / "pq.bin")
    print(f"loaded (reference validate passed) in {time.time() - t0:.0f}s", flush=True)
    gt3 = ground_truth(E, Q, 3, "cosine")
    gt10 = ground_truth(E, Q, 10, "cosine")
    cases = []
    for p in PARAMS:
        reps = []
        for q in Q:
            r = run_search(graph, q, SearchParams(**p), MatrixSource(E), "cosine", model, codes)
            reps.append(dict(ids=[int(i) for i, _ in r.results],
                             dist=np.asarray([d for _, d in r.results],
                                             dtype=np.float32).view(np.uint32).tolist(),
                             recomputations=r.recomputations, approx_lookups=r.approx_lookups))
        gt = gt3 if p["k"] == 3 else gt10
        rec = mean_recall([r["ids"] for r in reps], gt)
        cases.append(dict(params=p, recall=rec, reports=reps))
        print(f"{p}: recall@{p['k']} {rec:.4f} recomputes/q "
              f"{np.mean([r['recomputations'] for r in reps]):.0f} ({time.time() - t0:.0f}s)",
              flush=True)
    meta = dict(n=int(E.shape[0]), dim=int(E.shape[1]), n_queries=NQ, seed=c2shape.SEED,
                ground_truth_3=gt3.ids, ground_truth_10=gt10.ids, cases=cases)
    (OUT / "reference_results.json").write_text(json.dumps(meta))
    print("wrote", OUT, f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
