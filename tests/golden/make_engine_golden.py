"""Engine-level golden fixture from the UNMODIFIED reference: a pending
(buffered-add) buffer merged into search results (run in the build container).

Usage: python tests/golden/make_engine_golden.py

1. ItemStore.create + build_index_dir (index.py:173-213) with the reference's
   synthetic provider (dim 32, 1500 items, M=16).
2. Engine.open, then Engine.add(..., buffered=True) of 40 items: they are
   embedded and held in MutableIndex.buffer (update.py:459-481), not inserted.
3. Engine.search(q_ndarray, SearchParams) (index.py:305-328) for 80 queries —
   half are perturbed copies of pending vectors, so pending items enter the
   top-k through the merge (index.py:320-327, buffer_scan update.py:483-488).
   Two modes (two_level, exact_bestfirst), two k.
4. Saved: graph/pq/deleted files, the provider matrix of the base items, the
   pending ids + vectors, the queries and every report's results and counters.

tests/test_gpu_engine_merge.py replays this on the device (matrix source, then
lv_merge_pending) and compares ids and distance bits.
"""
from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from slimvec.builder import BuildParams  # noqa: E402
from slimvec.index import Engine, build_index_dir  # noqa: E402
from slimvec.search import SearchParams  # noqa: E402
from slimvec.store import ItemStore  # noqa: E402
from slimvec.vectors import EmbeddingRequest, ProviderConfig, embed_all, make_provider  # noqa

OUT = Path(__file__).resolve().parent / "engine_pending"
N, DIM, NP, NQ = 1500, 32, 40, 80
CASES = [dict(k=3, ef=32, rerank_percent=30.0), dict(k=10, ef=48, rerank_percent=60.0),
         dict(k=5, ef=40, mode="exact_bestfirst")]


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    tmp = Path(tempfile.mkdtemp())
    ix = tmp / "index"
    ItemStore.create(ix, [b"passage %d" % i for i in range(N)]).close()
    config = ProviderConfig(kind="synthetic", dim=DIM, seed=5, max_batch=64)
    build_index_dir(ix, BuildParams(ef_construction=32, max_degree=16, seed=3), config)
    provider = make_provider(config)
    matrix = embed_all([EmbeddingRequest(i, b"passage %d" % i) for i in range(N)], provider)
    engine = Engine.open(ix, config)
    new = [b"buffered %d" % j for j in range(NP)]
    ids = engine.add(new, buffered=True)
    pending = engine.mutable.buffer.pending
    pids = np.array([nid for nid, _, _ in pending], dtype=np.int64)
    pvec = np.stack([vec for _, _, vec in pending]).astype(np.float32)
    assert list(pids) == list(ids)
    rng = np.random.default_rng(9)
    Q = rng.standard_normal((NQ, DIM)).astype(np.float32)
    Q[: NQ // 2] = pvec[rng.integers(0, NP, NQ // 2)] + 0.05 * Q[: NQ // 2]
    cases = []
    for c in CASES:
        reps = []
        for q in Q:
            r = engine.search(q, SearchParams(**c))
            reps.append(dict(ids=[int(i) for i, _ in r.results],
                             dist=np.asarray([d for _, d in r.results],
                                             dtype=np.float32).view(np.uint32).tolist(),
                             recomputations=r.recomputations, approx_lookups=r.approx_lookups))
        cases.append(dict(params=c, reports=reps))
    engine.close()
    for name in ("graph.bin", "pq.bin", "deleted.bin", "meta.txt"):
        shutil.copy(ix / name, OUT / name)
    np.save(OUT / "matrix.npy", matrix)
    np.save(OUT / "pending_ids.npy", pids)
    np.save(OUT / "pending_vecs.npy", pvec)
    np.save(OUT / "queries.npy", Q)
    (OUT / "cases.json").write_text(json.dumps(dict(n=N, dim=DIM, cases=cases)))
    shutil.rmtree(tmp)
    hits = sum(any(i >= N for i in r["ids"]) for c in cases for r in c["reports"])
    print("wrote", OUT, f"({hits} reports contain pending items)")


if __name__ == "__main__":
    main()
