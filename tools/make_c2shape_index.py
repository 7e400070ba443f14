"""GPU-built index for the config-2-shaped parity fixture (run on the B200 box):

    python tools/make_c2shape_index.py gpurun_out/c2shape

Regenerates the seeded 100k x 768 embeddings (tests/golden/c2shape.py),
builds the pruned graph (M=32, m=6, hub 2%) and PQ m=64 with the GPU builder
(paper_2506_08276_b200/builder.py), and writes graph.bin (LGR1), pq.bin (LPQ1).
tests/golden/make_c2shape_golden.py then runs the reference's run_search on
these files in the build container."""
from __future__ import annotations

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def main() -> None:
    import torch
    import __graft_entry__ as ge
    ge.build()
    import c2shape
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
    out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c2shape")
    out.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    E, _ = c2shape.make()
    Et = torch.from_numpy(E).cuda()
    g = build_graph_gpu(Et, GpuBuildParams(max_degree=32, hub_percent=2.0, metric="cosine",
                                           seed=0, pq_subspaces=64))
    model, codes = train_pq_gpu(Et, 64, "cosine", seed=0)
    lv.save_graph(g, out / "graph.bin")
    lv.save_pq(model, codes, out / "pq.bin")
    print(f"c2shape index: n={g.n} levels={g.level_count} "
          f"avg_deg={g.out_degrees(0).mean():.2f} in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
