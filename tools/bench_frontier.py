"""Matrix-source frontier kernel A/B: the query's ADC table staged in shared
memory by one bulk copy (LV_SMEM_LUT) vs read from global memory per lookup
(default). Config-2-shape index (tests/golden/c2shape: 100k x 768,
M=32, PQ m=64), 4096 queries (the 512 fixture queries tiled, perturbed)."""
import json
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests/golden")
import __graft_entry__ as ge  # noqa: E402
ge.build()
import c2shape  # noqa: E402
import paper_2506_08276_b200 as lv  # noqa: E402

d = "/root/repo/tests/golden/c2shape/"
E, Q = c2shape.make()
g = lv.load_graph(d + "graph.bin")
model, codes = lv.load_pq(d + "pq.bin")
rng = np.random.default_rng(0)
Qb = np.tile(Q, (8, 1)) + 0.05 * rng.standard_normal((8 * Q.shape[0], Q.shape[1])).astype(np.float32)
dev = lv.search.device_index_for(g, model, codes)
Et, Qt = torch.from_numpy(E).cuda(), torch.from_numpy(Qb.astype(np.float32)).cuda()
out = {}
for ef in (64, 128):
    p = lv.SearchParams(k=3, ef=ef, rerank_percent=30.0)
    res = {}
    for name, kw in (("smem", dict(smem_lut=True)), ("global", {}),
                     ("hashset", dict(hash_visited=True))):
        dev.search_device(Qt, p, lv.MatrixSource(Et), **kw)   # warm
        torch.cuda.synchronize()
        r = dev.search_device(Qt, p, lv.MatrixSource(Et), **kw)
        st = dev.last_stats()
        res[name] = (r["ids"].cpu().numpy(), st)
    for name in res:
        assert (res[name][0] == res["global"][0]).all(), name
    for k, (_, st) in res.items():
        gbs = st["adc_bytes"] / (st["frontier_ms"] / 1e3) / 1e9
        out[f"ef{ef}_{k}"] = dict(ms=round(st["frontier_ms"], 3), algorithmic_GBps=round(gbs, 1),
                                  qps=round(Qt.shape[0] / (st["frontier_ms"] / 1e3), 1))
        print(f"ef={ef} {k:6s}: frontier {st['frontier_ms']:.2f} ms, {gbs:.0f} GB/s algorithmic, "
              f"{Qt.shape[0] / (st['frontier_ms'] / 1e3):.0f} QPS", flush=True)
print(json.dumps(out))
