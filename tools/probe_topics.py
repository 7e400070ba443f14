"""Calibrate the topic-structured corpus: recall@3 vs ef in resident-matrix mode."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge; ge.build()
import paper_2506_08276_b200 as lv
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, topic_tokens, lda_tokens
from paper_2506_08276_b200 import builder as B
n, name, S, pqm = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
ecfg = ENCODERS[name]
enc = GpuEncoder(ecfg, init_weights(ecfg, 2), precision="bf16")
for spec in sys.argv[5:]:
    K, a, bgf = spec.split(":")
    K, a, bgf = int(K), float(a), float(bgf)
    per, frac, T = K, a, K
    tok = torch.from_numpy(lda_tokens(n, S, ecfg.vocab, 0, K, a, background=bgf).view(np.int16)).cuda()
    qt = torch.from_numpy(lda_tokens(500, S, ecfg.vocab, 1, K, a, background=bgf).view(np.int16)).cuda()
    E = enc.encode(tok); Q = enc.encode(qt)
    gt = B.brute_force_topk(E, Q, 3, "cosine")
    c = E[:2000] @ E[:2000].T
    g = B.build_graph_gpu(E, B.GpuBuildParams(max_degree=32))
    model, codes = B.train_pq_gpu(E, pqm, "cosine")
    dev = lv.search.device_index_for(g, model, codes)
    res = []
    for ef in (32, 64, 128, 256, 512, 1024):
        out = dev.search_device(Q, lv.SearchParams(k=3, ef=ef, rerank_percent=30.0), lv.MatrixSource(E))
        res.append("ef%d:%.3f/%.0f" % (ef, B.mean_recall(out["ids"].cpu().numpy(), gt), out["counters"][:, 0].float().mean().item()))
    print(f"per_topic={per} frac={frac} T={T} cos={float(c.mean()):.4f}+-{float(c.std()):.4f} deg={g.out_degrees(0).mean():.1f}", " ".join(res), flush=True)
