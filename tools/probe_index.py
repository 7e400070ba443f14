"""Recall vs ef for corpus x builder x alpha variants (resident-matrix mode)."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge; ge.build()
import paper_2506_08276_b200 as lv
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens, synthetic_tokens
from paper_2506_08276_b200 import builder as B
n, name, S = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
ecfg = ENCODERS[name]
enc = GpuEncoder(ecfg, init_weights(ecfg, 2), precision="bf16")
corpora = {
    "uniform": (lambda m, sd: synthetic_tokens(m, S, ecfg.vocab, sd)),
    "lda32": (lambda m, sd: lda_tokens(m, S, ecfg.vocab, sd, 32, 0.05, background=0.05)),
}
for cname in sys.argv[4].split(","):
    gen = corpora[cname]
    E = enc.encode(torch.from_numpy(gen(n, 0).view(np.int16)).cuda())
    Q = enc.encode(torch.from_numpy(gen(300, 1).view(np.int16)).cuda())
    gt = B.brute_force_topk(E, Q, 3, "cosine")
    for spec in sys.argv[5].split(","):   # M/m/pqm
        M, m, pqm = (int(x) for x in spec.split("/"))
        t = time.time()
        g = B.build_graph_gpu(E, B.GpuBuildParams(max_degree=M, low_degree=m, candidates=max(64, 2 * M)))
        model, codes = B.train_pq_gpu(E, pqm, "cosine")
        dev = lv.search.device_index_for(g, model, codes)
        for alpha in (30.0, 100.0):
            res = []
            for ef in (32, 64, 128, 256, 512):
                out = dev.search_device(Q, lv.SearchParams(k=3, ef=ef, rerank_percent=alpha), lv.MatrixSource(E))
                res.append("%d:%.3f/%.0f" % (ef, B.mean_recall(out["ids"].cpu().numpy(), gt), out["counters"][:, 0].float().mean().item()))
            print(f"{cname} M={M} m={m} pq={pqm} deg={g.out_degrees(0).mean():.1f} a={alpha:.0f}", " ".join(res), flush=True)
