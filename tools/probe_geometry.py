"""Probe embedding geometry and graph quality on a subset of a bench config."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge; ge.build()
import paper_2506_08276_b200 as lv
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, synthetic_tokens
from paper_2506_08276_b200 import builder as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
name = sys.argv[2] if len(sys.argv) > 2 else "bert-base"
S = int(sys.argv[3]) if len(sys.argv) > 3 else 256
ecfg = ENCODERS[name]
enc = GpuEncoder(ecfg, init_weights(ecfg, 2), precision="bf16")
tok = torch.from_numpy(synthetic_tokens(n, S, ecfg.vocab, 0).view(np.int16)).cuda()
qt = torch.from_numpy(synthetic_tokens(1000, S, ecfg.vocab, 1).view(np.int16)).cuda()
E = enc.encode(tok); Q = enc.encode(qt); torch.cuda.synchronize()
mu = E.mean(0)
print("norm(mean)", float(mu.norm()))
sub = E[:2000]
c = sub @ sub.T
print("pairwise cos mean %.5f std %.5f min %.5f max(offdiag) %.5f" % (float(c.mean()), float(c.std()), float(c.min()), float((c - 2*torch.eye(2000, device=c.device)).max())))
gt = B.brute_force_topk(E, Q, 3, "cosine")
d = -(Q @ E.T)
top = d.topk(20, largest=False).values
print("query gaps: d1 %.6f d3 %.6f d20 %.6f" % tuple(float(top[:, i].mean()) for i in (0, 2, 19)))
# kNN candidate quality: bf16 raw vs centered vs fp32
x = E
ex_ids, _ = B._knn(x, 16, "cosine")  # current
torch.backends.cuda.matmul.allow_tf32 = False
sc = (x[:1000] @ x.T); sc[torch.arange(1000), torch.arange(1000)] = -9
exact = sc.topk(16).indices
ov = np.mean([len(set(a.tolist()) & set(b.tolist())) / 16 for a, b in zip(ex_ids[:1000].cpu(), exact.cpu())])
print("knn@16 overlap (bf16 raw cand) vs exact fp32: %.3f" % ov)
xc = (x - mu).to(torch.bfloat16)
sq = (xc.float() ** 2).sum(1)
scc = 2 * (xc[:1000] @ xc.T).float() - sq[None]
scc[torch.arange(1000), torch.arange(1000)] = -9
cc = scc.topk(24).indices
ov = np.mean([len(set(a[:16].tolist()) & set(b.tolist())) / 16 for a, b in zip(cc.cpu(), exact.cpu())])
ov2 = np.mean([len(set(a.tolist()) & set(b.tolist())) / 16 for a, b in zip(cc.cpu(), exact.cpu())])
print("knn@16 overlap (bf16 centered, top16 / top24 pool) vs exact: %.3f / %.3f" % (ov, ov2))
# graph + PQ + search recall in matrix mode
t = time.time()
g = B.build_graph_gpu(E, B.GpuBuildParams(max_degree=32))
model, codes = B.train_pq_gpu(E, int(sys.argv[4]) if len(sys.argv) > 4 else 64, "cosine")
torch.cuda.synchronize(); print("build %.1fs avg_deg %.2f levels %d" % (time.time() - t, g.out_degrees(0).mean(), g.level_count))
dev = lv.search.device_index_for(g, model, codes)
for alpha in (30.0, 100.0):
    for ef in (32, 64, 128, 256, 512):
        out = dev.search_device(Q, lv.SearchParams(k=3, ef=ef, rerank_percent=alpha), lv.MatrixSource(E))
        ids = out["ids"].cpu().numpy(); rc = out["counters"][:, 0].float().mean().item()
        print("alpha %.0f ef %d recall %.4f recomputes/q %.0f" % (alpha, ef, B.mean_recall(ids, gt), rc))
