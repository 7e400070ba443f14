"""Multi-rank search with the real device path: two ranks share
cuda:0 (this run has one GPU per box; gloo carries the gather), each searches
its query shard with lv_search_batch (dist.sharded_search), and the gathered
ids, distance bits and counters must equal the single-rank search of the
whole batch — for the matrix source on a reference golden fixture and for the
recompute source (GPU encoder + shared recomputation)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(source_kind):
    import torch
    import sys
    sys.path.insert(0, str(ROOT))
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    if source_kind == "matrix":
        d = GOLDEN / "small_cos"
        g = lv.load_graph(d / "graph.bin")
        model, codes = lv.load_pq(d / "pq.bin")
        Q = torch.from_numpy(np.load(d / "queries.npy")).cuda()
        E = torch.from_numpy(np.load(d / "matrix.npy")).cuda()
        return lv, g, model, codes, Q, lv.MatrixSource(E)
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
    from paper_2506_08276_b200.encoder import (EncoderConfig, EncoderProvider, GpuEncoder,
                                               init_weights, lda_tokens)
    cfg = EncoderConfig("t-2l-d256", 2, 256, 4, 1024, 30522, 128)
    enc = GpuEncoder(cfg, init_weights(cfg, seed=3), precision="bf16")
    tok = lda_tokens(3000, 64, cfg.vocab, seed=4, n_topics=16, alpha=0.1)
    qtok = lda_tokens(101, 64, cfg.vocab, seed=5, n_topics=16, alpha=0.1)
    E = torch.from_numpy(enc.encode(tok)).cuda()
    g = build_graph_gpu(E, GpuBuildParams(max_degree=32, metric="cosine"))
    model, codes = train_pq_gpu(E, 16, "cosine")
    Q = torch.from_numpy(enc.encode(qtok)).cuda()
    tok_dev = torch.from_numpy(tok.view(np.int16)).cuda()
    return lv, g, model, codes, Q, lv.ProviderSource(EncoderProvider(enc, tok_dev))


def _run(source_kind, world, rank):
    from paper_2506_08276_b200.dist import sharded_search
    lv, g, model, codes, Q, src = _setup(source_kind)
    dev = lv.search.device_index_for(g, model, codes)
    p = lv.SearchParams(k=3, ef=40, rerank_percent=30.0)
    ids, dist, cnt = sharded_search(dev, Q, p, src)
    return ids.cpu().numpy(), dist.cpu().numpy(), cnt.cpu().numpy()


def _worker(rank, world, port, kind, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(kind, world, rank)
        if rank == 0:
            out_q.put(res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["matrix", "encoder"])
def test_two_ranks_gather_equals_single_rank(kind):
    import torch.multiprocessing as mp
    single = _run(kind, 1, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, dist, cnt = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(ids, single[0])
    assert np.array_equal(dist.view(np.uint32), single[1].view(np.uint32))
    assert np.array_equal(cnt[:, :2], single[2][:, :2])   # recomputations, approx_lookups
