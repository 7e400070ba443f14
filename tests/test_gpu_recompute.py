"""GPU parity of the recompute path: the two-level search with embeddings
recomputed by the GPU encoder (ProviderSource, search.py:96-110) against
(a) the same search over the resident matrix of those embeddings
(MatrixSource, search.py:78-93) — identical because the encoder is
batch-invariant — and (b) the CPU oracle restatement of the reference
(oracle/search_port.py) given identical embeddings: ID-for-ID, distance
bits, recompute and lookup counters."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world(tmp_path_factory):
    import torch
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
    from paper_2506_08276_b200.encoder import (EncoderConfig, GpuEncoder, TokenStore,
                                               init_weights, synthetic_tokens)
    out = {}
    cfg = EncoderConfig("t-2l-d256", 2, 256, 4, 1024, 30522, 128)
    w = init_weights(cfg, seed=7)
    tok = synthetic_tokens(2500, 64, cfg.vocab, seed=1)
    qtok = synthetic_tokens(96, 64, cfg.vocab, seed=2)
    for prec in ("fp32", "bf16"):
        enc = GpuEncoder(cfg, w, precision=prec)
        E = enc.encode(tok)
        Q = enc.encode(qtok)
        Et = torch.from_numpy(E).cuda()
        g = build_graph_gpu(Et, GpuBuildParams(max_degree=32, metric="cosine"))
        model, codes = train_pq_gpu(Et, 16, "cosine")
        d = tmp_path_factory.mktemp(prec)
        lv.save_graph(g, d / "graph.bin")
        lv.save_pq(model, codes, d / "pq.bin")
        out[prec] = dict(enc=enc, E=E, Q=Q, tok=tok, dir=d, store=TokenStore(tok))
    out["lv"] = lv
    return out


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("ef,alpha", [(16, 30.0), (48, 10.0), (64, 100.0)])
def test_recompute_equals_matrix_source(world, prec, ef, alpha):
    lv = world["lv"]
    from paper_2506_08276_b200.encoder import EncoderProvider
    w = world[prec]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    params = lv.SearchParams(k=3, ef=ef, rerank_percent=alpha)
    qn = lv.search.query_norms(w["Q"])
    rm = lv.search_batch(g, w["Q"], params, lv.MatrixSource(w["E"]), "cosine", model, codes, qn=qn)
    prov = EncoderProvider(w["enc"], w["store"])
    re = lv.search_batch(g, w["Q"], params, lv.ProviderSource(prov), "cosine", model, codes, qn=qn)
    for a, b in zip(rm, re):
        assert [i for i, _ in a.results] == [i for i, _ in b.results]
        assert [np.float32(x).view(np.uint32) for _, x in a.results] == \
               [np.float32(x).view(np.uint32) for _, x in b.results]
        assert a.recomputations == b.recomputations
        assert a.approx_lookups == b.approx_lookups


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_recompute_matches_oracle(world, prec):
    """Given identical embeddings the device search equals the reference's
    algorithm ID-for-ID (north_star: integer work bit-exact)."""
    lv = world["lv"]
    from oracle import search_port as sp
    from paper_2506_08276_b200.encoder import EncoderProvider
    w = world[prec]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    og = sp.read_lgr1(w["dir"] / "graph.bin")
    params = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    qn = lv.search.query_norms(w["Q"])
    reps = lv.search_batch(g, w["Q"], params, lv.ProviderSource(EncoderProvider(w["enc"], w["store"])),
                           "cosine", model, codes, qn=qn)
    for i, rep in enumerate(reps):
        ref = sp.two_level(og, w["Q"][i], sp.SearchParams(k=3, ef=32, rerank_percent=30.0),
                           model.codebooks, codes.codes, sp.MatrixRows(w["E"]), "cosine", qn=qn[i])
        assert [j for j, _ in rep.results] == [j for j, _ in ref.results], i
        assert [np.float32(x).view(np.uint32) for _, x in rep.results] == \
               [np.float32(x).view(np.uint32) for _, x in ref.results], i
        assert rep.recomputations == ref.recomputations, i
        assert rep.approx_lookups == ref.approx_lookups, i


def test_recompute_cache_transparent(world):
    """EmbeddingCache changes counters, never results (search.py:113-142)."""
    lv = world["lv"]
    from paper_2506_08276_b200.encoder import EncoderProvider
    w = world["bf16"]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    params = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    qn = lv.search.query_norms(w["Q"])
    src = lv.ProviderSource(EncoderProvider(w["enc"], w["store"]))
    plain = lv.search_batch(g, w["Q"], params, src, "cosine", model, codes, qn=qn)
    cache = lv.build_embedding_cache(g, 10.0)
    cached = lv.search_batch(g, w["Q"], params, src, "cosine", model, codes, qn=qn, cache=cache)
    hits = 0
    for a, b in zip(plain, cached):
        assert a.results == b.results
        assert a.recomputations == b.recomputations + b.cache_hits
        hits += b.cache_hits
    assert hits > 0


def test_device_io_search_and_device_qnorm(world):
    import torch
    lv = world["lv"]
    w = world["bf16"]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    params = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    qn = lv.search.query_norms(w["Q"])
    host = lv.search_batch(g, w["Q"], params, lv.MatrixSource(w["E"]), "cosine", model, codes, qn=qn)
    dev = lv.search.device_index_for(g, model, codes)
    Et = torch.from_numpy(w["E"]).cuda()
    out = dev.search_device(torch.from_numpy(w["Q"]).cuda(), params, lv.MatrixSource(Et),
                            qn=torch.from_numpy(qn).cuda())
    torch.cuda.synchronize()
    ids = out["ids"].cpu().numpy()
    for i, rep in enumerate(host):
        assert list(ids[i][:len(rep.results)]) == [j for j, _ in rep.results]
    # device-computed norms (lv_query_norms, np.dot's OpenBLAS sdot order):
    # the same ids and distance bits as the host-norm run on every query
    out2 = dev.search_device(torch.from_numpy(w["Q"]).cuda(), params, lv.MatrixSource(Et))
    torch.cuda.synchronize()
    assert (out2["ids"].cpu().numpy() == ids).all()
    assert (out2["dist"].cpu().numpy().view(np.uint32) ==
            out["dist"].cpu().numpy().view(np.uint32)).all()


def test_shared_recompute_is_transparent(world):
    """Sharing recomputations across in-flight queries changes only the physical
    encode count: ids, distance bits and the per-query (logical) counters are
    those of the unshared run."""
    lv = world["lv"]
    from paper_2506_08276_b200.encoder import EncoderProvider
    w = world["bf16"]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    params = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    qn = lv.search.query_norms(w["Q"])
    dev = lv.search.device_index_for(g, model, codes)
    src = lv.ProviderSource(EncoderProvider(w["enc"], w["store"]))
    a = dev.search(w["Q"], params, src, qn=qn, shared_recompute=False)
    phys_a = dev.last_stats()["physical_encodes"]
    b = dev.search(w["Q"], params, src, qn=qn, shared_recompute=True)
    phys_b = dev.last_stats()["physical_encodes"]
    for x, y in zip(a, b):
        assert x.results == y.results
        assert x.recomputations == y.recomputations
        assert x.approx_lookups == y.approx_lookups
    assert phys_a == sum(x.recomputations for x in a)
    assert phys_b < phys_a


def test_hash_visited_recompute_mode_matches_bitmaps(world):
    """Recompute (encoder) source with bounded hash visited sets == bitmaps."""
    import torch
    lv = world["lv"]
    from paper_2506_08276_b200.encoder import EncoderProvider
    w = world["bf16"]
    g = lv.load_graph(w["dir"] / "graph.bin")
    model, codes = lv.load_pq(w["dir"] / "pq.bin")
    dev = lv.search.device_index_for(g, model, codes)
    src = lv.ProviderSource(EncoderProvider(w["enc"], w["store"]))
    Q = torch.from_numpy(w["Q"]).cuda()
    p = lv.SearchParams(k=3, ef=48, rerank_percent=30.0)
    a = dev.search_device(Q, p, src)
    a = {k: v.clone() for k, v in a.items()}
    b = dev.search_device(Q, p, src, hash_visited=True)
    assert torch.equal(a["ids"], b["ids"]) and torch.equal(a["dist"], b["dist"])
    assert torch.equal(a["counters"], b["counters"])
