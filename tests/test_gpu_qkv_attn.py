"""The fused QKV-projection + attention kernel (csrc/lv_qkv_attn.cu, one SM-pair
kernel per layer at S = 256, dh = 64) against the unfused path it replaces
(tcgen05 pair GEMM writing qkv to HBM + attn_tc_kernel): bit-identical encoder
outputs, batch invariance, and the torch fp32 oracle."""
from __future__ import annotations

import pathlib
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lv():
    import __graft_entry__ as ge
    ge.build()
    import paper_2506_08276_b200 as mod
    return mod


def _encode(enc, tok, fused: bool):
    from paper_2506_08276_b200 import _lib
    prev = _lib.lib().lv_set_fused_qkv_attention(1 if fused else 0)
    try:
        return enc.encode(tok)
    finally:
        _lib.lib().lv_set_fused_qkv_attention(prev)


def _cfg(name):
    from paper_2506_08276_b200.encoder import ENCODERS, EncoderConfig
    if name == "d256":
        return EncoderConfig("test-2l-d256-s256", 2, 256, 4, 1024, 30522, 256)
    if name == "bert-2l":
        b = ENCODERS["bert-base"]
        return EncoderConfig("bert-base-2l", 2, b.hidden, b.heads, b.ffn, b.vocab, b.max_seq)
    return ENCODERS["bert-base"]


@pytest.mark.parametrize("name,n", [("d256", 1), ("d256", 37), ("bert-2l", 3), ("bert-2l", 29),
                                    ("bert-base", 13), ("d256", 600), ("bert-2l", 700)])
def test_fused_qkv_attention_bit_identical_to_unfused(lv, name, n):
    from paper_2506_08276_b200.encoder import GpuEncoder, init_weights, synthetic_tokens
    cfg = _cfg(name)
    enc = GpuEncoder(cfg, init_weights(cfg, seed=41), precision="bf16")
    tok = synthetic_tokens(n, 256, cfg.vocab, seed=42 + n)
    enc.profile(True)
    enc.reset_stats()
    fused = _encode(enc, tok, True)
    st = enc.stats()
    assert st["fused_launches"] == cfg.layers, st
    assert st["attn_launches"] == 0, st
    plain = _encode(enc, tok, False)
    assert np.isfinite(fused).all()
    diff = np.abs(fused - plain).max()
    assert np.array_equal(fused, plain), diff


def test_fused_qkv_attention_batch_invariant(lv):
    """Large launches run sequence-major (a pair owns whole sequences), small ones deal
    (sequence, head) items round-robin: the split below mixes both."""
    from paper_2506_08276_b200.encoder import GpuEncoder, init_weights, synthetic_tokens
    cfg = _cfg("bert-2l")
    enc = GpuEncoder(cfg, init_weights(cfg, seed=5), precision="bf16")
    tok = synthetic_tokens(700, 256, cfg.vocab, seed=6)
    whole = _encode(enc, tok, True)
    parts = np.concatenate([_encode(enc, tok[:1], True), _encode(enc, tok[1:40], True),
                            _encode(enc, tok[40:], True)])
    assert np.array_equal(whole, parts)


def test_fused_qkv_attention_close_to_fp32_oracle(lv):
    from oracle.encoder_ref import RefEncoder
    from paper_2506_08276_b200.encoder import GpuEncoder, init_weights, synthetic_tokens
    cfg = _cfg("bert-2l")
    w = init_weights(cfg, seed=11)
    tok = synthetic_tokens(6, 256, cfg.vocab, seed=12)
    got = _encode(GpuEncoder(cfg, w, precision="bf16"), tok, True)
    ref = RefEncoder(cfg, w).encode(tok)
    cos = (got * ref).sum(1) / np.linalg.norm(got, axis=1) / np.linalg.norm(ref, axis=1)
    assert cos.min() > 0.995, cos.min()


def test_fused_recompute_search_equals_unfused_matrix_and_oracle(lv):
    """The recompute path at S = 256 (fused QKV + attention inside the device search loop,
    shared recomputation) returns the same ids, distance bits and counters as a
    resident matrix of embeddings computed with the fusion switched OFF, and as the
    reference's algorithm (oracle port) over that matrix."""
    import torch
    from oracle import search_port as sp
    from paper_2506_08276_b200 import _lib
    from paper_2506_08276_b200.builder import GpuBuildParams, build_graph_gpu, train_pq_gpu
    from paper_2506_08276_b200.encoder import (EncoderProvider, GpuEncoder, TokenStore,
                                               init_weights, lda_tokens)
    cfg = _cfg("d256")
    enc = GpuEncoder(cfg, init_weights(cfg, seed=9), precision="bf16")
    tok = lda_tokens(1500, 256, cfg.vocab, 3, 16, 0.05, background=0.05)
    qtok = lda_tokens(48, 256, cfg.vocab, 4, 16, 0.05, background=0.05)
    E = _encode(enc, tok, False)
    Q = _encode(enc, qtok, False)
    Et = torch.from_numpy(E).cuda()
    g = build_graph_gpu(Et, GpuBuildParams(max_degree=24, metric="cosine"))
    model, codes = train_pq_gpu(Et, 16, "cosine")
    params = lv.SearchParams(k=3, ef=32, rerank_percent=30.0)
    qn = lv.search.query_norms(Q)
    rm = lv.search_batch(g, Q, params, lv.MatrixSource(E), "cosine", model, codes, qn=qn)
    prev = _lib.lib().lv_set_fused_qkv_attention(1)
    try:
        enc.profile(True)
        enc.reset_stats()
        re = lv.search_batch(g, Q, params, lv.ProviderSource(EncoderProvider(enc, TokenStore(tok))),
                             "cosine", model, codes, qn=qn)
        assert enc.stats()["fused_launches"] > 0
    finally:
        _lib.lib().lv_set_fused_qkv_attention(prev)
    with tempfile.TemporaryDirectory() as td:
        lv.save_graph(g, pathlib.Path(td) / "graph.bin")
        og = sp.read_lgr1(pathlib.Path(td) / "graph.bin")
    for i, (a, b) in enumerate(zip(rm, re)):
        assert [j for j, _ in a.results] == [j for j, _ in b.results], i
        assert [np.float32(x).view(np.uint32) for _, x in a.results] == \
               [np.float32(x).view(np.uint32) for _, x in b.results], i
        assert a.recomputations == b.recomputations and a.approx_lookups == b.approx_lookups, i
        ref = sp.two_level(og, Q[i], sp.SearchParams(k=3, ef=32, rerank_percent=30.0),
                           model.codebooks, codes.codes, sp.MatrixRows(E), "cosine", qn=qn[i])
        assert [j for j, _ in b.results] == [j for j, _ in ref.results], i
        assert b.recomputations == ref.recomputations, i
