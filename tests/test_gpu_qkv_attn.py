"""The fused QKV-projection + attention kernel (csrc/lv_qkv_attn.cu, one SM-pair
kernel per layer at S = 256, dh = 64) against the unfused path it replaces
(tcgen05 pair GEMM writing qkv to HBM + attn_tc_kernel): bit-identical encoder
outputs, batch invariance, and the torch fp32 oracle."""
from __future__ import annotations

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
