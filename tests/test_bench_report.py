"""CPU checks of bench.py's report arithmetic: the L2 -> shared-memory operand-feed
figures attached to the encoder rooflines (algorithmic bytes of the tcgen05 kernels'
TMA loads), which profiles/r02_l2feed.csv pins against ncu's
l1tex__m_xbar2l1tex_read_bytes."""
from __future__ import annotations

import importlib.util
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Bert:
    hidden, heads = 768, 12


def test_gemm_l2_feed_is_one_byte_per_128_flop():
    b = _bench()
    flops = 2.0 * 524288 * 3072 * 768          # FFN1 of one 512K-token chunk
    r = b.gemm_l2_feed({"gemm_flops": flops, "gemm_ms": 2.037344})
    # ncu measured 19.41 GB of TMA loads for this launch (profiles/r02_l2feed.csv)
    assert abs(r["bytes"] - 19.41e9) / 19.41e9 < 0.01
    assert abs(r["achieved_TBps"] - 9.49) < 0.02
    assert b.L2_FEED_CAP_TBS >= 9.9
    assert abs(r["frac_of_cap"] - r["achieved_TBps"] / b.L2_FEED_CAP_TBS) < 2e-3
    assert b.gemm_l2_feed({"gemm_flops": 1.0, "gemm_ms": 0.0}) is None


def test_fused_l2_feed_counts_x_and_weight_rows_per_item():
    b = _bench()
    S, d, H = 256, 768, 12
    per_seq_layer = 2.0 * S * 3 * d * d + 4.0 * S * S * d
    est = {"fused_flops": per_seq_layer * 2048, "fused_ms": 1.802592}   # one layer, 2048 seqs
    r = b.fused_l2_feed(est, _Bert, S)
    items = 2048 * H
    assert r["bytes"] == items * 2 * (128 + 96) * d * 2
    # ncu: 17.33 GB for this launch; the model counts the TMA loads only (2.5% below)
    assert 0.95 < r["bytes"] / 17.33e9 < 1.0
