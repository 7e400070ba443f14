"""Warm BERT-base encode (n passages x 256 tokens) under GEMM kernel-variant switches
(lv_set_gemm_mode bits: 8 = kMode 5 for the short-K split-residual GEMM (O-projection),
4 = 2-buffer/4-stage variant for long-K residual GEMMs): passages/s and profiled GEMM time."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n = int(sys.argv[1])
modes = [int(x) for x in sys.argv[2].split(",")]
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
for rep in range(2):
    for m in modes:
        _lib.lib().lv_set_gemm_mode(m)
        enc.encode(tok)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3):
            enc.encode(tok)
        ev[1].record()
        torch.cuda.synchronize()
        pps = 3 * n / (ev[0].elapsed_time(ev[1]) / 1e3)
        print(f"mode {m}: {pps:.0f} passages/s", flush=True)
_lib.lib().lv_set_gemm_mode(0)
