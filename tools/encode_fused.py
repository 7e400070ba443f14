"""Warm BERT-base encode of n passages x 256 tokens with the fused QKV + attention
kernel on or off: passages/s and the profiled per-kernel split (fused / GEMM / attention)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n, fused, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
_lib.lib().lv_set_fused_qkv_attention(fused)
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
enc.encode(tok)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    enc.encode(tok)
ev[1].record()
torch.cuda.synchronize()
pps = reps * n / (ev[0].elapsed_time(ev[1]) / 1e3)
enc.profile(True)
enc.reset_stats()
enc.encode(tok)
st = enc.stats()
tot = st["gemm_ms"] + st["attn_ms"] + st["fused_ms"]
print(f"fused={fused}: {pps:.0f} passages/s | gemm {st['gemm_ms']:.2f} ms "
      f"({st['gemm_flops'] / st['gemm_ms'] / 1e9:.0f} TF/s) attn {st['attn_ms']:.2f} ms "
      f"fused {st['fused_ms']:.2f} ms"
      + (f" ({st['fused_flops'] / st['fused_ms'] / 1e9:.0f} TF/s)" if st['fused_ms'] else "")
      + f" | profiled total {tot:.2f} ms")
