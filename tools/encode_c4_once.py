"""Warm encodes of n config-4 (Qwen3-shaped) passages for ncu launch lists and
timing: python tools/encode_c4_once.py n [layers]."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200.encoder import ENCODERS, EncoderConfig, GpuEncoder, init_weights, synthetic_tokens  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
q = ENCODERS["qwen3-0.6b"]
L = int(sys.argv[2]) if len(sys.argv) > 2 else q.layers
cfg = EncoderConfig("qwen3-c4", L, q.hidden, q.heads, q.ffn, q.vocab, 512, arch=1,
                    kv_heads=q.kv_heads, head_dim=q.head_dim)
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
tok = torch.from_numpy(synthetic_tokens(n, 512, cfg.vocab, 0).view(np.int32)).cuda()
out = torch.empty(n, cfg.hidden, device="cuda")
for _ in range(2):
    enc.encode(tok, out=out)
torch.cuda.synchronize()
t0 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
enc.encode(tok, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"config-4 encoder ({L} layers): {n} passages in {ms:.1f} ms = {n / ms * 1e3:.0f} passages/s, "
      f"{n * cfg.flops_per_passage(512) / ms / 1e9:.0f} TF/s effective", flush=True)
