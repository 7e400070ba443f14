"""One warm BERT-base encode of n passages x 256 tokens with the split (hi, lo)
residual stream on or off (ncu launch lists of the residual GEMM modes)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n, split = int(sys.argv[1]), int(sys.argv[2])
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
enc.set_split_residual(bool(split))
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
enc.encode(tok)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(3):
    enc.encode(tok)
ev[1].record()
torch.cuda.synchronize()
print(f"split={split}: {3 * n / (ev[0].elapsed_time(ev[1]) / 1e3):.0f} passages/s")
