"""One warm BERT-base encoder forward over n passages (for an ncu launch list:
ncu --metrics gpu__time_duration.sum -s 86 -c 86 python tools/profile_encoder.py)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1300
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
for _ in range(2):
    enc.encode(tok)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
enc.encode(tok)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"encode {n} passages: {ms:.2f} ms, {n / ms * 1e3:.0f} passages/s, "
      f"{n * cfg.flops_per_passage(256) / ms / 1e9:.0f} TF/s effective")
