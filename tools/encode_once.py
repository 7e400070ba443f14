"""One warm BERT-base encode of n passages (fused LN on/off) for ncu launch lists."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n, fused = int(sys.argv[1]), int(sys.argv[2])
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
enc.set_fused_layernorm(bool(fused))
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
for _ in range(2):
    enc.encode(tok)
torch.cuda.synchronize()
