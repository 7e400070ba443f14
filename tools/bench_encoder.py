"""Sustained BERT-base encoder throughput (passages/s, effective TF/s) over
`reps` back-to-back forwards of n passages, with and without the fused
LayerNorm epilogues. CUDA events on the launching stream."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200.encoder import ENCODERS, GpuEncoder, init_weights, lda_tokens  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = ENCODERS["bert-base"]
enc = GpuEncoder(cfg, init_weights(cfg, 2), precision="bf16")
tok = torch.from_numpy(lda_tokens(n, 256, cfg.vocab, 0, 32, 0.05, background=0.05).view(np.int16)).cuda()
out = torch.empty(n, cfg.hidden, device="cuda")
for fused in (True, False, True):
    enc.set_fused_layernorm(fused)
    enc.encode(tok, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        enc.encode(tok, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"fused_ln={fused}: encode {n} passages: {ms:.1f} ms, {n / ms * 1e3:.0f} passages/s, "
          f"{n * cfg.flops_per_passage(256) / ms / 1e9:.0f} TF/s effective", flush=True)
