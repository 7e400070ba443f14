"""TEST INFRASTRUCTURE — torch fp32 CPU reference of the passage encoder.

The reference has no neural encoder (its providers are a BLAKE2b hash,
vectors.py:168-189, or a socket service, vectors.py:214-297), so the encoder
boundary is "parity unpinned" by the reference itself. This
module is the checker the GPU encoder is compared against: a plain PyTorch
fp32 restatement of the architecture documented in
paper_2506_08276_b200/csrc/lv_encoder.cu (BERT-style post-LN, erf-GELU,
mean-pool + L2 normalise) using the same weight list
(paper_2506_08276_b200.encoder.init_weights order).

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline may import it.
"""
from __future__ import annotations

import math

import numpy as np
import torch

LN_EPS = 1e-12


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))


class RefEncoder(torch.nn.Module):
    """fp32 CPU encoder over the C-ABI weight list (no grad)."""

    def __init__(self, cfg, weights) -> None:
        super().__init__()
        self.cfg = cfg
        w = [_t(x) for x in weights]
        self.tok, self.pos, self.eg, self.eb = w[:4]
        self.layers = [w[4 + 12 * i: 16 + 12 * i] for i in range(cfg.layers)]

    @torch.no_grad()
    def forward(self, tokens) -> torch.Tensor:
        cfg = self.cfg
        ids = torch.as_tensor(np.asarray(tokens, dtype=np.int64))
        n, S = ids.shape
        d, H = cfg.hidden, cfg.heads
        dh = d // H
        x = self.tok[ids] + self.pos[:S][None]
        x = torch.nn.functional.layer_norm(x, (d,), self.eg, self.eb, LN_EPS)
        for (wqkv, bqkv, wo, bo, g1, b1, w1, bb1, w2, bb2, g2, b2) in self.layers:
            qkv = x @ wqkv.T + bqkv
            q, k, v = qkv.split(d, dim=-1)
            q = q.view(n, S, H, dh).transpose(1, 2)
            k = k.view(n, S, H, dh).transpose(1, 2)
            v = v.view(n, S, H, dh).transpose(1, 2)
            att = torch.softmax((q @ k.transpose(-1, -2)) / math.sqrt(dh), dim=-1)
            ctx = (att @ v).transpose(1, 2).reshape(n, S, d)
            x = torch.nn.functional.layer_norm(ctx @ wo.T + bo + x, (d,), g1, b1, LN_EPS)
            hdn = torch.nn.functional.gelu(x @ w1.T + bb1)  # erf form
            x = torch.nn.functional.layer_norm(hdn @ w2.T + bb2 + x, (d,), g2, b2, LN_EPS)
        pooled = x.mean(dim=1)
        return pooled / pooled.norm(dim=-1, keepdim=True).clamp_min(1e-12)

    def encode(self, tokens, batch: int = 256) -> np.ndarray:
        tokens = np.asarray(tokens)
        outs = [self.forward(tokens[i:i + batch]).numpy() for i in range(0, len(tokens), batch)]
        return np.concatenate(outs, axis=0).astype(np.float32)


class RefProvider:
    """Duck-typed provider (vectors.py:201-211) over RefEncoder: decodes each
    request's payload as little-endian token ids. Used to drive the reference's
    own two_level_search as the CPU baseline."""

    def __init__(self, cfg, weights, token_dtype="<u2", max_batch: int = 1 << 20) -> None:
        from types import SimpleNamespace
        self.enc = RefEncoder(cfg, weights)
        self.dt = np.dtype(token_dtype)
        self.config = SimpleNamespace(dim=cfg.hidden, max_batch=max_batch, kind="ref-encoder")

    def embed_batch(self, requests) -> np.ndarray:
        rows = np.stack([np.frombuffer(r.content, dtype=self.dt) for r in requests])
        return self.enc.encode(rows.astype(np.int64))
