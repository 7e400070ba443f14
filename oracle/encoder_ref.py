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


def _rms(x, g, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def _rotate_half(x):
    h = x.shape[-1] // 2
    return torch.cat((-x[..., h:], x[..., :h]), dim=-1)


class RefDecoderEncoder(torch.nn.Module):
    """fp32 CPU restatement of the decoder-style (arch 1, Qwen3-Embedding-
    shaped) encoder: pre-RMSNorm blocks, grouped-query causal attention with
    per-head q/k RMSNorm and rotate-half RoPE (inv_freq = theta^(-2i/dh)),
    SwiGLU MLP, final RMSNorm, last-token pooling, L2 normalisation."""

    def __init__(self, cfg, weights) -> None:
        super().__init__()
        self.cfg = cfg
        w = [_t(x) for x in weights]
        self.tok = w[0]
        self.layers = [w[1 + 9 * i: 10 + 9 * i] for i in range(cfg.layers)]
        self.final = w[-1]

    @torch.no_grad()
    def forward(self, tokens) -> torch.Tensor:
        cfg = self.cfg
        ids = torch.as_tensor(np.asarray(tokens, dtype=np.int64))
        n, S = ids.shape
        Hq = cfg.heads
        Hk = cfg.kv_heads or Hq
        dh = cfg.head_dim or cfg.hidden // Hq
        eps = cfg.norm_eps
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, dh, 2, dtype=torch.float32) / dh))
        ang = torch.arange(S, dtype=torch.float32)[:, None] * inv[None]
        cos = torch.cat((ang.cos(), ang.cos()), -1)
        sin = torch.cat((ang.sin(), ang.sin()), -1)
        mask = torch.full((S, S), float("-inf")).triu(1)
        x = self.tok[ids]
        for (g1, wqkv, qg, kg, wo, g2, wg, wu, wd) in self.layers:
            h = _rms(x, g1, eps)
            qkv = h @ wqkv.T
            q = qkv[..., :Hq * dh].view(n, S, Hq, dh)
            k = qkv[..., Hq * dh:(Hq + Hk) * dh].view(n, S, Hk, dh)
            v = qkv[..., (Hq + Hk) * dh:].view(n, S, Hk, dh)
            q, k = _rms(q, qg, eps), _rms(k, kg, eps)
            q = q * cos[None, :, None] + _rotate_half(q) * sin[None, :, None]
            k = k * cos[None, :, None] + _rotate_half(k) * sin[None, :, None]
            rep = Hq // Hk
            k = k.repeat_interleave(rep, dim=2)
            v = v.repeat_interleave(rep, dim=2)
            q, k, v = (t.transpose(1, 2) for t in (q, k, v))
            att = torch.softmax(q @ k.transpose(-1, -2) / math.sqrt(dh) + mask, dim=-1)
            ctx = (att @ v).transpose(1, 2).reshape(n, S, Hq * dh)
            x = x + ctx @ wo.T
            h = _rms(x, g2, eps)
            x = x + (torch.nn.functional.silu(h @ wg.T) * (h @ wu.T)) @ wd.T
        e = _rms(x[:, -1], self.final, eps)
        return e / e.norm(dim=-1, keepdim=True).clamp_min(1e-12)

    def encode(self, tokens, batch: int = 16) -> np.ndarray:
        tokens = np.asarray(tokens)
        outs = [self.forward(tokens[i:i + batch]).numpy() for i in range(0, len(tokens), batch)]
        return np.concatenate(outs, axis=0).astype(np.float32)


def make_ref_encoder(cfg, weights):
    """The fp32 oracle for either architecture."""
    return RefDecoderEncoder(cfg, weights) if getattr(cfg, "arch", 0) == 1 else RefEncoder(cfg, weights)


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
        self.enc = make_ref_encoder(cfg, weights)
        self.dt = np.dtype(token_dtype)
        self.config = SimpleNamespace(dim=cfg.hidden, max_batch=max_batch, kind="ref-encoder")

    def embed_batch(self, requests) -> np.ndarray:
        rows = np.stack([np.frombuffer(r.content, dtype=self.dt) for r in requests])
        return self.enc.encode(rows.astype(np.int64))
