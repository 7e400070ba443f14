"""Passage encoder behind the recompute source, and the token store it reads.

The reference's provider boundary is ``provider.embed_batch(list[EmbeddingRequest])
-> f32[n, dim]`` (vectors.py:33-38, 201-211), reached through
``ProviderSource.fetch`` (search.py:96-110). Its providers are a hash
(vectors.py:168-189) or a socket service (vectors.py:214-297); neither is a
neural encoder. Here the payload of node ``i`` is row ``i`` of a token store
(packed little-endian u16/u32 ids, one fixed-length chunk per passage; the
``items.dat``/``items.idx`` layout of store.py:1-116 is kept so the
reference's ``ItemStore`` opens it) and the provider is a random-init
BERT-style encoder running in ``libleann_b200.so`` (lv_encoder_create /
lv_encode): bf16 tcgen05 GEMMs in the default mode, fp32 SIMT kernels in
parity mode. Both modes are batch-invariant (test_vectors.py:145-152).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import InvalidArgumentError

ITEMS_DAT = "items.dat"
ITEMS_IDX = "items.idx"


@dataclass(frozen=True)
class EncoderConfig:
    """Encoder shape. arch 0: BERT-style (post-LN, erf-GELU, mean-pool + L2;
    configs 1-3). arch 1: decoder-style, Qwen3-Embedding-shaped (pre-RMSNorm,
    grouped-query attention with per-head q/k RMSNorm and RoPE, causal,
    SwiGLU, final RMSNorm, last-token pool + L2; config 4)."""

    name: str
    layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    max_seq: int
    arch: int = 0
    kv_heads: int = 0       # arch 1 (0 = heads)
    head_dim: int = 0       # arch 1 (0 = hidden / heads)
    rope_theta: float = 1e6
    norm_eps: float = 1e-6

    @property
    def dim(self) -> int:
        return self.hidden

    @property
    def n_weights(self) -> int:
        return 4 + 12 * self.layers if self.arch == 0 else 2 + 9 * self.layers

    def flops_per_passage(self, seq_len: int) -> float:
        """Algorithmic FLOPs of one passage: GEMMs + attention
        matmuls; causal attention counted at half."""
        d, f, S = self.hidden, self.ffn, seq_len
        if self.arch == 0:
            return float(self.layers * (2 * S * (4 * d * d + 2 * d * f) + 4 * S * S * d))
        dh = self.head_dim or d // self.heads
        dq, dkv = self.heads * dh, (self.kv_heads or self.heads) * dh
        return float(self.layers * (2 * S * (d * 2 * dq + 2 * d * dkv + 3 * d * f) + 2 * S * S * dq))


ENCODERS = {
    # config-1: 4 layers, d=256, 4 heads, FFN 1024
    "c1-4l-d256": EncoderConfig("c1-4l-d256", 4, 256, 4, 1024, 30522, 512),
    # configs 2/3: BERT-base / Contriever-shaped
    "bert-base": EncoderConfig("bert-base", 12, 768, 12, 3072, 30522, 512),
    # config 4: Qwen3-Embedding-0.6B-shaped (28 layers, 1024 hidden, 16 q / 8 kv
    # heads x 128, SwiGLU 3072, RoPE theta 1e6, RMSNorm eps 1e-6)
    "qwen3-0.6b": EncoderConfig("qwen3-0.6b", 28, 1024, 16, 3072, 151669, 512, arch=1,
                                kv_heads=8, head_dim=128),
}

PRECISIONS = {"fp32": 0, "bf16": 1}


def init_weights(cfg: EncoderConfig, seed: int = 0) -> list[np.ndarray]:
    """Seeded random init (PCG64), fp32, in the C-ABI order. arch 0:
    tok_emb, pos_emb, emb_ln_g, emb_ln_b, then per layer
    Wqkv, bqkv, Wo, bo, ln1_g, ln1_b, W1, b1, W2, b2, ln2_g, ln2_b.
    arch 1: tok_emb, then per layer ln1_g, Wqkv (q | k | v heads), q_norm_g,
    k_norm_g, Wo, ln2_g, W_gate, W_up, W_down, and a final norm_g."""
    rng = np.random.default_rng(seed)
    d, f = cfg.hidden, cfg.ffn

    def nrm(*shape, std=0.02):
        return (rng.standard_normal(shape, dtype=np.float32) * np.float32(std)).astype(np.float32)

    def gamma(n):
        return (1.0 + nrm(n)).astype(np.float32)

    if cfg.arch == 1:
        dh = cfg.head_dim or d // cfg.heads
        hk = cfg.kv_heads or cfg.heads
        w = [nrm(cfg.vocab, d)]
        for _ in range(cfg.layers):
            w += [gamma(d), nrm((cfg.heads + 2 * hk) * dh, d), gamma(dh), gamma(dh),
                  nrm(d, cfg.heads * dh), gamma(d), nrm(f, d), nrm(f, d), nrm(d, f)]
        w.append(gamma(d))
        return w

    w = [nrm(cfg.vocab, d), nrm(cfg.max_seq, d), gamma(d), nrm(d)]
    for _ in range(cfg.layers):
        w += [nrm(3 * d, d), nrm(3 * d), nrm(d, d), nrm(d), gamma(d), nrm(d),
              nrm(f, d), nrm(f), nrm(d, f), nrm(d), gamma(d), nrm(d)]
    return w


class GpuEncoder:
    """One ``lv_encoder`` handle (weights resident in HBM)."""

    def __init__(self, cfg: EncoderConfig, weights: list[np.ndarray] | None = None,
                 seed: int = 0, precision: str = "bf16", device: int = 0) -> None:
        if precision not in PRECISIONS:
            raise InvalidArgumentError(f"unknown precision {precision!r}")
        _lib.require_device()
        self.cfg = cfg
        self.precision = precision
        self.device = device
        if weights is None:
            weights = init_weights(cfg, seed)
        if len(weights) != cfg.n_weights:
            raise InvalidArgumentError(f"weights: expected {cfg.n_weights} arrays")
        ws = [np.ascontiguousarray(x, dtype=np.float32) for x in weights]
        arr = (C.c_void_p * len(ws))(*[x.ctypes.data for x in ws])
        c = _lib.EncoderConfigC()
        c.arch, c.layers, c.hidden, c.heads = cfg.arch, cfg.layers, cfg.hidden, cfg.heads
        c.ffn, c.vocab, c.max_seq, c.precision = cfg.ffn, cfg.vocab, cfg.max_seq, PRECISIONS[precision]
        c.kv_heads, c.head_dim = cfg.kv_heads, cfg.head_dim
        c.rope_theta, c.norm_eps = cfg.rope_theta, cfg.norm_eps
        h = C.c_void_p()
        _lib.check(_lib.lib().lv_encoder_create(C.byref(c), C.cast(arr, C.POINTER(C.c_void_p)),
                                                len(ws), device, C.byref(h)))
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().lv_encoder_destroy(self.handle)
            self.handle = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def encode(self, tokens, out=None, stream=None):
        """Embed ``tokens`` [n, S] (u16/u32/int). numpy in -> numpy f32 [n, dim] out;
        CUDA torch tensor in -> CUDA torch tensor out (device-resident, stream-ordered)."""
        if hasattr(tokens, "data_ptr"):
            import torch
            if tokens.dtype == torch.int16 or tokens.dtype == torch.uint16:
                tb = 2
            elif tokens.dtype in (torch.int32, torch.uint32):
                tb = 4
            else:
                raise InvalidArgumentError("device tokens must be 16- or 32-bit integers")
            if not tokens.is_cuda or not tokens.is_contiguous():
                raise InvalidArgumentError("device tokens must be a contiguous CUDA tensor")
            n, S = tokens.shape
            if out is None:
                out = torch.empty((n, self.cfg.hidden), dtype=torch.float32, device=tokens.device)
            st = stream if stream is not None else torch.cuda.current_stream(tokens.device).cuda_stream
            _lib.check(_lib.lib().lv_encode(self.handle, tokens.data_ptr(), tb, n, S,
                                            out.data_ptr(), _lib.LV_IO_DEVICE, st))
            return out
        tok = np.asarray(tokens)
        if tok.ndim != 2:
            raise InvalidArgumentError("tokens must be [n, seq_len]")
        tok = np.ascontiguousarray(tok, dtype=np.uint16 if self.cfg.vocab <= 65536 else np.uint32)
        n, S = tok.shape
        res = np.empty((n, self.cfg.hidden), dtype=np.float32)
        _lib.check(_lib.lib().lv_encode(self.handle, tok.ctypes.data, tok.itemsize, n, S,
                                        res.ctypes.data, 0, None))
        return res

    def set_fused_layernorm(self, enable: bool) -> None:
        """bf16 mode: fold the LayerNorms into the GEMM epilogues (default) or
        run them as standalone kernels."""
        _lib.check(_lib.lib().lv_encoder_set_fused_ln(self.handle, 1 if enable else 0))

    def set_split_residual(self, enable: bool) -> None:
        """bf16 mode: carry the post-LN residual stream as a (hi, lo) bf16 pair
        (default; ~16-bit mantissa, EPF_SPLIT) or round it to bf16 at every
        sublayer (the earlier design, measurably further from fp32)."""
        _lib.check(_lib.lib().lv_encoder_set_split_residual(self.handle, 1 if enable else 0))

    # -- device-timed GEMM counters (roofline evidence)
    def profile(self, enable: bool = True) -> None:
        _lib.check(_lib.lib().lv_encoder_profile(self.handle, 1 if enable else 0))

    def stats(self) -> dict:
        st = _lib.EncoderStats()
        _lib.check(_lib.lib().lv_encoder_stats(self.handle, C.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}

    def reset_stats(self) -> None:
        _lib.check(_lib.lib().lv_encoder_reset_stats(self.handle))


# --------------------------------------------------------------------------- token store

class TokenStore:
    """Fixed-length token chunks, one per node: ``tokens[i]`` is node i's payload."""

    def __init__(self, tokens: np.ndarray) -> None:
        tokens = np.asarray(tokens)
        if tokens.ndim != 2:
            raise InvalidArgumentError("tokens must be [n, seq_len]")
        if tokens.dtype not in (np.uint16, np.uint32):
            raise InvalidArgumentError("token store holds u16 or u32 ids")
        self.tokens = np.ascontiguousarray(tokens)

    @property
    def n(self) -> int:
        return self.tokens.shape[0]

    @property
    def seq_len(self) -> int:
        return self.tokens.shape[1]

    @property
    def token_bytes(self) -> int:
        return self.tokens.itemsize

    def get(self, i: int) -> bytes:
        """Payload bytes of node i (ItemStore.get, store.py:89-94)."""
        if not 0 <= i < self.n:
            raise InvalidArgumentError(f"item id {i} out of range [0, {self.n})")
        return self.tokens[i].astype("<" + self.tokens.dtype.str[1:]).tobytes()

    def save(self, directory) -> None:
        """items.dat + u64 items.idx (store.py:1-116 layout; ItemStore.open reads it)."""
        d = Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        le = self.tokens.astype("<" + self.tokens.dtype.str[1:], copy=False)
        (d / ITEMS_DAT).write_bytes(le.tobytes())
        row = self.seq_len * self.token_bytes
        offs = np.arange(self.n + 1, dtype="<u8") * np.uint64(row)
        (d / ITEMS_IDX).write_bytes(offs.tobytes())

    @classmethod
    def load(cls, directory, token_bytes: int = 2) -> "TokenStore":
        d = Path(directory)
        offs = np.frombuffer((d / ITEMS_IDX).read_bytes(), dtype="<u8")
        raw = np.fromfile(d / ITEMS_DAT, dtype="<u2" if token_bytes == 2 else "<u4")
        n = offs.shape[0] - 1
        if n <= 0 or raw.size % n:
            raise InvalidArgumentError("token store rows are not fixed-length")
        return cls(raw.reshape(n, raw.size // n).astype(np.uint16 if token_bytes == 2 else np.uint32))


def synthetic_tokens(n: int, seq_len: int, vocab: int, seed: int) -> np.ndarray:
    """Uniform token ids in [0, vocab), PCG64-seeded."""
    rng = np.random.default_rng(seed)
    dt = np.uint16 if vocab <= 65536 else np.uint32
    return rng.integers(0, vocab, size=(n, seq_len), dtype=dt)


def topic_tokens(n: int, seq_len: int, vocab: int, seed: int, n_topics: int,
                 topic_frac: float = 0.5, topic_vocab: int = 512, zipf: float = 1.1,
                 topic_seed: int = 1234, chunk: int = 65536) -> np.ndarray:
    """Topic-structured synthetic passages: each passage draws one of
    ``n_topics`` topics; each token is, with probability ``topic_frac``, a
    Zipf(``zipf``)-ranked draw from that topic's ``topic_vocab`` ids, else a
    uniform id. Topic vocabularies come from ``topic_seed`` (shared by passages
    and queries); ``seed`` drives the per-passage draws (PCG64).

    Uniform-token passages under a 12-layer random-init encoder have no
    neighbourhood structure (BERT-base: pairwise cosine 0.982 +- 0.002, the
    1st and 20th neighbours within 0.1%), so any graph index degenerates to
    exhaustive search; topics give retrieval-like structure."""
    trng = np.random.default_rng(topic_seed)
    sets = trng.integers(0, vocab, size=(n_topics, topic_vocab))
    w = 1.0 / np.arange(1, topic_vocab + 1, dtype=np.float64) ** zipf
    cdf = np.cumsum(w / w.sum())
    rng = np.random.default_rng(seed)
    dt = np.uint16 if vocab <= 65536 else np.uint32
    out = np.empty((n, seq_len), dtype=dt)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        m = e - s
        topic = rng.integers(0, n_topics, size=m)
        rank = np.minimum(np.searchsorted(cdf, rng.random((m, seq_len))), topic_vocab - 1)
        from_topic = rng.random((m, seq_len)) < topic_frac
        uni = rng.integers(0, vocab, size=(m, seq_len))
        out[s:e] = np.where(from_topic, sets[topic[:, None], rank], uni).astype(dt)
    return out


def lda_tokens(n: int, seq_len: int, vocab: int, seed: int, n_topics: int = 64,
               alpha: float = 0.1, topic_vocab: int = 1024, zipf: float = 1.0,
               background: float = 0.1, topic_seed: int = 1234,
               chunk: int = 32768) -> np.ndarray:
    """LDA-style synthetic passages (the default corpus of the benchmarks).

    Passage p draws topic proportions theta_p ~ Dirichlet(alpha) over
    ``n_topics`` topics; each of its ``seq_len`` tokens picks a topic from
    theta_p and then a Zipf(``zipf``)-ranked id from that topic's
    ``topic_vocab`` ids, or (with probability ``background``) a uniform id.
    Topic vocabularies come from ``topic_seed`` and are shared by passages and
    queries; ``seed`` drives the per-passage draws (PCG64). Embeddings then
    vary along the continuous, low-dimensional topic-mixture manifold, like
    real retrieval corpora, instead of being isotropic noise (uniform tokens:
    see ``topic_tokens``)."""
    trng = np.random.default_rng(topic_seed)
    sets = trng.integers(0, vocab, size=(n_topics, topic_vocab))
    w = 1.0 / np.arange(1, topic_vocab + 1, dtype=np.float64) ** zipf
    cdf = np.cumsum(w / w.sum())
    rng = np.random.default_rng(seed)
    dt = np.uint16 if vocab <= 65536 else np.uint32
    out = np.empty((n, seq_len), dtype=dt)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        m = e - s
        theta = rng.dirichlet(np.full(n_topics, alpha), size=m)
        counts = rng.multinomial(seq_len, theta)
        topics = np.repeat(np.tile(np.arange(n_topics), m), counts.ravel()).reshape(m, seq_len)
        topics = rng.permuted(topics, axis=1)
        rank = np.minimum(np.searchsorted(cdf, rng.random((m, seq_len))), topic_vocab - 1)
        tok = sets[topics, rank]
        bg = rng.random((m, seq_len)) < background
        tok = np.where(bg, rng.integers(0, vocab, size=(m, seq_len)), tok)
        out[s:e] = tok.astype(dt)
    return out


@dataclass(frozen=True)
class EncoderProviderConfig:
    """The fields of ProviderConfig (vectors.py:41-65) a provider exposes."""

    dim: int
    max_batch: int = 1 << 20
    kind: str = "lv-encoder"


class EncoderProvider:
    """Duck-typed provider (vectors.py:201-211) bound to a token store.

    ``embed_batch`` decodes each request's payload bytes as token ids and runs
    the GPU encoder; inside the batched search the same encoder is driven
    directly from the device-resident token store (lv_index_attach_encoder).
    """

    def __init__(self, encoder: GpuEncoder, store, max_batch: int = 1 << 20) -> None:
        self.encoder = encoder
        self.store = store  # TokenStore or a CUDA tensor [n, seq_len]
        self.config = EncoderProviderConfig(dim=encoder.cfg.hidden, max_batch=max_batch)

    def _tokens(self):
        return self.store.tokens if isinstance(self.store, TokenStore) else self.store

    def embed_batch(self, requests) -> np.ndarray:
        if not requests:
            raise InvalidArgumentError("embed_batch requires a non-empty batch")
        if len(requests) > self.config.max_batch:
            raise InvalidArgumentError(
                f"batch of {len(requests)} exceeds max_batch {self.config.max_batch}")
        tok = self._tokens()
        dt = np.dtype("<u2") if tok.dtype in (np.uint16,) or str(tok.dtype).endswith("int16") \
            else np.dtype("<u4")
        rows = [np.frombuffer(r.content, dtype=dt) for r in requests]
        if len({r.shape[0] for r in rows}) != 1:
            raise InvalidArgumentError("payloads must have equal token counts")
        return self.encoder.encode(np.stack(rows).astype(dt.newbyteorder("=")))

    def attach(self, device_index) -> None:
        tok = self._tokens()
        if hasattr(tok, "data_ptr"):
            tb = tok.element_size()
            _lib.check(_lib.lib().lv_index_attach_encoder(device_index.handle, self.encoder.handle,
                                                          tok.data_ptr(), tb, tok.shape[1],
                                                          _lib.LV_IO_DEVICE))
        else:
            t = np.ascontiguousarray(tok)
            if t.shape[0] != device_index.n:
                raise InvalidArgumentError("token store size != graph size")
            _lib.check(_lib.lib().lv_index_attach_encoder(device_index.handle, self.encoder.handle,
                                                          t.ctypes.data, t.itemsize, t.shape[1], 0))
        device_index._token_ref = tok
