"""LPQ1 product-quantisation artefacts (reference pq.py:1-244) and the device ADC.

``adc_build`` / ``approx_distance_many`` run the sm_100a kernels through the
C-ABI (lut_kernel / adc_score_kernel) and are bit-exact with the reference
(einsum-order LUT entries, numpy-pairwise float64 sums).
"""
from __future__ import annotations

import io
import struct
from dataclasses import dataclass

import numpy as np

from .errors import FormatError, InvalidArgumentError

CENTROIDS_PER_SUBSPACE = 256
METRICS = ("l2", "ip", "cosine")
_MAGIC = b"LPQ1"
_HEADER = struct.Struct("<4sHIIHBxQ")


def default_m_pq(dim: int) -> int:
    """pq.py:35-37."""
    return max(1, int(round(dim / 25.6)))


@dataclass
class PQModel:
    dim: int
    padded_dim: int
    m_pq: int
    metric: str
    codebooks: np.ndarray  # (m, 256, padded_dim // m) float32

    @property
    def sub_dim(self) -> int:
        return self.padded_dim // self.m_pq


@dataclass
class PQCodes:
    codes: np.ndarray  # (n, m) uint8

    @property
    def n(self) -> int:
        return self.codes.shape[0]

    @property
    def m_pq(self) -> int:
        return self.codes.shape[1]


def save_pq(model: PQModel, codes: PQCodes, path) -> None:
    buf = io.BytesIO()
    buf.write(_HEADER.pack(_MAGIC, 1, model.dim, model.padded_dim, model.m_pq,
                           METRICS.index(model.metric), codes.n))
    buf.write(np.ascontiguousarray(model.codebooks, dtype="<f4").tobytes())
    buf.write(np.ascontiguousarray(codes.codes, dtype=np.uint8).tobytes())
    with open(path, "wb") as fh:
        fh.write(buf.getvalue())


def load_pq(path) -> tuple[PQModel, PQCodes]:
    """pq.py:213-244."""
    data = open(path, "rb").read()
    if len(data) < _HEADER.size:
        raise FormatError("pq.header", "file truncated before header")
    magic, version, dim, padded, m, tag, n = _HEADER.unpack_from(data)
    if magic != _MAGIC:
        raise FormatError("pq.magic", f"bad magic {magic!r}")
    if version != 1:
        raise FormatError("pq.version", f"unsupported version {version}")
    if tag >= len(METRICS):
        raise FormatError("pq.metric", f"unknown metric tag {tag}")
    if m < 1 or padded % m != 0:
        raise FormatError("pq.header", f"invalid geometry dim={dim} m={m}")
    cb_bytes = m * CENTROIDS_PER_SUBSPACE * (padded // m) * 4
    pos = _HEADER.size
    if len(data) < pos + cb_bytes:
        raise FormatError("pq.codebooks", "file truncated inside codebooks")
    cb = np.frombuffer(data, "<f4", cb_bytes // 4, pos).reshape(
        m, CENTROIDS_PER_SUBSPACE, padded // m).copy()
    if not np.all(np.isfinite(cb)):
        raise FormatError("pq.codebooks", "non-finite centroid entries")
    pos += cb_bytes
    if len(data) != pos + n * m:
        raise FormatError("pq.codes", f"expected {n * m} code bytes, found {len(data) - pos}")
    codes = np.frombuffer(data, np.uint8, n * m, pos).reshape(n, m).copy()
    return PQModel(dim, padded, m, METRICS[tag], cb), PQCodes(codes)


def adc_build(model: PQModel, q: np.ndarray, device_index=None) -> np.ndarray:
    """(m, 256) LUT on the device (pq.py:153-178)."""
    from .search import DeviceIndex, query_norm
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.shape[0] != model.dim:
        raise InvalidArgumentError(f"expected dim {model.dim}, got {q.shape[0]}")
    qn = np.array([query_norm(q)], dtype=np.float32)
    if model.metric == "cosine" and qn[0] == 0.0:
        raise InvalidArgumentError("cosine ADC undefined for zero query")
    dev = device_index or DeviceIndex.for_pq(model)
    return dev.adc_tables(q.reshape(1, -1), qn)[0]


def approx_distance_many(table: np.ndarray, codes_or_ids, device_index) -> np.ndarray:
    """Table-lookup distances of the given node ids on the device (pq.py:186-189)."""
    return device_index.adc_score(table, np.asarray(codes_or_ids, dtype=np.int64))
