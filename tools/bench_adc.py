"""Streaming ADC microbenchmark (approx_distance_many, pq.py:186-189): score n
random node ids against one query LUT through lv_adc_score (device pointers).
Algorithmic bytes per id: m code bytes + 8 (id) + 4 (score). CUDA events."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
import ctypes as C  # noqa: E402
from paper_2506_08276_b200 import _lib  # noqa: E402
from paper_2506_08276_b200.graph import PrunedGraph  # noqa: E402
from paper_2506_08276_b200.pq import PQCodes, PQModel  # noqa: E402
from paper_2506_08276_b200.search import DeviceIndex  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dim = 768
rng = np.random.default_rng(0)
g = PrunedGraph(n=n, max_degree=1, entry_point=0, levels=np.zeros(n, np.uint16),
                level_offsets=[np.zeros(n + 1, np.uint64)], level_neighbors=[np.zeros(0, np.uint32)])
model = PQModel(dim=dim, padded_dim=dim if dim % m == 0 else dim + m - dim % m, m_pq=m,
                metric="cosine",
                codebooks=rng.standard_normal((m, 256, (dim + m - 1) // m), dtype=np.float32))
codes = PQCodes(codes=rng.integers(0, 256, (n, m), dtype=np.uint8))
dev = DeviceIndex(g, model, codes)
lut = torch.randn(m * 256, device="cuda")
out = torch.empty(n, device="cuda")
st = torch.cuda.current_stream().cuda_stream
L = _lib.lib()
for order in ("random", "sorted"):
    ids = torch.randperm(n, device="cuda") if order == "random" else torch.arange(n, device="cuda")
    for _ in range(3):
        _lib.check(L.lv_adc_score(dev.handle, lut.data_ptr(), ids.data_ptr(), n, out.data_ptr(),
                                  _lib.LV_IO_DEVICE, st))
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.lv_adc_score(dev.handle, lut.data_ptr(), ids.data_ptr(), n, out.data_ptr(),
                                  _lib.LV_IO_DEVICE, st))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[2]
    gb = n * (m + 12) / 1e9
    print(f"ADC stream ({order} ids): {n} ids x m={m}: {t:.3f} ms, {gb / (t / 1e3):.0f} GB/s "
          f"algorithmic ({n / t / 1e6:.2f} G ids/s)", flush=True)
# correctness: tests/test_gpu_search.py checks lv_adc_score bit-for-bit against the
# reference-produced golden ADC vectors (m = 32 and m = 64)
