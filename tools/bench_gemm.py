"""Microbenchmark of the encoder GEMM shapes: 1-CTA vs 2-CTA tcgen05 kernels vs cuBLAS.

CUDA events on the launching stream, warm-up first, L2 flushed between runs
(the activations exceed L2 anyway at these M)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402

ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402

L = _lib.lib()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
shapes = [("qkv", 2304, 768, 0), ("out", 768, 768, 2), ("ffn1", 3072, 768, 1), ("ffn2", 768, 3072, 2)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for name, N, K, epi in shapes:
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    line = [f"{name:5s} M={M} N={N} K={K}"]
    for mode in (4, 0):
        L.lv_set_gemm_mode(mode)
        for _ in range(3):
            _lib.check(L.lv_gemm_bf16(A.data_ptr(), W.data_ptr(), bias.data_ptr(), res.data_ptr(),
                                      out.data_ptr(), M, N, K, epi, st.cuda_stream))
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(L.lv_gemm_bf16(A.data_ptr(), W.data_ptr(), bias.data_ptr(), res.data_ptr(),
                                      out.data_ptr(), M, N, K, epi, st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        line.append(f"{"2cta-2buf4st" if mode else "2cta"} {fl / t / 1e9:7.1f} TF/s")
    ref = torch.nn.functional.linear(A, W, bias.to(torch.bfloat16))
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        torch.nn.functional.linear(A, W, bias.to(torch.bfloat16))
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    line.append(f"cublas {fl / t / 1e9:7.1f} TF/s")
    print("  ".join(line), flush=True)
L.lv_set_gemm_mode(0)
