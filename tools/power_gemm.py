"""Sustained (power-capped) GEMM efficiency: ours vs cuBLAS on the encoder
shapes, each run back to back for ~4 s with nvidia-smi sampling power and SM
clock. Reports TF/s, median clock, mean power and TFLOP per joule."""
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402

ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402

L = _lib.lib()
M = 262144
shapes = [("qkv", 2304, 768, 0), ("out", 768, 768, 2), ("ffn1", 3072, 768, 1), ("ffn2", 768, 3072, 2)]


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append([float(x) for x in line.split(",")])
    p.terminate()


st = torch.cuda.current_stream()
for name, N, K, epi in shapes:
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    bb = bias.to(torch.bfloat16)
    for impl in ("ours", "cublas"):
        def run():
            if impl == "ours":
                _lib.check(L.lv_gemm_bf16(A.data_ptr(), W.data_ptr(), bias.data_ptr(), res.data_ptr(),
                                          out.data_ptr(), M, N, K, epi, st.cuda_stream))
            else:
                torch.nn.functional.linear(A, W, bb, out=None)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        rows, stop = [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, rows))
        th.start()
        time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        e0.record(st)
        t0 = time.time()
        while time.time() - t0 < 4.0:
            for _ in range(20):
                run()
            n += 20
            torch.cuda.synchronize()
        e1.record(st)
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / n
        tf = fl / ms / 1e9
        pw = statistics.mean(r[0] for r in rows[5:]) if len(rows) > 6 else float("nan")
        clk = statistics.median(r[1] for r in rows[5:]) if len(rows) > 6 else float("nan")
        print(f"{name:5s} {impl:6s} {tf:7.1f} TF/s  sm {clk:6.0f} MHz  {pw:6.1f} W  "
              f"{tf / pw:5.2f} TFLOP/J", flush=True)
