"""Sustained (power-capped) config-2 attention: mode 0 (MUFU exponentials) vs
mode 2 (every third exponential by polynomial on the FMA pipe), ~4 s back to
back each with nvidia-smi power/clock sampling."""
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
n, S, H, dh = 2048, 256, 12, 64
qkv = torch.randn(n * S, 3 * H * dh, device="cuda").to(torch.bfloat16)
out = torch.empty(n * S, H * dh, device="cuda", dtype=torch.bfloat16)
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append([float(x) for x in line.split(",")])
    p.terminate()


for mode in (0, 2, 0, 2):
    L.lv_set_attention_mode(mode)
    for _ in range(3):
        _lib.check(L.lv_attention_bf16(qkv.data_ptr(), out.data_ptr(), n, S, H, dh, st))
    torch.cuda.synchronize()
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, rows))
    th.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            _lib.check(L.lv_attention_bf16(qkv.data_ptr(), out.data_ptr(), n, S, H, dh, st))
        k += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = e0.elapsed_time(e1) / k * 1e3
    pw = statistics.mean(r[0] for r in rows[5:]) if len(rows) > 6 else float("nan")
    clk = statistics.median(r[1] for r in rows[5:]) if len(rows) > 6 else float("nan")
    print(f"attention mode {mode}: {us:.1f} us/launch sustained, sm {clk:.0f} MHz, {pw:.0f} W", flush=True)
L.lv_set_attention_mode(0)
