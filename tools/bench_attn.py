"""Microbenchmark of the encoder attention (config-2 shape by default): tcgen05
kernel (mode 0) vs mma.sync kernel (mode 1) vs torch SDPA, CUDA events."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256
H, dh = 12, 64
qkv = torch.randn(n * S, 3 * H * dh, device="cuda").to(torch.bfloat16)
out = torch.empty(n * S, H * dh, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream()
fl = 4.0 * S * S * dh * H * n
L = _lib.lib()
for mode in (0, 1):
    L.lv_set_attention_mode(mode)
    for _ in range(3):
        _lib.check(L.lv_attention_bf16(qkv.data_ptr(), out.data_ptr(), n, S, H, dh, st.cuda_stream))
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(L.lv_attention_bf16(qkv.data_ptr(), out.data_ptr(), n, S, H, dh, st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[3]
    print(f"attention mode={mode} n={n} S={S} H={H} dh={dh}: {t*1e3:.1f} us  {fl / t / 1e9:.1f} TF/s  "
          f"{(3 + 1) * n * S * H * dh * 2 / t / 1e6:.0f} GB/s (qkv+ctx)", flush=True)
L.lv_set_attention_mode(0)
q = qkv.view(n, S, 3, H, dh)
args = (q[:, :, 0].transpose(1, 2), q[:, :, 1].transpose(1, 2), q[:, :, 2].transpose(1, 2))
for _ in range(2):
    torch.nn.functional.scaled_dot_product_attention(*args)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
torch.nn.functional.scaled_dot_product_attention(*args)
e1.record(st)
torch.cuda.synchronize()
print(f"torch sdpa (incl. strided views): {e0.elapsed_time(e1)*1e3:.1f} us")
