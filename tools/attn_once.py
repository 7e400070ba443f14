"""Run the encoder attention once per mode given (for ncu captures)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as ge  # noqa: E402
ge.build()
from paper_2506_08276_b200 import _lib  # noqa: E402
n, S, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
H, dh = 12, 64
qkv = torch.randn(n * S, 3 * H * dh, device="cuda").to(torch.bfloat16)
out = torch.empty(n * S, H * dh, device="cuda", dtype=torch.bfloat16)
L = _lib.lib()
L.lv_set_attention_mode(mode)
for _ in range(3):
    _lib.check(L.lv_attention_bf16(qkv.data_ptr(), out.data_ptr(), n, S, H, dh,
                                   torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
