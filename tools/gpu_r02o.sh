#!/bin/bash
# Fused QKV + attention kernel: parity tests first (bounded), then encoder A/B.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_qkv_attn.py -q -x -rf > gpurun_out/qkv_tests.log 2>&1; echo qtests=$?
tail -15 gpurun_out/qkv_tests.log
if grep -q " passed" gpurun_out/qkv_tests.log && ! grep -q "failed" gpurun_out/qkv_tests.log; then
  for f in 0 1 0 1; do timeout 300 python tools/encode_fused.py 2048 $f 3 2>&1 | tail -1; done
  timeout 600 python -m pytest tests/test_gpu_encoder.py -q -x -k "encoder" > gpurun_out/enc_tests.log 2>&1; echo etests=$?; tail -3 gpurun_out/enc_tests.log
fi
