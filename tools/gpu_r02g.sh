#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_c1_parity.py tests/test_gpu_encoder_parity.py -q -s -rf > gpurun_out/gputests_g.log 2>&1; echo tests=$?
grep -E "split|bf16 \{|passed|failed" gpurun_out/gputests_g.log | head
bash tools/gpu_split_ab.sh
