#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_c2_encoder_parity.py tests/test_gpu_dropin.py -q -s -rf > gpurun_out/gputests_m.log 2>&1; echo tests=$?
grep -E "BERT|passed|failed|Error" gpurun_out/gputests_m.log | head
