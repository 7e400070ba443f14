#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
grep -E "split|bf16 \{|fp32 \{" gpurun_out/gputests.log | head -20
bash tools/gpu_split_ab.sh
