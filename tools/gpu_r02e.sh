#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_builder_parity.py tests/test_gpu_c2shape_parity.py tests/test_gpu_c1_parity.py -q -s -rf > gpurun_out/gputests_e.log 2>&1; echo tests=$?
grep -E "GPU graph|codes differ|passed|failed|Error" gpurun_out/gputests_e.log | head -20
timeout 2400 python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02e.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["config"]["recall_at_3"], d["config"]["heldout_recall_at_3"], d["cpu_baseline"])
PY
grep -E "setup|embedded|index built|chosen" gpurun_out/bench_r02e.err
