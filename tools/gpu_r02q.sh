#!/bin/bash
# Round-2 (session 3) evidence with the fused QKV+attention kernel: smoke, full GPU suite,
# default bench, ncu launch list of the timed step (first 1500 launches).
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
timeout 2400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["config"]["ef"], d["config"]["rerank_percent"], d["config"]["recall_at_3"], d["config"]["heldout_recall_at_3"], d["clocks"])
for r in d["rooflines"]: print(r["kernel"][:40], r["achieved"], r["frac"], r.get("share_of_step"))
open("gpurun_out/tuned.txt", "w").write(f"{d['config']['ef']} {d['config']['rerank_percent']}")
PY
read EF ALPHA < gpurun_out/tuned.txt
ARGS="--config c2 --steps 1 --warmup 1 --ef $EF --alphas $ALPHA --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" -c 1500 --csv --log-file gpurun_out/launches_c2_r02s3.csv python bench.py $ARGS > gpurun_out/ncu_launch_r02s3.log 2>&1; echo ncu=$?
python tools/summarize_launches.py gpurun_out/launches_c2_r02s3.csv --json gpurun_out/traffic_r02s3.json > gpurun_out/launches_c2_r02s3.txt; head -14 gpurun_out/launches_c2_r02s3.txt
