#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_builder_parity.py -q -s > gpurun_out/gputests_f.log 2>&1; echo tests=$?
grep -E "GPU graph|passed|failed" gpurun_out/gputests_f.log
timeout 2400 python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02f.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["config"]["ef"], d["config"]["rerank_percent"], d["config"]["recall_at_3"], d["config"]["heldout_recall_at_3"], d["recomputes_per_query"], d["recomputed_embeddings_per_s"], d["roofline"]["achieved"], d["roofline"]["frac"])
open("gpurun_out/tuned.txt", "w").write(f"{d['config']['ef']} {d['config']['rerank_percent']}")
PY
read EF ALPHA < gpurun_out/tuned.txt
ARGS="--config c2 --steps 1 --warmup 1 --ef $EF --alphas $ALPHA --no-cpu-baseline --no-e2e"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_c2_r02.csv python bench.py $ARGS > gpurun_out/ncu_launch_r02.log 2>&1; echo ncu=$?
python tools/summarize_launches.py gpurun_out/launches_c2_r02.csv --json gpurun_out/traffic_r02.json > gpurun_out/launches_c2_r02.txt; head -12 gpurun_out/launches_c2_r02.txt
