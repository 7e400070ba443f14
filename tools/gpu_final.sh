#!/bin/bash
# Round-end evidence: GPU tests, smoke, the default bench, a 2-rank (gloo, one GPU) bench,
# and an ncu launch list (device time + DRAM bytes) of the timed config-2 step's first launches.
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
timeout 2400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["config"]["ef"], d["config"]["rerank_percent"], d["config"]["recall_at_3"], d["config"]["heldout_recall_at_3"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"])
open("gpurun_out/tuned.txt", "w").write(f"{d['config']['ef']} {d['config']['rerank_percent']}")
PY
read EF ALPHA < gpurun_out/tuned.txt
LV_BENCH_BACKEND=gloo LV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --corpus-size 100000 --batch 1024 --steps 2 --warmup 1 --ef $EF --alphas $ALPHA --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo tworank=$?
tail -c 600 gpurun_out/bench_2rank_gloo.json
ARGS="--config c2 --steps 1 --warmup 1 --ef $EF --alphas $ALPHA --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" -c 1500 --csv --log-file gpurun_out/launches_c2_r02.csv python bench.py $ARGS > gpurun_out/ncu_launch_r02.log 2>&1; echo ncu=$?
python tools/summarize_launches.py gpurun_out/launches_c2_r02.csv --json gpurun_out/traffic_r02.json > gpurun_out/launches_c2_r02.txt; head -14 gpurun_out/launches_c2_r02.txt
