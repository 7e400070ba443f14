#!/bin/bash
# Launch list (device time + DRAM bytes per launch) of one timed config-2 step on a reduced
# corpus (the committed profiles/traffic.json and r01_launches_c2_final.* come from this).
python -c "import __graft_entry__ as g; g.build()" || exit 1
ARGS="--config c2 --corpus-size 50000 --steps 1 --warmup 1 --batch 512 --ef 73 --alphas 75 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_c2_final.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_c2_final.csv --json gpurun_out/traffic.json
