#!/bin/bash
# Launch list (device time + DRAM bytes per launch) of one timed config-2 step on a
# reduced corpus, then full captures of the top kernels inside the timed range.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
ARGS="--config c2 --n 100000 --steps 1 --warmup 1 --batch 512 --ef 51 --alphas 90 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_c2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:tc_gemm_pair -s 20 -c 4 -o gpurun_out/prof_gemm_step -f python bench.py $ARGS > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:attn_tc -s 2 -c 1 -o gpurun_out/prof_attn_step -f python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:frontier_kernel -s 5 -c 1 -o gpurun_out/prof_frontier -f python bench.py $ARGS > gpurun_out/ncu_frontier.log 2>&1
ls -la gpurun_out
