#!/bin/bash
# Launch list of one timed step (reduced corpus) + full captures of the top kernels.
set -x
ARGS="--config c2 --n 100000 --steps 1 --warmup 1 --batch 256 --ef 47 --alphas 100 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_c2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:tc_gemm_kernel -s 20 -c 2 -o gpurun_out/prof_gemm -f python bench.py $ARGS > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:attn_bf16 -s 2 -c 1 -o gpurun_out/prof_attn -f python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:frontier_kernel -s 5 -c 1 -o gpurun_out/prof_frontier -f python bench.py $ARGS > gpurun_out/ncu_frontier.log 2>&1
ls -la gpurun_out
