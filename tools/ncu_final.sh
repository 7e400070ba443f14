#!/bin/bash
# Final evidence for profiles/: launch list (time + DRAM bytes) of one reduced
# config-2 step, and full captures of the GEMM (residual + LN-in variants),
# attention and frontier kernels inside the timed range.
python -c "import __graft_entry__ as g; g.build()" || exit 1
ARGS="--config c2 --n 50000 --steps 1 --warmup 1 --batch 512 --ef 51 --alphas 90 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_c2_final.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_c2_final.csv --json gpurun_out/traffic.json
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair -s 4 -c 4 -o gpurun_out/prof_gemm_final -f python tools/encode_once.py 1024 1 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/prof_attn_final -f python tools/attn_once.py 1024 256 0 > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:frontier_kernel -s 5 -c 1 -o gpurun_out/prof_frontier_final -f python bench.py $ARGS > gpurun_out/ncu_frontier.log 2>&1
ls -la gpurun_out
