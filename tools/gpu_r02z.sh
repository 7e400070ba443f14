#!/bin/bash
# Concurrent-query sweep on the 1M config-2 index with the final kernels.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 3000 python bench.py --config c2 --batch 4096 --steps 1 --warmup 1 --alphas 70 --no-cpu-baseline --no-e2e --batch-sweep 256,1024,4096,16384 > gpurun_out/bench_c2_sweep.json 2> gpurun_out/bench_c2_sweep.err; echo sweep=$?
grep sweep gpurun_out/bench_c2_sweep.err | tail -5
