#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 3300 python bench.py --config c3 --batch 4096 --steps 1 --warmup 1 --alphas 75,90 --ef-max 512 --no-cpu-baseline --no-e2e --batch-sweep 1024,4096,16384 > gpurun_out/bench_c3_r02b.json 2> gpurun_out/bench_c3_r02b.err; echo c3=$?
grep sweep gpurun_out/bench_c3_r02b.err
