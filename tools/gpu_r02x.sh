#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py --config c1 --steps 2 --warmup 3 > gpurun_out/bench_c1_t.json 2> gpurun_out/bench_c1_t.err; echo c1=$?
grep "step=" gpurun_out/bench_c1_t.err | tail -12
tail -c 300 gpurun_out/bench_c1_t.json
