#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 3300 python bench.py --config c4 --steps 1 --warmup 1 --ef-max 1024 --alpha-sweep --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_1m.json 2> gpurun_out/bench_c4_1m.err; echo c4=$?
grep -E "chosen|rerank sweep" gpurun_out/bench_c4_1m.err
