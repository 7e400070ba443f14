#!/bin/bash
# Re-entry check: build, smoke, full GPU suite, then one short default-config bench.
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err; echo bench=$?
tail -c 3000 gpurun_out/bench_n.json
