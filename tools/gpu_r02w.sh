#!/bin/bash
# ADC with 8-byte code loads: bit-exact search tests, then the frontier A/B (tools/bench_frontier.py).
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_c2shape_parity.py tests/test_gpu_c1_parity.py tests/test_gpu_recompute.py -q -x -rf > gpurun_out/search_tests.log 2>&1; echo stests=$?; tail -2 gpurun_out/search_tests.log
timeout 600 python tools/bench_frontier.py 2>&1 | tail -8
