#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_search.py tests/test_gpu_c2shape_parity.py tests/test_gpu_recompute.py tests/test_gpu_c1_parity.py -q -rf -x > gpurun_out/gputests_i.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests_i.log
python tools/bench_frontier.py > gpurun_out/frontier_ab.txt 2>&1; tail -8 gpurun_out/frontier_ab.txt
