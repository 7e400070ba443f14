#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frontier_kernel -s 3 -c 1 -o gpurun_out/r02_frontier_global python tools/bench_frontier.py > /dev/null 2>&1; echo ncu=$?
