#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_search.py tests/test_gpu_c2shape_parity.py tests/test_gpu_c1_parity.py tests/test_gpu_dropin.py tests/test_gpu_engine_merge.py -q -rf > gpurun_out/gputests_h.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests_h.log
python tools/bench_frontier.py > gpurun_out/frontier_ab.txt 2>&1; tail -6 gpurun_out/frontier_ab.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:frontier --csv --log-file gpurun_out/frontier_ncu.csv python tools/bench_frontier.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/frontier_ncu.csv > gpurun_out/frontier_ncu.txt; cat gpurun_out/frontier_ncu.txt
