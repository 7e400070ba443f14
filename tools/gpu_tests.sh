#!/bin/bash
# GPU test pass + host BLAS identification (which sdot kernel numpy uses here).
python -c "import __graft_entry__ as g; g.build()" || exit 1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt
python -c "import numpy; from threadpoolctl import threadpool_info; print([(d.get('internal_api'), d.get('architecture')) for d in threadpool_info()])" >> gpurun_out/host_cpu.txt
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -s ${PYTEST_ARGS:--x} > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputests.log
