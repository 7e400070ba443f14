#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/make_c2shape_index.py gpurun_out/c2shape > gpurun_out/c2shape.log 2>&1; echo c2shape=$?
tail -2 gpurun_out/c2shape.log
PYTEST_ARGS="--deselect nothing" bash tools/gpu_tests.sh
