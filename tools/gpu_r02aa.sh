#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -x -rf -k "decoder or gqa or tc_gemm" > gpurun_out/dec_tests.log 2>&1; echo dtests=$?; tail -3 gpurun_out/dec_tests.log
grep -E "Error|assert" gpurun_out/dec_tests.log | head -5
python - <<'PY'
import subprocess, sys
from paper_2506_08276_b200 import _lib
PY
for f in 1 0 1 0; do timeout 300 python -c "
import sys; sys.argv=['x','256']
from paper_2506_08276_b200 import _lib
import __graft_entry__ as g; g.build()
_lib.lib().lv_set_fused_qk_rope($f)
exec(open('tools/encode_c4_once.py').read())
" 2>&1 | tail -1; done
