#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_c1_parity.py -q -x > gpurun_out/gputests_l.log 2>&1; echo tests=$?; tail -1 gpurun_out/gputests_l.log
for i in 1 2; do python tools/encode_split.py 2048 1 2>&1 | tail -1; done
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm_pair -s 4 -c 4 --csv --log-file gpurun_out/gemm4.csv python tools/encode_split.py 512 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/gemm4.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r); hdr=rows[h]
for r in rows[h+1:]:
    print(r[hdr.index("Kernel Name")][:40], r[hdr.index("Metric Name")], r[hdr.index("Metric Value")])
PY
