#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
timeout 2400 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo bench=$?
tail -2 gpurun_out/bench_r02d.err
timeout 1800 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02d.json 2> gpurun_out/bench_ref_r02d.err; echo ref=$?
tail -2 gpurun_out/bench_ref_r02d.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_r02d.json", "gpurun_out/bench_ref_r02d.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d.get("e2e", {}).get("value"), d["config"].get("recall_at_3"), d["config"].get("heldout_recall_at_3"), d.get("cpu_baseline", {}).get("value"), d.get("cpu_baseline", {}).get("sample", "")[:400])
    except Exception as e:
        print(f, "error", e)
PY
