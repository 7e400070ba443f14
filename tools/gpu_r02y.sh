#!/bin/bash
# Final-state default bench (config-2) + GPU suite.
python -c "import __graft_entry__ as g; g.build()" || exit 1
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
timeout 2400 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final2.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["config"]["ef"], d["config"]["rerank_percent"], d["config"]["recall_at_3"], d["config"]["heldout_recall_at_3"], d["clocks"])
for r in d["rooflines"]: print(r["kernel"][:40], r["achieved"], r["frac"], r.get("share_of_step"), (r.get("l2_feed") or {}).get("frac_of_cap"))
PY
