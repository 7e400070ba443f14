#!/bin/bash
# bench.py smoke of the new report fields (small config-2), config-4 encoder throughput.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py --config c2 --corpus-size 100000 --batch 1024 --steps 1 --warmup 3 --ef 113 --alphas 70 --no-cpu-baseline > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err; echo small=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_small.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"] if d.get("e2e") else None)
for r in d["rooflines"]: print(r["kernel"][:30], r["achieved"], r["frac"], r.get("l2_feed"))
PY
for i in 1 2; do timeout 600 python tools/encode_c4_once.py 2>&1 | tail -1; done
