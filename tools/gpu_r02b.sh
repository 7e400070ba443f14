#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
PYTEST_ARGS="-rf" bash tools/gpu_tests.sh
grep -E "split|bf16 \{|fp32 \{" gpurun_out/gputests.log | head -20
timeout 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err; echo bench=$?
tail -3 gpurun_out/bench_split.err
python -c "import json; d=json.load(open('gpurun_out/bench_split.json')); print(d['value'], d['e2e']['value'], d['config']['ef'], d['config']['rerank_percent'], d['roofline']['achieved'], d['recomputed_embeddings_per_s'])"
