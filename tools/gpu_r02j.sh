#!/bin/bash
# 2-rank bench (gloo on one GPU: the multi-rank path with query shards, gather, max-over-ranks)
# and the corpus-geometry probe behind DESIGN.md's corpus deviation.
python -c "import __graft_entry__ as g; g.build()" || exit 1
LV_BENCH_BACKEND=gloo LV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --n 100000 --batch 1024 --steps 2 --warmup 1 --ef 96 --alphas 70 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo tworank=$?
tail -2 gpurun_out/bench_2rank_gloo.err
timeout 900 python tools/probe_geometry.py 100000 bert-base 256 > gpurun_out/probe_geometry_uniform_bert.txt 2>&1; echo probe=$?
cat gpurun_out/probe_geometry_uniform_bert.txt | grep -v Warn | head -20
LV_TRACE_ITERS=1 timeout 1500 python bench.py --steps 1 --warmup 1 --ef 114 --alphas 70 --no-cpu-baseline --no-e2e > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err; echo trace=$?
grep -c "\[lv\] iter" gpurun_out/bench_trace.err
