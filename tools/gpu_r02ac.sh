#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
LV_BENCH_BACKEND=gloo LV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config c2 --corpus-size 100000 --batch 1024 --steps 1 --warmup 3 --alphas 70 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank_tune.json 2> gpurun_out/bench_2rank_tune.err; echo tworank=$?
grep -E "chosen" gpurun_out/bench_2rank_tune.err | head -4
tail -c 300 gpurun_out/bench_2rank_tune.json
