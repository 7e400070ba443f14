#!/bin/bash
# Secondary evidence with the final kernels: config-1 bench, 2-rank (gloo, one GPU) config-2 bench line.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py --config c1 --steps 2 --warmup 3 > gpurun_out/bench_c1_final.json 2> gpurun_out/bench_c1_final.err; echo c1=$?
tail -c 400 gpurun_out/bench_c1_final.json
LV_BENCH_BACKEND=gloo LV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --corpus-size 100000 --batch 1024 --steps 2 --warmup 3 --ef 113 --alphas 70 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo tworank=$?
tail -c 300 gpurun_out/bench_2rank_gloo.json
