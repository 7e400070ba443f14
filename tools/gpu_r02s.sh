#!/bin/bash
# Search-level parity of the fused kernel, then the config-3 / config-5 sweep at 10M with the fused encoder.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_qkv_attn.py -q -x -rf > gpurun_out/qkv_tests.log 2>&1; echo qtests=$?; tail -3 gpurun_out/qkv_tests.log
timeout 3300 python bench.py --config c3 --batch 4096 --steps 1 --warmup 1 --alphas 75 --ef-max 512 --no-cpu-baseline --no-e2e --batch-sweep 1024,4096,16384 > gpurun_out/bench_c3_fused.json 2> gpurun_out/bench_c3_fused.err; echo c3=$?
grep sweep gpurun_out/bench_c3_fused.err | tail -5
