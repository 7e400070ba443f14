# kernel-level checks: attention parity (both kernels) + micro-benchmarks
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_encoder.py -x -q 2>&1 | tail -15
timeout 300 python tools/bench_attn.py 2048 256
timeout 300 python tools/bench_attn.py 4096 128
timeout 300 python tools/bench_gemm.py 524288
