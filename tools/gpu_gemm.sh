python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_encoder.py -x -q 2>&1 | tail -5
timeout 300 python tools/bench_gemm.py 524288
timeout 300 python tools/bench_gemm.py 100000
