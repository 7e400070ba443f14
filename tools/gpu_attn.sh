python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_encoder.py -x -q -k attention 2>&1 | tail -3
timeout 300 python tools/bench_attn.py 2048 256
timeout 300 python tools/bench_attn.py 4096 128
bash tools/ncu_c2.sh
python tools/summarize_launches.py gpurun_out/launches_c2.csv
