# full ncu captures of the encoder's top kernels at config-2 shapes (micro-benchmarks)
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair -s 3 -c 1 -o gpurun_out/prof_gemm_qkv -f python tools/bench_gemm.py 131072 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair -s 14 -c 1 -o gpurun_out/prof_gemm_out -f python tools/bench_gemm.py 131072 >> gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/prof_attn_tc -f python tools/bench_attn.py 1024 256 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
