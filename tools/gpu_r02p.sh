#!/bin/bash
# Fused QKV + attention, 4-stage ring: parity, encoder A/B, ncu of fused vs unfused QKV GEMM.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_qkv_attn.py -q -x -rf > gpurun_out/qkv_tests.log 2>&1; echo qtests=$?
tail -3 gpurun_out/qkv_tests.log
grep -q failed gpurun_out/qkv_tests.log && exit 1
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -x > gpurun_out/enc_tests.log 2>&1; echo etests=$?; tail -2 gpurun_out/enc_tests.log
for f in 0 1 0 1; do timeout 300 python tools/encode_fused.py 2048 $f 3 2>&1 | tail -1; done
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
timeout 300 ncu --metrics $M --clock-control none -k regex:qkv_attn_pair -s 2 -c 2 --csv --log-file gpurun_out/qa_fused.csv python tools/encode_fused.py 512 1 1 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --metrics $M --clock-control none -k regex:"tc_gemm_pair|attn_tc" -s 8 -c 8 --csv --log-file gpurun_out/qa_unfused.csv python tools/encode_fused.py 512 0 1 > /dev/null 2>&1; echo ncu2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qkv_attn_pair -s 2 -c 1 -o gpurun_out/qa_fused_full python tools/encode_fused.py 512 1 1 > /dev/null 2>&1; echo ncu3=$?
python tools/ncu_csv.py gpurun_out/qa_fused.csv
python tools/ncu_csv.py gpurun_out/qa_unfused.csv
python tools/ncu_metrics.py gpurun_out/qa_fused_full.ncu-rep
