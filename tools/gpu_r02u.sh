#!/bin/bash
# After removing the experimental kernel variants: encoder/attention/fused GPU tests; then the
# L2 -> SM operand feed of every encoder kernel at the bench chunk size (ncu, one layer).
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_qkv_attn.py -q -x -rf > gpurun_out/enc_tests.log 2>&1; echo etests=$?; tail -2 gpurun_out/enc_tests.log
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -k regex:"tc_gemm_pair|qkv_attn_pair" -s 12 -c 8 --csv --log-file gpurun_out/l2feed.csv python tools/encode_fused.py 2048 1 1 > /dev/null 2>&1; echo ncu=$?
python tools/ncu_csv.py gpurun_out/l2feed.csv
