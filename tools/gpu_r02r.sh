#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python tools/encode_modes.py 2048 0,8,4,12
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qkv_attn_pair -s 2 -c 1 -o gpurun_out/r02_qkv_attn_fused python tools/encode_fused.py 2048 1 1 > /dev/null 2>&1; echo ncu=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc_gemm_pair_kernel<6>" -s 2 -c 1 -o gpurun_out/r02_gemm_oproj python tools/encode_fused.py 2048 1 1 > /dev/null 2>&1; echo ncu2=$?
python tools/ncu_metrics.py gpurun_out/r02_qkv_attn_fused.ncu-rep | grep -E "duration|tensor_cycles_active.avg|dram__bytes|lts__throughput"
python tools/ncu_metrics.py gpurun_out/r02_gemm_oproj.ncu-rep | grep -E "duration|tensor_cycles_active.avg|dram__bytes|lts__throughput|dram__throughput"
