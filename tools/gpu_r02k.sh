#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
bash tools/gpu_chunk.sh > gpurun_out/chunk_sweep.txt 2>&1; cat gpurun_out/chunk_sweep.txt
# full ncu captures of one split-residual O-projection (kMode 6), one FFN2 (kMode 5) and one
# plain GEMM (kMode 0) of a 512 x 256-token BERT-base encode (launch order per layer: QKV,
# O-proj, FFN1, FFN2 -> launches 1, 3, 2 of the second layer = indices 5, 7, 6)
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair -s 5 -c 3 -o gpurun_out/r02_gemm_layer2 -f python tools/encode_split.py 512 1 > gpurun_out/ncu_gemm_r02.log 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/r02_attn -f python tools/encode_split.py 512 1 >> gpurun_out/ncu_gemm_r02.log 2>&1; echo ncu2=$?
ls -la gpurun_out/*.ncu-rep
