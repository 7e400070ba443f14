#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/encode_split.py 2048 1 > gpurun_out/split_ab.txt 2>&1
python tools/encode_split.py 2048 0 >> gpurun_out/split_ab.txt 2>&1
for s in 1 0; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_gemm_pair --csv --log-file gpurun_out/split_launch_$s.csv python tools/encode_split.py 512 $s > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/split_launch_$s.csv >> gpurun_out/split_ab.txt
done
cat gpurun_out/split_ab.txt
