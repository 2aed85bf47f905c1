#!/bin/bash
# Dev: per-launch K1 times of one C4 run for libseraph variants
mkdir -p gpurun_out/abl
for v in "$@"; do
SERAPH_LIB=$PWD/variants/libseraph_$v.so timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/abl/$v.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/abl/$v.txt 2>&1
echo "== $v"; python tools/launch_table.py gpurun_out/abl/$v.csv --full 2>&1 | head -16
done
