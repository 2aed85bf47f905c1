#!/bin/bash
# Dev: refresh the C4 evidence of the committed state (one GPU):
# launch list of the default bench command, per-launch table of one C4 run,
# one --set full capture of the heavy K1 launches, the reference arm line.
mkdir -p gpurun_out/fin
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_bench.log 2>&1
echo launches rc=$?
timeout 600 $NCU --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin/c4_run.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/fin/c4_run.txt 2>&1
echo run rc=$?
timeout 1200 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:pull_relax -c 6 -o gpurun_out/fin/c4_k1_full -f python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/fin/ncu_full.log 2>&1
echo full rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/ref_arm.log 2>&1
echo ref rc=$?
tail -1 gpurun_out/fin/ref_arm.log > gpurun_out/fin/ref_arm.json
