#!/bin/bash
# Dev: refresh the evidence of the committed state (one GPU): launch list of
# the default bench command, per-launch table of one C4 run, one --set full
# capture of every K1 launch of a C4 run, the reference arm, C1/C2/C3 lines.
mkdir -p gpurun_out/fin
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_bench.log 2>&1
echo launches rc=$?
timeout 600 $NCU --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin/c4_run.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/fin/c4_run.txt 2>&1
echo run rc=$?
timeout 1500 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:pull_relax -c 10 -o gpurun_out/fin/c4_k1_full -f python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/fin/ncu_full.log 2>&1
echo full rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/ref_arm.log 2>&1
echo ref rc=$?
tail -1 gpurun_out/fin/ref_arm.log > gpurun_out/fin/ref_arm.json
timeout 600 python bench.py --config C1 > gpurun_out/fin/c1.json 2> gpurun_out/fin/c1.err; echo c1 rc=$?
timeout 600 python bench.py --config C2 > gpurun_out/fin/c2.json 2> gpurun_out/fin/c2.err; echo c2 rc=$?
timeout 900 python bench.py --config C3 --budget-gb 0 --pages 16 --steps 3 --warmup 3 > gpurun_out/fin/c3res.json 2> gpurun_out/fin/c3res.err; echo c3 rc=$?
