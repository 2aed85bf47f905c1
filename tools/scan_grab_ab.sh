#!/bin/bash
# Dev: gate-scan unroll variants x unblocked K1 grab size on C4 (+C1)
for r in 1 2; do for v in s1 s4 s8; do for g in 8 32; do
  SERAPH_K1_GRAB=$g SERAPH_LIB=$PWD/variants/libseraph_$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/sg.log 2>&1
  echo SG $v $g $(tail -1 gpurun_out/sg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['fixpoint_violations'])")
done; done; done
for v in s1 s4; do
  SERAPH_K1_GRAB=32 SERAPH_LIB=$PWD/variants/libseraph_$v.so timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abl/sg_$v.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > /dev/null 2>&1
  echo "== $v"; python tools/launch_table.py gpurun_out/abl/sg_$v.csv --full 2>&1 | grep pull_relax | head -12
done
