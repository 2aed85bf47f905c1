#!/bin/bash
# Dev: ncu evidence for the C2 headline (launch list of the bench command +
# one --set full capture of the three dense K1 launches of a converge run).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:pull_relax -s 3 -c 3 -o gpurun_out/k1_sssp_s24 -f python tools/profile_sweep.py --converge 2 --reps 1 > gpurun_out/ncu_k1.log 2>&1
echo done
