#!/bin/bash
# Dev: re-measure the bench lines committed under profiles/ (one GPU).
mkdir -p gpurun_out/lines
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/lines/$name.log 2>&1; tail -1 gpurun_out/lines/$name.log > gpurun_out/lines/$name.json; echo "$name rc=$?"; }
run r01_bench_line
run r01_bench_c2_reference_arm --impl reference --steps 3 --warmup 3
run r01_bench_c1_bfs20 --algo bfs --scale 20
run r01_bench_c4_cc_uniform27 --algo cc --uniform --scale 27 --steps 5
run r01_bench_sssp26_resident --scale 26 --steps 5
run r01_bench_sssp26_streamed --scale 26 --pages 256 --window 4 --budget-gb 5 --steps 3 --no-cpu-baseline --no-e2e
