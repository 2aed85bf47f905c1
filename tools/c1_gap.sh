#!/bin/bash
# Dev: C1 (BFS RMAT-20) per-run kernel list vs the device-timed step: the host gap
mkdir -p gpurun_out/c1gap
timeout 600 python tools/pass_probe.py --algo bfs --scale 20 --reps 5 > gpurun_out/c1gap/probe.txt 2>&1
timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1gap/launches.csv python tools/pass_probe.py --algo bfs --scale 20 --reps 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/c1gap/launches.csv --full > gpurun_out/c1gap/table.txt 2>&1
tail -25 gpurun_out/c1gap/table.txt; tail -12 gpurun_out/c1gap/probe.txt
