#!/bin/bash
# Dev: K1 LIST threshold (gathers / edges of the previous dense pass or block)
for r in 1 2; do for c in C4 C1 "C1 --algo cc" "C1 --algo bfs --uniform --scale 22"; do for f in 0.3 0.6 0.9; do
  SERAPH_LIST_FRAC=$f timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/lf.log 2>&1
  echo LF "$c" $f $(tail -1 gpurun_out/lf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['fixpoint_violations'])")
done; done; done
