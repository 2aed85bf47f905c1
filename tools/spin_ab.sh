#!/bin/bash
# Dev: pass-result waits by spinning on pinned words vs stream sync
for r in 1 2; do for c in C1 C2 "C1 --algo sssp" "C1 --algo cc"; do for e in 1 0; do
  SERAPH_NO_SPIN=$e timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/sp.log 2>&1
  echo SPIN "$c" no_spin=$e $(tail -1 gpurun_out/sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('wall_ms_per_step'), d['parity']['fixpoint_violations'])")
done; done; done
