#!/bin/bash
# Dev: C4 under SERAPH_ROOT_DIAG_REPS (root-block diagonal sweeps)
for r in 4 5 6 7 8; do
  SERAPH_ROOT_DIAG_REPS=$r timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/rr.log 2>&1
  echo REPS $r $(tail -1 gpurun_out/rr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['fixpoint_violations'], d['passes']['total'])")
done
