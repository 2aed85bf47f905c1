#!/bin/bash
# Dev: A/B libseraph variants (variants/libseraph_<name>.so) on the C2 bench.
# usage: bash tools/ab_variants.sh "<bench args>" name1 name2 ...
ARGS=$1; shift
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
  SERAPH_LIB=$PWD/variants/libseraph_$v.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 $ARGS > gpurun_out/ab_${v}_$r.log 2>&1
  echo AB $v $r $(tail -1 gpurun_out/ab_${v}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('launch_ms'))")
done; done
