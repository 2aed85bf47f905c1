#!/bin/bash
# Dev: A/B libseraph variants (variants/libseraph_<name>.so) on several bench configs.
# usage: bash tools/ab_lib.sh "C4|C2|C1|--config C2 --algo bfs ..." name1 name2 ...
CFGS=$1; shift
mkdir -p gpurun_out
IFS='|' read -ra CS <<< "$CFGS"
for r in 1 2; do for c in "${CS[@]}"; do for v in "$@"; do
  args="$c"; [[ "$c" != -* ]] && args="--config $c"
  tag=$(echo "$args" | tr -c 'A-Za-z0-9' _)
  SERAPH_LIB=$PWD/variants/libseraph_$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 $args > gpurun_out/ab_${tag}_${v}_$r.log 2>&1
  echo AB "$c" $v $r $(tail -1 gpurun_out/ab_${tag}_${v}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r.get('launch_ms'), r.get('frac'), d.get('parity',{}).get('fixpoint_violations'), d.get('parity',{}).get('bit_exact_vs_reference_run'))" 2>&1 | tail -1)
done; done; done
