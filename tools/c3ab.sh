# A/B of K8 source-block sizes (with the default hot table) on C3 resident
B="python bench.py --config C3 --budget-gb 0 --pages 16 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
run() { tag=$1; shift; env "$@" $B > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err;
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', d['ms_per_step'], r.get('frac'), r.get('launch_ms'), r['gather_roofline']['frac'])" || tail -3 gpurun_out/ab_$tag.err; }
run blk32 SERAPH_PR_BLOCK_VERTS=33554432
run blk16 SERAPH_PR_BLOCK_VERTS=16777216
run blk22 SERAPH_PR_BLOCK_VERTS=22369622
run blk8 SERAPH_PR_BLOCK_VERTS=8388608
run hot4k_blk16 SERAPH_PR_BLOCK_VERTS=16777216 SERAPH_PR_HOT=4096
run hot1k SERAPH_PR_HOT=1024
