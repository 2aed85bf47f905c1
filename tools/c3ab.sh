# A/B of K8 variants on C3 resident (RMAT-26, 16 pages)
python -m pytest tests/test_engine_gpu.py -q -x -k "pagerank or out_of_core or streaming" > gpurun_out/pr_tests.log 2>&1; tail -3 gpurun_out/pr_tests.log
B="python bench.py --config C3 --budget-gb 0 --pages 16 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
run() { tag=$1; shift; env "$@" $B > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err;
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', d['ms_per_step'], r.get('frac'), r.get('launch_ms'), r['gather_roofline']['frac'])" || tail -3 gpurun_out/ab_$tag.err; }
run nohot SERAPH_PR_HOT=0
run nohot_unblk SERAPH_PR_HOT=0 SERAPH_PR_BLOCK_VERTS=0
for w in 8 16 32; do for h in 2048 8192; do
  run w${w}_h${h} SERAPH_PR_HOT_WARPS=$w SERAPH_PR_HOT=$h
done; done
run w32_h16384 SERAPH_PR_HOT_WARPS=32 SERAPH_PR_HOT=16384
