# round-2 A/B: segmented merges (K1 BFS/CC, K8) + hot-staged K8 table sizes
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
j() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', d['ms_per_step'], r.get('frac'), r.get('launch_ms'), r['gather_roofline']['frac'])" || tail -3 ${1%.json}.err; }
for c in C4 C1 C2; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err; j gpurun_out/ab_$c.json
done
B="python bench.py --config C3 --budget-gb 0 --pages 16 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for v in "0 8" "1024 8" "2048 8" "4096 8" "4096 16"; do set -- $v
  SERAPH_PR_HOT=$1 SERAPH_PR_HOT_WARPS=$2 $B > gpurun_out/ab_pr_$1_$2.json 2> gpurun_out/ab_pr_$1_$2.err; j gpurun_out/ab_pr_$1_$2.json
done
