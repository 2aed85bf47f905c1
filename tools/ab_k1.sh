# K1 A/B on C4 / C2 / C1 (device time per converge run)
python -m pytest tests/test_engine_gpu.py -x -q -k "rmat or fixpoint or mode or pred or blocked or golden or scale20" > gpurun_out/k1_tests.log 2>&1; tail -2 gpurun_out/k1_tests.log
for c in C4 C2 C1; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abk_$c.json 2> gpurun_out/abk_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/abk_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', d['ms_per_step'], r['frac'], r['launch_ms'])" || tail -3 gpurun_out/abk_$c.err
done
