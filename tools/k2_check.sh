python -m pytest tests/test_engine_gpu.py -x -q -k "modes or mode_independence or predictors or reentry or streaming or loopback or group" > gpurun_out/k2_tests.log 2>&1; tail -2 gpurun_out/k2_tests.log
for k in 0 1; do
  if [ $k = 1 ]; then export SERAPH_NO_K2=1; fi
  python bench.py --config C2 --mode reentry --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k2_c2_$k.json 2> gpurun_out/k2_c2_$k.err
  python -c "
import json; d=json.loads(open('gpurun_out/k2_c2_$k.json').read().strip().splitlines()[-1]); print('noK2=$k', d['ms_per_step'], d['passes'], d['gpu_launches'])" || tail -3 gpurun_out/k2_c2_$k.err
done
