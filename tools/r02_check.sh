python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
SERAPH_TIMING=1 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4e.json 2> gpurun_out/c4e.err
grep "seraph\] src blocks finish" gpurun_out/c4e.err | tail -3
python -c "
import json; d=json.loads(open('gpurun_out/c4e.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e']))" || tail gpurun_out/c4e.err
python bench.py --config C3 --budget-gb 0 --pages 16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3e.json 2> gpurun_out/c3e.err
python -c "
import json; d=json.loads(open('gpurun_out/c3e.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e']))" || tail gpurun_out/c3e.err
