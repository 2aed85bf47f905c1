# out-of-core SSSP RMAT-26 under a 5 GB TOTAL budget (pages + adjacency), and C3 streamed
python bench.py --config C2 --scale 26 --pages 256 --window 4 --budget-gb 5 --mode baseline --steps 3 --warmup 1 > gpurun_out/ooc_sssp26.json 2> gpurun_out/ooc_sssp26.err
python -c "
import json; d=json.loads(open('gpurun_out/ooc_sssp26.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], json.dumps(d.get('device_footprint')), json.dumps(d['roofline']), d['parity'], d.get('e2e'))" || tail -20 gpurun_out/ooc_sssp26.err
python bench.py --config C3 --steps 2 --warmup 1 --no-e2e > gpurun_out/ooc_c3.json 2> gpurun_out/ooc_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/ooc_c3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], json.dumps(d.get('device_footprint')), json.dumps(d['roofline']), d['parity'])" || tail -20 gpurun_out/ooc_c3.err
