# C4: stage timings of the e2e call (source-block build) + launch list of one run
SERAPH_TIMING=1 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c4t.json 2> gpurun_out/c4t.err
grep seraph gpurun_out/c4t.err | tail -30
python -c "
import json; d=json.loads(open('gpurun_out/c4t.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e']))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_table.py gpurun_out/c4_launches.csv 2>&1 | tail -40
