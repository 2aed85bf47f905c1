# C4 e2e legs (pinned + pageable through the stager), stager knobs
for v in "8 32" "12 32" "16 32" "12 64"; do set -- $v
SERAPH_STAGE_THREADS=$1 SERAPH_STAGE_CHUNK_MB=$2 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_c4_$1_$2.json 2> gpurun_out/e2e_c4_$1_$2.err
python -c "
import json; d=json.loads(open('gpurun_out/e2e_c4_$1_$2.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$v', d['ms_per_step'], e['seconds_per_step'], e['upload_seconds'], e['pageable'])" || tail gpurun_out/e2e_c4_$1_$2.err
done
