for cfg in "1 1024" "2 64" "2 128" "2 256" "1 64"; do set -- $cfg
DPM_STREAMS=$1 DPM_CHUNK_MB=$2 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/b.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('streams=$1 chunkMB=$2', round(d['value']), round(d['ms_per_step'],2))"
done
