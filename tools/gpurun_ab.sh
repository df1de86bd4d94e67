for cm in 64 80 96 112; do
DPM_CHUNK_MB=$cm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/b$cm.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b$cm.log').read().strip().splitlines()[-1]); print('CHUNK_MB=$cm', d['value'], d['ms_per_step'])"
done
