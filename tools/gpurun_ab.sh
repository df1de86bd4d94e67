for cm in 224 1024 20000; do
DPM_CHUNK_MB=$cm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/b$cm.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b$cm.log').read().strip().splitlines()[-1]); r=d['roofline']
print('CHUNK_MB=$cm', round(d['value']), round(d['ms_per_step'],2), {k:(round(v['ms']/v['launches']*1e3,1), round(16*v['points']/v['launches']/(v['ms']/v['launches']/1e3)/1e12,2)) for k,v in r['passes'].items()})"
done
