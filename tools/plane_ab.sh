# n=128 plane-pass parity subset + two short cfg4 bench runs; prints value and plane ms per launch
python -m pytest tests/test_gpu_parity.py -x -q -k "plane_kernels or chunked_inplace or aux_solve_parity_large_dt" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/pab_$i.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/pab_$i.log').read().strip().splitlines()[-1]); y=d['roofline']['passes']['y']; x=d['roofline']['passes']['x']; print('run $i', round(d['value']), 'plane', y['ms']/y['launches'], 'x', x['ms']/x['launches'], d['roofline']['frac'])"; done
