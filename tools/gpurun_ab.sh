for tc in 64 32; do
DPM_TC128=$tc python -m pytest tests/test_gpu_parity.py -x -q -k "aux_solve_parity and 128 or cfg4" 2>&1 | tail -1
DPM_TC128=$tc python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/bench_tc$tc.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_tc$tc.log').read().strip().splitlines()[-1]); print('TC=$tc', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fp64']['frac'])"
done
