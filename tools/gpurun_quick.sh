python -m pytest tests/test_gpu_parity.py -x -q -k "aux_solve or eigenfunction or cfg4" 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/bench_q.log 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['fp64'])"
if [ "$1" = "ncu" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks > /dev/null 2>&1; echo ncu=$?
fi
