# quick: n=128 parity + all aux-solve parity + cfg4 bench (no e2e/cpu/pks)
python -m pytest tests/test_gpu_parity.py -x -q -k "aux_solve or cfg4 or eigenfunction" 2>&1 | tail -2 > gpurun_out/quick_tests.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/bench_q.log 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" || tail -20 gpurun_out/bench_q.log
cat gpurun_out/quick_tests.log
