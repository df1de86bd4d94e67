cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_dd_full.py tests/test_gpu_dd_case1.py -x -q > gpurun_out/dd_tests.log 2>&1; echo rc=$?
tail -4 gpurun_out/dd_tests.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/bench_dd.log 2>gpurun_out/bench_dd.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_dd.log').readline()); print(json.dumps(d.get('dd'))[:700])"
