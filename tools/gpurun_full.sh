# Full check on one B200: GPU tests, smoke, default bench, reference arm, ncu launch list of the
# bench command and one full capture of the dominant kernel (the FACR plane pass).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.log; tail -5 gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref_rc=$?
cat gpurun_out/bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dst128|ztri|plane" -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"plane128_facr" -s 2 -c 1 -o gpurun_out/prof_full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
