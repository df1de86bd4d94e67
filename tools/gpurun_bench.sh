set -x
free -g | head -2
nproc
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$?
cat gpurun_out/bench.log; tail -5 gpurun_out/bench.err
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks > gpurun_out/ncu1.log 2>&1
echo ncu1=$?
