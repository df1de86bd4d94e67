CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dst_pass_kernel -s ${SKIP:-5} -c ${COUNT:-3} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_full.log
