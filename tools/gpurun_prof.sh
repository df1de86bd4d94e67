# ncu --set full of one kernel (regex $KREGEX), after the plain command exits 0
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-dst128_pass_kernel} -s ${SKIP:-4} -c ${COUNT:-2} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_full.log
