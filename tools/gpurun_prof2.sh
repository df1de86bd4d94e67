# launch list without cache flush (L2 state carries across kernels) + ncu full of one kernel
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --cache-control none --clock-control none -k regex:"${LREGEX:-dst128|ztri|dst_pass|plane}" -c 10 --csv --log-file gpurun_out/launches_nc.csv $CMD > /dev/null 2>&1; echo ncu_list=$?
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-dst128_pass_kernel} -s ${SKIP:-4} -c ${COUNT:-2} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
