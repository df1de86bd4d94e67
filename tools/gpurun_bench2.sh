# Bench line, reference arm, the launch list of the headline bench and ncu captures of the dominant kernel
# (plane128_facr) and of the octant BEP path's yz GEMM pass.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dst128|ztri|plane" -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-pks > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
SYM_CFGS=cfg4 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sym_|potential_list|permute|scatter_|gram|chol|gemm_tri|rinv|colnorm|scale_cols|trmm|rdinv" --csv --log-file gpurun_out/sym_launches.csv python tools/sym_ab.py > /dev/null 2>&1; echo ncu_sym_rc=$?
SYM_CFGS=cfg4 ncu --set full --clock-control none --import-source on -k regex:"sym_yz_kernel" -s 2 -c 1 -o gpurun_out/sym_yz_full python tools/sym_ab.py > /dev/null 2>&1; echo ncu_full_rc=$?
