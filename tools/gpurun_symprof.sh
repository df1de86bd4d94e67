cd $GRAFT_REPO_ROOT
SYM_CFGS=cfg4 timeout 300 python tools/sym_ab.py > gpurun_out/symp.log 2>&1; echo rc=$?; tail -2 gpurun_out/symp.log
SYM_CFGS=cfg4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sym_|potential_list" --csv --log-file gpurun_out/sym_launches.csv python tools/sym_ab.py > /dev/null 2>&1; echo ncu_rc=$?
python tools/ncu_csv_summary.py gpurun_out/sym_launches.csv 2>/dev/null | head -30 || head -30 gpurun_out/sym_launches.csv
SYM_CFGS=cfg4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sym_yz_kernel" -s 2 -c 1 -o gpurun_out/sym_yz_full python tools/sym_ab.py > /dev/null 2>&1; echo ncu_full_rc=$?
SYM_CFGS=cfg4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sym_x_kernel" -s 1 -c 1 -o gpurun_out/sym_x_full python tools/sym_ab.py > /dev/null 2>&1; echo ncu_full_rc=$?
