cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "bep_columns or pks or projection or build" > gpurun_out/symtests.log 2>&1; echo rc=$?
tail -15 gpurun_out/symtests.log
