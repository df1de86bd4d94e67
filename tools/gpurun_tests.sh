set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -m pytest tests/test_gpu_parity.py -x -q -k "aux_solve_parity" 2>&1 | tail -30 > gpurun_out/t1.log
cat gpurun_out/t1.log
python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -40 > gpurun_out/t2.log
cat gpurun_out/t2.log
