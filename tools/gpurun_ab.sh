# A/B of compile-time variants: for each "name|flags" in $VARIANTS, rebuild libdpm.so with
# DPM_NVCC_EXTRA=flags, run the n=128 parity subset and a short bench; prints value + plane ms.
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%|*}"; flags="${v#*|}"
  DPM_NVCC_EXTRA="$flags" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)" || { echo "$name build failed"; continue; }
  python -m pytest tests/test_gpu_parity.py -x -q -k "aux_solve_parity_large_dt or plane_kernels or chunked_inplace" > gpurun_out/ab_$name.t 2>&1
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
t = open(f"gpurun_out/ab_{name}.t").read().strip().splitlines()[-1]
try:
    d = json.loads(open(f"gpurun_out/ab_{name}.log").read().strip().splitlines()[-1])
    print(f"AB {name}: {d['value']:.0f} solves/s plane {d['roofline']['passes']['y']['ms'] / max(1, d['roofline']['passes']['y']['launches']):.4f} ms/launch | {t}")
except Exception as e:
    print(f"AB {name}: failed {e} | {t}")
PY
done
