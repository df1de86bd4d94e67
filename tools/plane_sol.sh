# Speed-of-light A/B of the FACR plane pass: rebuild with each PLANE_SOL_* switch (wrong results,
# timing only) and print the plane-pass ms per 64-field launch from a short cfg4 bench.
VARIANTS=${VARIANTS:-"base|;noload|-DPLANE_SOL_NOLOAD=1;nostore|-DPLANE_SOL_NOSTORE=1;nols|-DPLANE_SOL_NOLOAD=1 -DPLANE_SOL_NOSTORE=1;nop1|-DPLANE_SOL_NOP1=1;noxf|-DPLANE_SOL_NOXF=1;nop3|-DPLANE_SOL_NOP3=1;nop5|-DPLANE_SOL_NOP5=1"}
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%|*}"; flags="${v#*|}"
  DPM_NVCC_EXTRA="$flags" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "$name build failed"; continue; }
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/sol_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sol_{name}.log").read().strip().splitlines()[-1])
    y = d['roofline']['passes']['y']
    print(f"SOL {name}: plane {y['ms'] / max(1, y['launches']):.4f} ms/launch, {d['value']:.0f} solves/s")
except Exception as e:
    print(f"SOL {name}: failed {e}")
PY
done
