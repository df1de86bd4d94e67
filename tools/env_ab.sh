# A/B of runtime switches: for each "name|ENV=val ..." in $VARIANTS run a short cfg4 bench with that
# environment (after an optional parity subset with $TESTS) and print value + plane ms per launch.
python -c "from paper_1811_03557_b200 import build as B; B.build()" > /dev/null 2>&1
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%|*}"; envs="${v#*|}"
  if [ -n "$TESTS" ]; then env $envs python -m pytest tests/test_gpu_parity.py -x -q -k "$TESTS" 2>&1 | tail -1; fi
  env $envs python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/env_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/env_{name}.log").read().strip().splitlines()[-1])
    y = d['roofline']['passes']['y']; x = d['roofline']['passes']['x']
    print(f"ENV {name}: {d['value']:.0f} solves/s plane {y['ms'] / max(1, y['launches']):.4f} ms/launch x {x['ms'] / max(1, x['launches']):.4f}")
except Exception as e:
    print(f"ENV {name}: failed {e}")
PY
done
