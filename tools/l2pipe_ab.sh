#!/bin/bash
# A/B of the n = 128 L2-resident solve pipeline (DPM_L2PIPE = fields per chunk; 0 = three 1 GiB passes)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 0 2 3 4 6; do
  DPM_L2PIPE=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-pks --no-dd > gpurun_out/l2p_$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/l2p_{c}.log") if l.startswith("{")][-1])
r = d["roofline"]
print(f"L2PIPE={c}: {d['value']:.0f} solves/s, {d['ms_per_step']:.3f} ms/step, passes " +
      ", ".join(f"{k}: {v['ms']/max(v['launches'],1):.3f} ms x{v['launches']}" for k, v in r["passes"].items()))
PY
done
DPM_L2PIPE=4 python -m pytest tests/test_gpu_parity.py -q -x -k "aux_solve_parity and 128 or cfg4_full" 2>&1 | tail -2
