cd $GRAFT_REPO_ROOT
timeout 300 python tools/sym_ab.py gpurun_out/sym1 > gpurun_out/sym1.log 2>&1; echo rc=$?; cat gpurun_out/sym1.log | tail -5
DPM_BEP_SYM=${SYM0:-0} timeout 300 python tools/sym_ab.py gpurun_out/sym0 > gpurun_out/sym0.log 2>&1; echo rc=$?; tail -3 gpurun_out/sym0.log
python - <<'PY'
import numpy as np
for c in ("cfg1","cfg2","cfg3","cfg4"):
    for w in ("pg","b","coef","ug"):
        try:
            a=np.load(f"gpurun_out/sym1_{c}_{w}.npy"); b=np.load(f"gpurun_out/sym0_{c}_{w}.npy")
            print(c,w,a.shape, float(np.abs(a-b).max()/np.abs(b).max()))
        except Exception as e: print(c,w,e)
PY
rm -f gpurun_out/sym*_*.npy
