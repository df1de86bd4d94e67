# A/B of compile-time variants on the PKS step: for each "name|flags" in $VARIANTS rebuild libdpm.so,
# run the small-n parity subset ($TESTS) and tools/pks_ab.py (cfg2 / cfg3 steps/s).
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%|*}"; flags="${v#*|}"
  DPM_NVCC_EXTRA="$flags" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "$name build failed"; continue; }
  if [ -n "$TESTS" ]; then python -m pytest tests/test_gpu_parity.py -x -q -k "$TESTS" 2>&1 | tail -1; fi
  echo "PKS $name: $(python tools/pks_ab.py 2>&1 | tail -1)"
done
