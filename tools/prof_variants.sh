# ncu --set full (with source) of the FACR plane pass for compile-time variants "name|flags;..."
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%|*}"; flags="${v#*|}"
  DPM_NVCC_EXTRA="$flags" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "$name build failed"; continue; }
  CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-pks --no-dd"
  $CMD > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-plane128_facr} -s 2 -c 1 -o gpurun_out/prof_$name $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name ncu=$?"
done
