# PKS steps/s for PDL variants: trigger at kernel start (default build) / implicit trigger at block exit
# (-DDPM_PDL_TRIGGER=0), each with PDL inside the step graph for n <= 32 and n <= 64 (DPM_PDL_NMAX).
for trig in 1 0; do
  DPM_NVCC_EXTRA="-DDPM_PDL_TRIGGER=$trig" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)" > /dev/null || { echo build failed; continue; }
  for nmax in 32 64 0; do
    echo "trigger=$trig nmax=$nmax $(DPM_PDL_NMAX=$nmax python tools/pks_ab.py 2>/dev/null | tail -1)"
  done
done
python -m pytest tests/test_gpu_parity.py -x -q -k "pks or determin" 2>&1 | tail -1
