for c in cfg3 cfg2; do
python tools/pks_cfg_launches.py $c 10
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/pks_${c}_warm.csv python tools/pks_cfg_launches.py $c 10 > /dev/null 2>&1; echo ncu=$?
done
