# Steady-state DRAM traffic of each config's hot kernel: launches 20..35 of a back-to-back
# --plain run under `ncu --cache-control none` (no flush between launches), so the dirty
# output lines a launch leaves in L2 are written back during the following launches and are
# counted.  -> gpurun_out/traffic_c<cfg>.csv (one row per launch)
set -u
for c in ${CONFIGS:-2 3 1 5b 5a 4}; do
  case $c in 5a) K=regex:mlp_kernel;; 4) K=regex:chain;; *) K=regex:tile_pipeline;; esac
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --cache-control none --clock-control none -k $K -s 20 -c 16 --csv --log-file gpurun_out/traffic_c$c.csv \
    python bench.py --config $c --plain --steps 40 --warmup 0 > gpurun_out/traffic_c$c.log 2>&1
  echo "traffic c$c rc=$?"
done
