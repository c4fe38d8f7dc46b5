# Round-end refresh: bench lines of every config, the default launch list, ncu --set full of
# the hot kernel of the configs given in $FULL (default "2 3").  Outputs under gpurun_out/.
set -u
for c in ${CONFIGS:-1 2 3 4 5a 5b}; do
  timeout 600 python bench.py --config $c > gpurun_out/final_c$c.json 2> gpurun_out/final_c$c.err; echo "bench c$c rc=$?"
done
if [ "${LAUNCHES:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 16 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_default.log 2>&1; echo "launches rc=$?"
fi
for c in ${FULL:-2 3}; do
  case $c in 5a) K=regex:mlp_kernel;; 4) K=regex:chain;; 6) K=regex:de76;; 7) K=regex:render_samples;; 8|9) K=regex:line_parse;; 10) K=regex:grad_reduce;; *) K=regex:tile_pipeline;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k $K -s 2 -c 1 -f -o gpurun_out/full_c$c \
    python bench.py --config $c --plain --steps 4 > gpurun_out/ncu_full_c$c.log 2>&1; echo "ncu full c$c rc=$?"
done
