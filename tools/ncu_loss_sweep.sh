# ncu counters of the loss kernel (config 5b) for each tools/bin/libhc_loss_*.so variant
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,idc__request_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_loss_*.so; do
  echo "== $lib"
  HC_LIB=$lib timeout 300 ncu --metrics $M --clock-control none -k regex:tile_pipeline -s 2 -c 1 --csv python bench.py --config 5b --no-cpu-baseline --steps 3 --warmup 0 --plain 2>/dev/null | grep -E '"(gpu__|dram__|l1tex__|idc__|smsp__|sm__)' | awk -F'","' '{print $(NF-2), $NF}'
done
