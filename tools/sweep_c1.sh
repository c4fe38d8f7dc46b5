for r in 1 2; do for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_c1_*.so; do
  HC_LIB=$lib timeout 200 python bench.py --config 1 --no-cpu-baseline --no-naive --steps ${STEPS:-800} > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],4), d["ms_per_step_dist"]["p50"])')"
done; done
