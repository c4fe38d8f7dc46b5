# MLP variant sweep: bench config 5a + the phase trace for each variant library.
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_mlp_*.so; do
  HC_LIB=$lib timeout 200 python bench.py --config 5a --no-cpu-baseline --steps ${STEPS:-400} > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')"
  HC_LIB=$lib timeout 100 python tools/mlp_trace.py 2>&1 | tail -1
done
