set -u
for lib in tools/bin/libhc_mlp_noepi.so tools/bin/libhc_mlp_noepi4.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 5a --no-cpu-baseline --steps 50 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])' 2>&1)"
  HC_LIB=$lib timeout 100 python tools/mlp_trace.py 2>&1 | tail -1
done
