set -u
mkdir -p gpurun_out
for r in 1 2; do for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_c4_t320.so tools/bin/libhc_c4_t256.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --no-naive --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done
