set -u
mkdir -p gpurun_out
for r in 1 2; do for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_c4_shflonly.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --no-naive --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done
timeout 900 python bench.py --verify --config 4 > gpurun_out/verify4.log 2>&1; echo "verify4 rc=$?"; tail -2 gpurun_out/verify4.log | cut -c1-600
for mix in "339738624 390070272" "74649600 49766400" "1094860800 2786918400" "10871635968 0" "201326592 402653184"; do tools/bin/rw_ceiling $mix 20; done
