set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "multibounce or config4 or c4 or chain" 2>&1 | tail -1
for r in 1 2; do for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_c4_stg.so tools/bin/libhc_c4_old.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --no-naive --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_latent_v3 -s 3 -c 1 -o gpurun_out/full_c4 -f python bench.py --config 4 --plain --no-cpu-baseline --no-naive --steps 4 --warmup 0 > gpurun_out/ncu_chain.log 2>&1; echo "ncu rc=$?"
