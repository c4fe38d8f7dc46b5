set -u
mkdir -p gpurun_out
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_chain_i128.so; do
HC_LIB=$lib timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "multibounce" 2>&1 | tail -1
done
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_chain_i128.so tools/bin/libhc_chain_v3smem.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))' 2>&1)"
done
HC_LIB=tools/bin/libhc_chain_i128.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_latent_v3 -s 3 -c 1 -o gpurun_out/chain_v3r -f python bench.py --config 4 --plain --no-cpu-baseline --steps 4 --warmup 0 > gpurun_out/ncu_chain.log 2>&1; echo "ncu rc=$?"
