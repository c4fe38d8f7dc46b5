set -u
mkdir -p gpurun_out
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_mlp_a3s4.so tools/bin/libhc_mlp_a3s3.so; do
  HC_LIB=$lib timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k mlp 2>&1 | tail -1
  HC_LIB=$lib timeout 300 python bench.py --config 5a --no-cpu-baseline --steps 50 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))' 2>&1)"
  HC_LIB=$lib timeout 100 python tools/mlp_trace.py 2>&1 | tail -1
done
