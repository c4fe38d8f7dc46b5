set -u
mkdir -p gpurun_out
for lib in paper_2602_18741_b200/libhadacodec_b200.so ${LIBS:-}; do
  HC_LIB=$lib timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "multibounce" 2>&1 | tail -1
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 10 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); n=d["naive_n81"]; print(round(d["value"]), round(d["roofline"]["frac"],3), "naive", round(n["value"],1), round(n["roofline"]["frac"],3))' 2>&1)"
done
