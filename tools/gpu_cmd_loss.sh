set -u
mkdir -p gpurun_out
for lib in paper_2602_18741_b200/libhadacodec_b200.so ${LIBS:-tools/bin/libhc_loss_abreg.so}; do
  HC_LIB=$lib timeout 300 python -m pytest -q -x tests/test_gpu_loss_numerics.py tests/test_gpu_parity.py -k "loss or flat or trained" 2>&1 | tail -1
  HC_LIB=$lib timeout 300 python bench.py --config 5b --no-cpu-baseline --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))' 2>&1)"
done
