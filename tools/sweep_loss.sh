# Loss kernel (config 5b) variant sweep over tools/bin/libhc_loss_*.so: value (M pairs/s),
# HBM fraction, and the loss parity tests under each variant.
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_loss_*.so; do
  HC_LIB=$lib timeout 200 python bench.py --config 5b --no-cpu-baseline --steps ${STEPS:-20} > gpurun_out/sw.log 2>&1
  r=$(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))' 2>&1)
  t=$(HC_LIB=$lib timeout 300 python -m pytest -q -x tests/test_gpu_loss_numerics.py tests/test_gpu_parity.py -k loss 2>&1 | tail -1)
  echo "$lib $r | $t"
done
