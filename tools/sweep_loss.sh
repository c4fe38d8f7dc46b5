# Loss kernel (config 5b) variant sweep over tools/bin/libhc_loss_*.so
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_loss_*.so; do
  HC_LIB=$lib timeout 200 python bench.py --config 5b --no-cpu-baseline --steps ${STEPS:-20} > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')"
done
