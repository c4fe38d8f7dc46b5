# Tuning sweep over variant builds (python -m paper_2602_18741_b200.build -D ... --out tools/bin/libhc_X.so).
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_*.so; do
  HC_LIB=$lib timeout 200 python bench.py --config ${CFG:-2} --no-cpu-baseline --no-naive --steps ${STEPS:-2000} > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')"
done
