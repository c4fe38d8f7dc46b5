# Naive shading legs of configs 2 and 3 over variant libraries
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_naive_*.so; do
  for c in 2 3; do
    HC_LIB=$lib timeout 300 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-40} > gpurun_out/sw.log 2>&1
    echo "$lib c$c $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["naive_n81"]["value"],1))')"
  done
done
