for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_chainspec_*.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 8 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["naive_n81"]["value"],1))')"
done
