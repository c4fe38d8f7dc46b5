timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loss_numerics.py tests/test_gpu_metrics.py -x -q > gpurun_out/t_pipe.log 2>&1; tail -2 gpurun_out/t_pipe.log
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_pipe0.so; do
  for c in 2 1 3 5b; do
    HC_LIB=$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-naive --no-k9 --no-parity --steps 40 > gpurun_out/sw.log 2>&1
    echo "$lib c$c $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])' 2>&1)"
  done
done
