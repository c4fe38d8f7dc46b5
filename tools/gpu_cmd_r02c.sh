set -u
for lib in paper_2602_18741_b200/libhadacodec_b200.so tools/bin/libhc_naive_t512.so tools/bin/libhc_naive_t1024.so; do
  HC_LIB=$lib timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-k9 --no-parity > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["naive_n81"]["value"]), round(d["naive_n81"]["roofline"]["frac"],3))' 2>&1)"
done
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:LossOp -s 1 -c 1 -o gpurun_out/loss_r02 -f python bench.py --config 5b --no-cpu-baseline --steps 2 --warmup 0 --plain > gpurun_out/ncu_loss.log 2>&1; echo "ncu loss rc=$?"
timeout 300 python bench.py --config 5b --no-cpu-baseline --steps 20 > gpurun_out/b5b.log 2>&1; tail -1 gpurun_out/b5b.log | cut -c1-300
timeout 300 python bench.py --config 1 --no-cpu-baseline --steps 20 > gpurun_out/b1.log 2>&1; tail -1 gpurun_out/b1.log | cut -c1-300
timeout 300 python bench.py --config 5a --no-cpu-baseline --steps 20 > gpurun_out/b5a.log 2>&1; tail -1 gpurun_out/b5a.log | cut -c1-300
