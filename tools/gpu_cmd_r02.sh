# round-2 measurement batch (see profiles/r02/README.md)
set -x
for lib in tools/bin/libhc_mlp2_bf16.so tools/bin/libhc_mlp2_f32.so paper_2602_18741_b200/libhadacodec_b200.so; do
  HC_LIB=$lib timeout 300 python bench.py --config 5a --no-cpu-baseline --steps 20 > gpurun_out/sw.log 2>&1
  echo "$lib $(tail -1 gpurun_out/sw.log | cut -c1-120)"
  HC_LIB=$lib timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k mlp 2>&1 | tail -1
done
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/b4.log 2>&1; tail -1 gpurun_out/b4.log | cut -c1-400
timeout 600 python bench.py --config 3 --no-cpu-baseline --steps 20 > gpurun_out/b3.log 2>&1; tail -1 gpurun_out/b3.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b2.log 2>&1; tail -1 gpurun_out/b2.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_latent_rep -c 1 -o gpurun_out/chain -f python bench.py --config 4 --no-cpu-baseline --steps 1 --warmup 0 --plain > gpurun_out/ncu_chain.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ShadeSpectralF2 -c 1 -o gpurun_out/naive2 -f python bench.py --config 2 --no-cpu-baseline --steps 1 --warmup 0 --plain --naive-plain > gpurun_out/ncu_naive.log 2>&1
timeout 1500 python bench.py --verify > gpurun_out/verify.log 2>&1; cat gpurun_out/verify.log | cut -c1-600
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/memcheck.log 2>&1; tail -5 gpurun_out/memcheck.log
