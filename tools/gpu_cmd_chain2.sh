set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "multibounce or config4 or c4 or chain" 2>&1 | tail -1
timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 20 > gpurun_out/b4.log 2>&1; tail -1 gpurun_out/b4.log | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_latent_v3 -s 3 -c 1 -o gpurun_out/full_c4 -f python bench.py --config 4 --plain --no-cpu-baseline --steps 4 --warmup 0 > gpurun_out/ncu_chain.log 2>&1; echo "ncu rc=$?"
CONFIGS=4 bash tools/ncu_traffic.sh
