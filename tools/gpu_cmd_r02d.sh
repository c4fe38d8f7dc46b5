set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/gputest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bdef.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bdef.log | cut -c1-600
for c in 4 5a 5b; do
timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b$c.log 2>&1; tail -1 gpurun_out/b$c.log | cut -c1-300
done
