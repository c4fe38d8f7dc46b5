# e2e leg of config 2, repeated (profiles/r01/e2e_sweep.md): python bench.py's "e2e" object per run.
for i in 1 2 3; do
  timeout 200 python bench.py --no-cpu-baseline --no-naive --steps 100 > gpurun_out/e2e.log 2>&1
  tail -1 gpurun_out/e2e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"], d["e2e_matches_device"])'
done
