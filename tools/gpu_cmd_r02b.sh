set -u
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ShadeSpectralF2 -c 1 -o gpurun_out/naive2 -f python bench.py --config 2 --no-cpu-baseline --steps 1 --warmup 0 --plain --naive-plain > gpurun_out/ncu_naive.log 2>&1; echo "ncu naive rc=$?"
STEPS=20 bash tools/sweep_loss.sh > gpurun_out/sweep_loss.log 2>&1; cat gpurun_out/sweep_loss.log
bash tools/ncu_traffic.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
