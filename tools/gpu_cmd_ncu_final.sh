set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ShadeLatentOp -s 2 -c 1 -f -o gpurun_out/full_c2 python bench.py --config 2 --plain --steps 4 > gpurun_out/ncu_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ShadeLatentOp -s 2 -c 1 -f -o gpurun_out/full_c3 python bench.py --config 3 --plain --steps 4 > gpurun_out/ncu_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:naive_lanes -s 1 -c 1 -f -o gpurun_out/full_c3naive python bench.py --config 3 --plain --naive-plain --steps 2 > gpurun_out/ncu_c3n.log 2>&1; echo "c3 naive rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_spectral_lanes -s 1 -c 1 -f -o gpurun_out/full_c4naive python bench.py --config 4 --plain --naive-plain --steps 2 > gpurun_out/ncu_c4n.log 2>&1; echo "c4 naive rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_kernel -s 2 -c 1 -f -o gpurun_out/full_c5a python bench.py --config 5a --plain --steps 4 > gpurun_out/ncu_c5a.log 2>&1; echo "c5a rc=$?"
