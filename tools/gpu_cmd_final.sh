set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
CONFIGS="1 2 3 4 5a 5b" LAUNCHES=0 FULL="" bash tools/refresh_profiles.sh
timeout 1500 python bench.py --verify > gpurun_out/verify.log 2>&1; echo "verify rc=$?"; tail -8 gpurun_out/verify.log | cut -c1-200
