set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/gputest.log
CONFIGS="2 4" LAUNCHES=1 FULL="4" bash tools/refresh_profiles.sh
CONFIGS=4 bash tools/ncu_traffic.sh
