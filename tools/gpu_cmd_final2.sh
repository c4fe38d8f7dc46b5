set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
CONFIGS="3 2" LAUNCHES=0 FULL="none" bash tools/refresh_profiles.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
