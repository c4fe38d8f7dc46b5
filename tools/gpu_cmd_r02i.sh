# Round 2, fourth session: final refresh (tests, smoke, every config's bench line, full-size verify, launch list).
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CONFIGS="1 2 3 4 5a 5b" LAUNCHES=1 FULL="none" bash tools/refresh_profiles.sh
timeout 600 python bench.py --config 4 --steps 20 > gpurun_out/final_c4_20.json 2> gpurun_out/final_c4_20.err; echo "bench c4 (20 steps) rc=$?"
timeout 1500 python bench.py --verify > gpurun_out/verify_fullsize.jsonl 2> gpurun_out/verify.err; echo "verify rc=$?"; tail -c 600 gpurun_out/verify_fullsize.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference arm rc=$?"; tail -c 400 gpurun_out/bench_reference.json
