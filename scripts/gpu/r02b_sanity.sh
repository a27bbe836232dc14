# Round 2 (re-entry): GPU suite + smoke + default bench on the rebuilt library
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/parity_sanity.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity_sanity.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/gpu_tests_sanity.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests_sanity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_sanity.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_sanity.log
timeout 900 python bench.py > gpurun_out/bench_sanity.json 2> gpurun_out/bench_sanity.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_sanity.json
