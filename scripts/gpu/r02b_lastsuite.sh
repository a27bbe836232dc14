# The final commit: GPU suite (parity log) + smoke
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/last
rm -f gpurun_out/last/parity.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/last/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/last/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/last/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/last/smoke.log
