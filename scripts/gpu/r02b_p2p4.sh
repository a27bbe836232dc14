export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_p2p.py -q --tb=short -rf > gpurun_out/p2p4_tests.log 2>&1; echo "p2p tests rc=$?"; tail -3 gpurun_out/p2p4_tests.log
