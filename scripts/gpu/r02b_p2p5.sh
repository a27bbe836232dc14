export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_p2p_ipc.py tests/test_gpu_full.py -q --tb=short -rf -k "p2p or vocab" > gpurun_out/p2p5_tests.log 2>&1; echo "p2p tests rc=$?"; tail -3 gpurun_out/p2p5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
