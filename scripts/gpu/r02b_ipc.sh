export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_p2p_ipc.py -q --tb=short > gpurun_out/ipc.log 2>&1; echo "ipc rc=$?"; tail -2 gpurun_out/ipc.log
