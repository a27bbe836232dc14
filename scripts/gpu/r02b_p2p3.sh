# Round 2 (re-entry): p2p exchange for all four kinds + the IPC setup test
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_p2p_ipc.py tests/test_gpu_full.py -q --tb=short -rf -k "p2p or vocab" > gpurun_out/p2p3_tests.log 2>&1; echo "p2p tests rc=$?"; tail -3 gpurun_out/p2p3_tests.log
timeout 900 python bench.py --config c3_jsd --sim-p2p 4 --steps 5 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_simp2p4_jsd.json 2> gpurun_out/bench_simp2p4_jsd.err; echo "simp2p jsd rc=$?"
