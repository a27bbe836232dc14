# Round 2 (re-entry): p2p exchange + reduce_dh rewrite: GPU suite, default bench, one-GPU p2p emulation at c2 / c3_rkl
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -q --tb=short -rf > gpurun_out/p2p_tests.log 2>&1; echo "p2p tests rc=$?"; tail -3 gpurun_out/p2p_tests.log
rm -f gpurun_out/parity_p2p.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity_p2p.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/gpu_tests_p2p.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests_p2p.log
timeout 900 python bench.py --no-variants > gpurun_out/bench_p2p_default.json 2> gpurun_out/bench_p2p_default.err; echo "bench rc=$?"
timeout 900 python bench.py --sim-p2p 8 --steps 5 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_simp2p8.json 2> gpurun_out/bench_simp2p8.err; echo "simp2p rc=$?"
timeout 900 python bench.py --config c3_rkl --sim-p2p 4 --steps 5 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_simp2p4_rkl.json 2> gpurun_out/bench_simp2p4_rkl.err; echo "simp2p rkl rc=$?"
