set -x
export PYTHONUNBUFFERED=1
# 1. tests that failed + the sanitizer test + the whole general file
KD_PARITY_LOG=$PWD/gpurun_out/parity2.jsonl timeout 1200 python -m pytest tests/test_gpu_general.py tests/test_gpu_full.py tests/test_gpu_sanitizer.py -m gpu -q --tb=short -rf -s > gpurun_out/gpu_tests2.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/gpu_tests2.log
# 2. new bench, default
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_default.err
# 3. promotion period A/B with the new GEMM epilogue
for k in 64 16 8; do KD_KB_PER_ACC=$k timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_kbn$k.json 2> gpurun_out/bench_kbn$k.err; done
# 4. pass-2 store/staging variants (timing only)
for v in gv4 nog nost; do KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_$v.so timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_var_$v.json 2> gpurun_out/bench_var_$v.err; done
timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/bench_var_base.json 2> gpurun_out/bench_var_base.err
# 5. the N>1 vocab headline path: 2 gloo ranks sharing the GPU (exchange logic only; not a throughput)
KD_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; echo "n2 rc=$?"; tail -5 gpurun_out/bench_n2_gloo.err
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d.get("clocks",{}) and d["clocks"].get("sm_mhz"), d.get("roofline",{}).get("frac"))
P
