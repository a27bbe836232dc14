# quick parity subset + epilogue probe + c2/c4 bench lines
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x --tb=short -k "${KD_TESTS:-c2 or tiny or self or edge or determinism or shift}" > gpurun_out/gpuq.log 2>&1; tail -2 gpurun_out/gpuq.log
for c in c2 c4; do KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_tim.so timeout 300 python scripts/probe_epi.py $c 2>&1 | grep -E "MMA warp|epilogue warps|busy" | grep -v nan; done
run() { cfg=$1; shift; env "$@" timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_x.log 2>&1; python - "$cfg $*" <<'PY'
import json,sys; d=json.loads(open("gpurun_out/b_x.log").read().strip().splitlines()[-1]); k=d["kernels"]; print(sys.argv[1], round(d["value"]), d["clocks"]["sm_mhz"], "p2/p1 %.3f" % (k["pass2"]["ms_per_step"]/k["pass1"]["ms_per_step"]), {n:round(v["ms_per_step"],2) for n,v in k.items() if v["ms_per_step"]>0.5})
PY
}
for c in c2 c4; do run $c $BENCH_ENV; done
