for c in c4 c2; do for v in tim x1; do echo "== $c $v"; KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_$v.so timeout 300 python scripts/probe_epi.py $c 2>&1 | grep -E "MMA warp|busy" | grep -v nan; done; done
run() { cfg=$1; shift; env "$@" timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_x.log 2>&1; python - "$cfg $*" <<'PY'
import json,sys; d=json.loads(open("gpurun_out/b_x.log").read().strip().splitlines()[-1]); k=d["kernels"]; print(sys.argv[1], round(d["value"]), d["clocks"]["sm_mhz"], "p2/p1 %.3f" % (k["pass2"]["ms_per_step"]/k["pass1"]["ms_per_step"]), {n:round(v["ms_per_step"],2) for n,v in k.items() if v["ms_per_step"]>0.5})
PY
}
for c in c2 c4; do run $c; done
