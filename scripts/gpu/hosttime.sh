KD_HOST_TIMING=1 timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_ht.json 2> gpurun_out/bench_ht.err
grep "kd host" gpurun_out/bench_ht.err
python - <<'PY'
import time, torch, numpy as np
import paper_2603_01875_b200 as kd
import kd_inputs as KI
inp = KI.make_inputs(4096, 256, 128, 4096, seed=1)
up = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
a = [up(x) for x in (inp.H_t, inp.W_t, inp.H_s, inp.W_s)]
for _ in range(3): kd.fused_fwd_bwd(*a, chunk_tokens=256)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): kd.fused_fwd_bwd(*a, chunk_tokens=256)
h = (time.perf_counter() - t) / 20 * 1e3
torch.cuda.synchronize()
print("tiny-problem host ms per call (16 chunks):", round(h, 3), "launches", kd.last_launch_count())
PY
