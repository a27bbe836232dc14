./scripts/probe/die_map > gpurun_out/die_map_orig.txt 2>&1; head -3 gpurun_out/die_map_orig.txt
KD_DIE_DEBUG=2 python - <<'P' 2>&1 | tail -25
import torch, numpy as np, sys
sys.path.insert(0, ".")
import kd_inputs as KI, paper_2603_01875_b200 as kd
inp = KI.make_inputs(512, 256, 128, 4096, seed=1)
up = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
r = kd.fused_fwd_bwd(up(inp.H_t), up(inp.W_t), up(inp.H_s), up(inp.W_s))
torch.cuda.synchronize(); print("ok")
P
python - <<'P'
import numpy as np
rows=[l.split() for l in open("gpurun_out/die_map_orig.txt") if l[0].isdigit()]
a=np.array(rows,dtype=float)
for b in range(1,a.shape[1]):
    v=np.sort(a[:,b]); print("orig buf",b-1,"min",v[0],"p25",v[37],"med",v[74],"p75",v[111],"max",v[-1])
P
