"""Probe: isolate which stage causes the residual dh_s[:,0] error on the known ill-conditioned rows."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
from oracle.kd_oracle import kd_fused_fwd_bwd, lm_head_logits
cfg = KI.CONFIGS["c4"]
W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
H_t, H_s = KI.make_hidden(512, W_t, W_s, seed=1005, head_seed=1000)
rows = [281, 320, 0, 1]
Ht, Hs = H_t[rows], H_s[rows]
up = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)
f = KI.bf16_to_f64
loss, dh, _ = kd_fused_fwd_bwd(f(Ht), f(W_t), f(Hs), f(W_s), T=1.0, kind="fkl")
r = kd.fused_fwd_bwd(up(Ht), up(W_t), up(Hs), up(W_s), T=1.0, kind="fkl"); torch.cuda.synchronize()
print("KD_KB_PER_ACC", os.environ.get("KD_KB_PER_ACC"), "dh[:,0] err", r.dh_s[:, 0].double().cpu().numpy() - dh[:, 0], "ref", dh[:, 0])
rec = kd.vocab_stats(up(Ht), up(W_t), up(Hs), up(W_s), vocab=cfg.vocab, v_begin=0, T=1.0).double().cpu().numpy()
zt = lm_head_logits(f(Ht), f(W_t)); zs = lm_head_logits(f(Hs), f(W_s))
lse_t = np.log(np.exp(zt - zt.max(1, keepdims=True)).sum(1)) + zt.max(1)
lse_s = np.log(np.exp(zs - zs.max(1, keepdims=True)).sum(1)) + zs.max(1)
L2t = rec[0] + np.log2(rec[2]); L2s = rec[1] + np.log2(rec[3])
print("LSE err (nats) teacher", L2t * np.log(2) - lse_t, " student", L2s * np.log(2) - lse_s)
print("M2 - max(z)*log2e teacher", rec[0] - zt.max(1) / np.log(2))
