"""Diagnostic: KD_GRAD_BF16 dW vs an emulation (oracle G rounded to bf16, fp64 product)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
from oracle.kd_oracle import grad_student_logits, lm_head_logits
cfg = KI.CONFIGS["c2"]
W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
n = 256
H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1011, head_seed=1000)
up = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
f = KI.bf16_to_f64
rf = kd.fused_fwd_bwd(up(H_t), up(W_t), up(H_s), up(W_s), T=1.0, kind="fkl", want_dW=True, grad_precision="bf16")
rs = kd.fused_fwd_bwd(up(H_t), up(W_t), up(H_s), up(W_s), T=1.0, kind="fkl", want_dW=True)
torch.cuda.synchronize()
G = grad_student_logits("fkl", lm_head_logits(f(H_t), f(W_t)), lm_head_logits(f(H_s), f(W_s)), 1.0, 0.5)
Hs = f(H_s)
ref = G.T @ Hs
Gb = torch.from_numpy(G).float().bfloat16().double().numpy()
emul = Gb.T @ Hs
b = 2.0 ** -9 * (np.abs(G).T @ np.abs(Hs))
fast = rf.dW_s.cpu().numpy().astype(np.float64)
split = rs.dW_s.cpu().numpy().astype(np.float64)
for name, x in (("fast", fast), ("split", split), ("emul", emul)):
    d = np.abs(x - ref)
    i = np.unravel_index(np.argmax(d / (b + 1e-5 + 2e-3 * np.abs(ref))), d.shape)
    print(name, "max |d|", d.max(), "worst ratio", (d / (b + 1e-5 + 2e-3 * np.abs(ref))).max(), "at", i,
          "got", x[i], "ref", ref[i], "b", b[i], "emul", emul[i])
v, j = np.unravel_index(np.argmax(np.abs(fast - ref) / (b + 1e-5 + 2e-3 * np.abs(ref))), ref.shape)
col = G[:, v]
top = np.argsort(-np.abs(col))[:6]
print("G[:, v] top entries", [(int(t), float(col[t]), float(Hs[t, j])) for t in top])
print("fast - emul at worst", fast[v, j] - emul[v, j], "split - ref", split[v, j] - ref[v, j])
dh = rf.dh_s.cpu().numpy()
