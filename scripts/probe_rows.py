"""Probe: do the tcgen05-accumulated logits explain the residual dh_s[:,0] error on the failing rows?
dh[r, :] recomputed in fp64 from GPU logits (reversed K order as in kd_pass, optionally K-chunked)."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd

def gpu_logits(H, W, chunks):
    Hd = torch.from_numpy(H.view(np.int16)).cuda().view(torch.bfloat16).flip(1).contiguous()
    Wd = torch.from_numpy(W.view(np.int16)).cuda().view(torch.bfloat16).flip(1).contiguous()
    K = H.shape[1]; out = 0
    for c in range(chunks):
        a, b = K * c // chunks, K * (c + 1) // chunks
        out = out + kd.gemm_bf16_f32(Hd[:, a:b].contiguous(), Wd[:, a:b].contiguous(), M=H.shape[0], N=W.shape[0], K=b - a).double().cpu().numpy()
    return out

def dh_from(zt, zs, Ws, T=1.0):
    def ls(z):
        a = z / T; m = a.max(1, keepdims=True); return a - m - np.log(np.exp(a - m).sum(1, keepdims=True))
    G = (np.exp(ls(zs)) - np.exp(ls(zt))) / T
    return G @ Ws

for name, n, seed, rows in (("c2", 32768, 1001, None), ("c4", 512, 1005, [281, 320])):
    cfg = KI.CONFIGS[name]
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
    H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=seed, head_seed=1000)
    if rows is None:
        r = np.sort(np.random.default_rng(0).choice(n, 64, replace=False)); r[0], r[-1] = 0, n - 1; rows = [r[49]]
    Ht, Hs = H_t[rows], H_s[rows]
    Wtf, Wsf = KI.bf16_to_f64(W_t), KI.bf16_to_f64(W_s)
    ref = dh_from(KI.bf16_to_f64(Ht) @ Wtf.T, KI.bf16_to_f64(Hs) @ Wsf.T, Wsf)[:, 0]
    for ch in (1, 2, 4):
        got = dh_from(gpu_logits(Ht, W_t, ch), gpu_logits(Hs, W_s, ch), Wsf)[:, 0]
        print(name, rows, f"chunks={ch}", "ref", np.round(ref, 7), "err", np.array2string(got - ref, precision=2), "tol", np.array2string(1e-5 + 2e-3 * np.abs(ref), precision=2))
