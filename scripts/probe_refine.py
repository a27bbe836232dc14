"""Probe: would an exact re-evaluation of each row's top logits remove the logit-accuracy-limited gradient errors?

Takes tcgen05 fp32-accumulated logits (the plain GEMM entry point, K fed last-to-first like the fused passes), then
computes the FKL gradient three ways in fp64 from the SAME logits: (a) as the kernels do (every logit from the tensor
cores), (b) with each row's top-K teacher and student logits replaced by their exact values and the two LSEs corrected
for them, (c) exact.  Prints the worst |Δ| / (2e-3|ref| + 1e-5) of dh_s and dW_s for (a) and (b).

    python scripts/probe_refine.py [c2|c4] [T]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI  # noqa: E402
import paper_2603_01875_b200 as kd  # noqa: E402


def up(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)


def gpu_logits(H, W):
    # reversed K order (bias column last), as kd_pass feeds its K blocks
    Hr, Wr = up(H).flip(1).contiguous(), up(W).flip(1).contiguous()
    return kd.gemm_bf16_f32(Hr, Wr, M=H.shape[0], N=W.shape[0], K=H.shape[1]).double().cpu().numpy()


def grad_fkl(zt, zs, T):
    a, b = zt / T, zs / T
    lp = a - a.max(1, keepdims=True)
    lp -= np.log(np.exp(lp).sum(1, keepdims=True))
    lq = b - b.max(1, keepdims=True)
    lq -= np.log(np.exp(lq).sum(1, keepdims=True))
    return (np.exp(lq) - np.exp(lp)) / T


def ratio(got, ref):
    return (np.abs(got - ref) / (1e-5 + 2e-3 * np.abs(ref))).max()


name = sys.argv[1] if len(sys.argv) > 1 else "c2"
T = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = KI.CONFIGS[name]
W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
n = 512
H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1005, head_seed=1000)
f = KI.bf16_to_f64
Wt, Ws, Ht, Hs = f(W_t), f(W_s), f(H_t), f(H_s)
zt_x, zs_x = Ht @ Wt.T, Hs @ Ws.T
zt_g, zs_g = gpu_logits(H_t, W_t), gpu_logits(H_s, W_s)
print(f"{name} T={T}: logit error max teacher {np.abs(zt_g - zt_x).max():.2e} student {np.abs(zs_g - zs_x).max():.2e}")
G_x = grad_fkl(zt_x, zs_x, T)
dh_x, dW_x = G_x @ Ws, G_x.T @ Hs
G_a = grad_fkl(zt_g, zs_g, T)
print(f"  (a) tensor-core logits everywhere: dh ratio {ratio(G_a @ Ws, dh_x):.3f}  dW ratio {ratio(G_a.T @ Hs, dW_x):.3f}")
for K in (1, 2, 4, 8, 16):
    zt_r, zs_r = zt_g.copy(), zs_g.copy()
    rows = np.arange(n)[:, None]
    it = np.argsort(-zt_g, axis=1)[:, :K]
    is_ = np.argsort(-zs_g, axis=1)[:, :K]
    # exact logits at the union of both sides' top-K (the refine kernel's fp64 dot products); the softmax normalisers
    # then follow from the corrected values (the LSE correction)
    for idx in (it, is_):
        zt_r[rows, idx] = zt_x[rows, idx]
        zs_r[rows, idx] = zs_x[rows, idx]
    G_b = grad_fkl(zt_r, zs_r, T)
    print(f"  (b) top-{K} per side exact: dh ratio {ratio(G_b @ Ws, dh_x):.3f}  dW ratio {ratio(G_b.T @ Hs, dW_x):.3f}")
