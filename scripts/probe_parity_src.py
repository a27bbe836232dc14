"""Probe: where do the remaining strict gradient-tolerance violations come from?

For the reduced-N full-vocab configs (c2 / c4 shapes, N = 512, + dW) prints, for loss / dh_s / dW_s, the worst
|got - ref| / (atol + rtol |ref|) against the fp64 oracle, the number of strict violations and the columns where the
worst dh_s elements sit.  Run once per KD_KB_PER_ACC value (the backward GEMMs' TMEM promotion period, read once per
process) to separate the dh-GEMM accumulation error from the logit error of the fused passes.

    KD_KB_PER_ACC=8 python scripts/probe_parity_src.py c4
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI  # noqa: E402
import paper_2603_01875_b200 as kd  # noqa: E402
from oracle.kd_oracle import kd_fused_fwd_bwd  # noqa: E402


def up(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)


def report(name, got, ref, rtol, atol):
    got = got.astype(np.float64)
    d = np.abs(got - ref)
    r = d / (atol + rtol * np.abs(ref))
    i = np.unravel_index(np.argmax(r), r.shape)
    print(f"  {name:6s} max ratio {r.max():7.3f} at {tuple(int(x) for x in i)} (got {got[i]:.6e} ref {ref[i]:.6e}) "
          f"viol {(r > 1).sum()} / {r.size}; max|d| {d.max():.3e}", flush=True)
    return r


for name in sys.argv[1:] or ["c2", "c4"]:
    cfg = KI.CONFIGS[name]
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
    n = 512
    H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1005, head_seed=1000)
    r = kd.fused_fwd_bwd(up(H_t), up(W_t), up(H_s), up(W_s), None, T=cfg.temperature, kind=cfg.kind,
                         beta=cfg.jsd_beta, want_dW=True)
    torch.cuda.synchronize()
    f = KI.bf16_to_f64
    loss, dh, dW = kd_fused_fwd_bwd(f(H_t), f(W_t), f(H_s), f(W_s), None, T=cfg.temperature, kind=cfg.kind,
                                    beta=cfg.jsd_beta, want_dW=True)
    print(f"{name} N={n} KD_KB_PER_ACC={os.environ.get('KD_KB_PER_ACC', 'default')}")
    report("loss", r.loss.cpu().numpy(), loss, 1e-3, 1e-5)
    rd = report("dh_s", r.dh_s.cpu().numpy(), dh, 2e-3, 1e-5)
    rw = report("dW_s", r.dW_s.cpu().numpy(), dW, 2e-3, 1e-5)
    cols = np.argsort(rd.max(axis=0))[::-1][:5]
    print("  dh worst columns", [(int(c), round(float(rd[:, c].max()), 3)) for c in cols])
    cols = np.argsort(rw.max(axis=0))[::-1][:5]
    print("  dW worst columns", [(int(c), round(float(rw[:, c].max()), 3)) for c in cols])
    # logit accuracy of a whole-K tcgen05 accumulation vs 2 / 4 promoted pieces (plain GEMM entry point)
    Ht, Wt = up(H_t[:128]), up(W_t)
    Zx = f(H_t[:128]) @ f(W_t).T
    for pieces in (1, 2, 4):
        d = cfg.d_t
        Z = sum(kd.gemm_bf16_f32(Ht[:, c:c + d // pieces].contiguous(), Wt[:, c:c + d // pieces].contiguous(),
                                 M=128, N=cfg.vocab, K=d // pieces).double().cpu().numpy()
                for c in range(0, d, d // pieces))
        e = Z - Zx
        print(f"  teacher logits K={d} in {pieces} piece(s): max|err| {np.abs(e).max():.3e} rms "
              f"{np.sqrt((e ** 2).mean()):.3e} mean {e.mean():.3e}", flush=True)
