"""Small cases of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_case.py [all|tiny]

Covers: the fused decoupled passes (FKL), the coupled pass 1 (RKL), the JSD/TVD planes + K fix-up, both backward
GEMM layouts (dh: MN/MN, dW: K/MN) with split-K reduce and the residual fix, masked compaction/gather, ragged token
and vocab tails (N = 300 and 129, V = 1000 and 4097), the staged variant (stage_logits), the teacher-LSE path, the
top-k baseline and the vocab-shard entry points.  Outputs are checked for finiteness only (parity is the parity
tests' job); the point is that every launch runs under the sanitizer.
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


def finite(*ts):
    for t in ts:
        if t is not None:
            assert torch.isfinite(t).all().item(), "non-finite output"


def main(which):
    torch.cuda.set_device(0)
    cases = [(300, 256, 128, 1000), (129, 192, 64, 4097)] if which == "all" else [(300, 256, 128, 1000)]
    for N, d_t, d_s, V in cases:
        mask = (np.arange(N) % 5 != 0).astype(np.uint8)
        inp = KI.make_inputs(N, d_t, d_s, V, seed=N, mask=mask)
        Ht, Wt, Hs, Ws = up(inp.H_t), up(inp.W_t), up(inp.H_s), up(inp.W_s)
        m = torch.from_numpy(mask).cuda()
        kinds = ["fkl", "rkl", "jsd", "tvd"] if which == "all" else ["fkl", "rkl", "jsd"]
        for kind in kinds:
            for stage in ((False, True) if which == "all" or kind == "fkl" else (False,)):
                r = kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, m, T=1.3, kind=kind, want_dW=True, chunk_tokens=128,
                                     stage_logits=stage)
                torch.cuda.synchronize()
                finite(r.loss, r.dh_s, r.dW_s)
                print(f"ok N={N} V={V} {kind} stage={stage}", flush=True)
        if which != "all":
            continue
        lse = kd.teacher_lse(Ht, Wt, m, d_s=d_s, T=1.0, chunk_tokens=128)
        r = kd.fused_fwd_bwd_lse(Ht, Wt, Hs, Ws, lse, m, T=1.0, want_dW=True, chunk_tokens=128)
        torch.cuda.synchronize()
        finite(r.loss, r.dh_s, r.dW_s)
        idx, val = kd.teacher_topk(Ht, Wt, m, k=8, d_s=d_s, T=1.0, chunk_tokens=128)
        r = kd.topk_fwd_bwd(Hs, Ws, idx, val, m, d_t=d_t, T=1.0, want_dW=True, chunk_tokens=128)
        torch.cuda.synchronize()
        finite(r.loss, r.dh_s, r.dW_s)
        a, b = 0, (V // 256) * 128 or V
        rec = kd.vocab_stats(Ht, Wt[a:b], Hs, Ws[a:b], m, vocab=V, v_begin=a, T=1.0, kind="fkl")
        rec2 = kd.vocab_stats(Ht, Wt[b:], Hs, Ws[b:], m, vocab=V, v_begin=b, T=1.0, kind="fkl")
        recs = torch.stack([rec, rec2])
        r = kd.vocab_backward(Ht, Wt[a:b], Hs, Ws[a:b], recs, m, vocab=V, v_begin=a, T=1.0, kind="fkl", want_dW=True)
        kj, st = kd.vocab_partials(Ht, Wt[a:b], Hs, Ws[a:b], torch.stack([
            kd.vocab_stats(Ht, Wt[a:b], Hs, Ws[a:b], m, vocab=V, v_begin=a, T=2.0, kind="jsd"),
            kd.vocab_stats(Ht, Wt[b:], Hs, Ws[b:], m, vocab=V, v_begin=b, T=2.0, kind="jsd")]), m, vocab=V,
            v_begin=a, T=2.0, kind="jsd", want_dW=True)
        r2 = kd.vocab_finish(st, Ht, Wt[a:b], Hs, Ws[a:b], torch.stack([kj, kj]), m)
        torch.cuda.synchronize()
        finite(r.dh_s, r2.dh_s)
        print(f"ok N={N} V={V} lse/topk/vocab-shard entry points", flush=True)
    print("SANITIZE_CASE_DONE", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
