"""Probe: per-vocab-entry contributions to dh_s[r, 0] as computed by the CUDA pass-2 + dh GEMM, using
single-row vocab shards (kd_vocab_backward) with the full-vocab records (kd_vocab_stats)."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
from oracle.kd_oracle import lm_head_logits, log_softmax
cfg = KI.CONFIGS["c4"]
W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
H_t, H_s = KI.make_hidden(512, W_t, W_s, seed=1005, head_seed=1000)
rows = [281]
Ht, Hs = H_t[rows], H_s[rows]
up = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)
f = KI.bf16_to_f64
V = cfg.vocab
zt = lm_head_logits(f(Ht), f(W_t)); zs = lm_head_logits(f(Hs), f(W_s))
p = np.exp(log_softmax(zt, 1.0))[0]; q = np.exp(log_softmax(zs, 1.0))[0]
G = q - p
b = f(W_s)[:, 0]
contrib = G * b
order = np.argsort(-np.abs(contrib))
print("exact dh0", contrib.sum(), " top contributions", [(int(v), float(G[v]), float(b[v])) for v in order[:6]])
Htd, Hsd, Wtd, Wsd = up(Ht), up(Hs), up(W_t), up(W_s)
rec = kd.vocab_stats(Htd, Wtd, Hsd, Wsd, vocab=V, v_begin=0, T=1.0)
recs = rec[None]
full = kd.vocab_backward(Htd, Wtd, Hsd, Wsd, recs, vocab=V, v_begin=0, T=1.0).dh_s[0, 0].item()
print("pipeline dh0 (vocab_backward full range)", full, "err", full - contrib.sum())
tot = 0.0
for v in order[:12]:
    v = int(v)
    r = kd.vocab_backward(Htd, Wtd[v:v+1], Hsd, Wsd[v:v+1], recs, vocab=V, v_begin=v, T=1.0)
    gv = r.dh_s[0, 0].item() / b[v] if b[v] != 0 else float("nan")
    tot += r.dh_s[0, 0].item() - contrib[v]
    print(f"v={v:6d} G exact {G[v]: .9e} G gpu {gv: .9e} relerr {(gv - G[v]) / G[v]: .2e}  contrib err {r.dh_s[0,0].item() - contrib[v]: .2e}")
print("sum of top-12 contribution errors", tot)
# remaining vocab as a few big shards
edges = [0, V // 4, V // 2, 3 * V // 4, V]
rest = 0.0
for a, c in zip(edges, edges[1:]):
    r = kd.vocab_backward(Htd, Wtd[a:c], Hsd, Wsd[a:c], recs, vocab=V, v_begin=a, T=1.0)
    rest += r.dh_s[0, 0].item() - contrib[a:c].sum()
print("quarter-shard errors summed", rest)
