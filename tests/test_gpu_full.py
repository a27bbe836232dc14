"""GPU parity at BASELINE.json's full sizes + edge cases + invariants (through the C ABI).

Full-size runs use the launch configuration bench.py times (default chunking / splits) and compare
sampled tokens with the oracle, which computes them one by one (per-token outputs depend only on that
row and the heads).  dW_s, which needs every row, is checked on reduced-N instances at full V.
"""
import numpy as np
import pytest
import torch

import kd_inputs as KI
from tests.kdtest_util import (GRAD_ATOL, GRAD_RTOL, LOSS_ATOL, LOSS_RTOL, assert_grad_close, assert_kd_close,
                               dev_bf16, f64, oracle_run)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def kd():
    import paper_2603_01875_b200 as m
    return m


_HEADS = {}


def heads(V, d_t, d_s, seed=0):
    key = (V, d_t, d_s, seed)
    if key not in _HEADS:
        _HEADS.clear()
        _HEADS[key] = KI.make_heads(V, d_t, d_s, seed=1000 + seed)
    return _HEADS[key]


def run(inp, mask=None, **kw):
    m = None if mask is None else torch.from_numpy(mask).cuda()
    r = kd().fused_fwd_bwd(dev_bf16(inp.H_t), dev_bf16(inp.W_t), dev_bf16(inp.H_s), dev_bf16(inp.W_s), m, **kw)
    torch.cuda.synchronize()
    return r


def _sampled_check(inp, r, rows, *, T, kind, beta=0.5):
    loss, dh, _ = oracle_run(inp, T=T, kind=kind, beta=beta, rows=rows)
    got_loss = r.loss.cpu().numpy()[rows]
    got_dh = r.dh_s.cpu().numpy()[rows]
    assert_kd_close("loss", got_loss, loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", got_dh, dh)


# ------------------------------------------------------------------ full sizes, bench launch configuration
def test_config2_full_size_sampled():
    """configs[1]: 32768 tokens, d_t=4096, d_s=2048, V=151936, FKL T=1 — 64 sampled tokens vs oracle."""
    cfg = KI.CONFIGS["c2"]
    W_t, W_s = heads(cfg.vocab, cfg.d_t, cfg.d_s)
    H_t, H_s = KI.make_hidden(cfg.n_tokens, W_t, W_s, seed=1001, head_seed=1000)
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, None)
    r = run(inp, T=cfg.temperature, kind=cfg.kind)
    assert int(r.n_nonfinite.item()) == 0
    rows = np.sort(np.random.default_rng(0).choice(cfg.n_tokens, 64, replace=False))
    rows[0], rows[-1] = 0, cfg.n_tokens - 1  # first / last rows (chunk edges)
    _sampled_check(inp, r, rows, T=cfg.temperature, kind=cfg.kind)
    # property at any size: Σ_v G = 0 ⇒ dh_s · 1 = G · (W_s · 1)... checked via the constant-column pin below
    l = r.loss.cpu().numpy()
    assert np.all(np.isfinite(l)) and np.all(l >= -1e-5)


@pytest.mark.parametrize("name", ["c3_rkl", "c3_jsd"])
def test_config3_full_size_masked_sampled(name):
    """configs[2]: RKL / JSD(0.5) at T=2 with the prompt/padding mask, 32768 tokens."""
    cfg = KI.CONFIGS[name]
    W_t, W_s = heads(cfg.vocab, cfg.d_t, cfg.d_s)
    H_t, H_s = KI.make_hidden(cfg.n_tokens, W_t, W_s, seed=1001, head_seed=1000)
    mask = KI.make_mask(cfg)
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, mask)
    r = run(inp, mask, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta)
    live = np.flatnonzero(mask)
    rows = np.sort(np.random.default_rng(1).choice(live, 48, replace=False))
    _sampled_check(inp, r, rows, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta)
    dead = np.flatnonzero(mask == 0)
    assert np.all(r.loss.cpu().numpy()[dead] == 0)
    assert np.all(r.dh_s.cpu().numpy()[dead] == 0)
    if cfg.kind == "jsd":
        assert np.all(r.loss.cpu().numpy() <= np.log(2) + 1e-5)


# The only elements allowed beyond the plain north-star bound (R14, tests/kdtest_util.assert_grad_close):
# (allowed count, max ratio) per (config, output), from the committed parity record (profiles/r02_parity.md).  They are
# logit-accuracy-limited elements of fp32-accumulated K = d_t bf16 GEMMs (scripts/probe_parity_src.py); every other
# element of these runs — and every element of every other test — meets the plain bound.
R14_ALLOW = {("c2", "dh_s"): (1, 1.9), ("c2", "dW_s"): (3, 1.15), ("c4", "dW_s"): (1, 1.05),
             ("c3_rkl", "dW_s"): (2, 1.25)}


@pytest.mark.parametrize("cfg_name,n", [("c2", 512), ("c4", 512), ("c3_rkl", 384)])
def test_reduced_n_full_vocab_with_dW(cfg_name, n):
    """Config shapes at N=512 (full V, full d) including dW_s over all rows."""
    cfg = KI.CONFIGS[cfg_name]
    W_t, W_s = heads(cfg.vocab, cfg.d_t, cfg.d_s)
    H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1005, head_seed=1000)
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, None)
    r = run(inp, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, want_dW=True)
    loss, dh, dW = oracle_run(inp, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, want_dW=True)
    assert_kd_close("loss", r.loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    for name, got, ref in (("dh_s", r.dh_s, dh), ("dW_s", r.dW_s, dW)):
        allow, mr = R14_ALLOW.get((cfg_name, name), (0, 1.0))
        assert_grad_close(name, got.cpu().numpy(), ref, allow=allow, max_ratio=mr)


def test_config5_ragged_accumulate_dW():
    """configs[4]: ragged on-policy batch, RKL, dW_s accumulated over micro-batches ≡ one batch."""
    cfg = KI.CONFIGS["c5"]
    d_t, d_s, V = 512, 256, 20000  # reduced widths so the dW oracle stays seconds
    W_t, W_s = KI.make_heads(V, d_t, d_s, seed=1007)
    n = 1500
    H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1008, head_seed=1007)
    mask = KI.make_mask(KI.KDConfig("r", 1, n, d_t, d_s, V, mask="ragged"), seed=1009)
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, mask)
    m = torch.from_numpy(mask).cuda()
    Ht, Hs, Wt, Ws = dev_bf16(H_t), dev_bf16(H_s), dev_bf16(W_t), dev_bf16(W_s)
    dW = torch.zeros(V, d_s, dtype=torch.float32, device="cuda")
    bounds = [0, 333, 900, 901, n]  # 4 micro-batches, one of a single row
    for a, b in zip(bounds, bounds[1:]):
        kd().fused_fwd_bwd(Ht[a:b], Wt, Hs[a:b], Ws, m[a:b], T=1.0, kind="rkl", want_dW=True, accumulate_dW=True,
                           dW_s=dW, chunk_tokens=256)
    whole = kd().fused_fwd_bwd(Ht, Wt, Hs, Ws, m, T=1.0, kind="rkl", want_dW=True, chunk_tokens=256)
    torch.cuda.synchronize()
    _, _, dW_ref = oracle_run(inp, T=1.0, kind="rkl", want_dW=True)
    assert_grad_close("dW accumulated", dW.cpu().numpy(), dW_ref)
    assert_grad_close("dW whole", whole.dW_s.cpu().numpy(), dW_ref)


# ------------------------------------------------------------------ edge cases
def test_edge_empty_and_all_masked():
    W_t, W_s = KI.make_heads(300, 128, 64, seed=5)
    inp = KI.make_inputs(5, 128, 64, 300, seed=5, heads=(W_t, W_s))
    dW = torch.full((300, 64), 7.0, device="cuda")
    r = kd().fused_fwd_bwd(dev_bf16(inp.H_t[:0]), dev_bf16(W_t), dev_bf16(inp.H_s[:0]), dev_bf16(W_s),
                           want_dW=True, dW_s=dW)
    torch.cuda.synchronize()
    assert r.loss.numel() == 0 and float(dW.abs().max()) == 0.0
    mask = np.zeros(5, np.uint8)
    r = run(inp, mask, T=1.0, kind="fkl", want_dW=True)
    assert np.all(r.loss.cpu().numpy() == 0) and np.all(r.dh_s.cpu().numpy() == 0)
    assert np.all(r.dW_s.cpu().numpy() == 0)


@pytest.mark.parametrize("N,V,d_t,d_s", [(1, 1, 64, 64), (129, 64, 64, 128), (257, 129, 192, 64),
                                         (1000, 4097, 128, 320)])
def test_edge_shapes(N, V, d_t, d_s):
    """Single token, single vocab row, tails on every tile edge, d_s not a multiple of the 256 N tile."""
    inp = KI.make_inputs(N, d_t, d_s, V, seed=N + V)
    r = run(inp, T=1.3, kind="fkl", want_dW=True, chunk_tokens=256)
    loss, dh, dW = oracle_run(inp, T=1.3, kind="fkl", want_dW=True)
    assert_kd_close("loss", r.loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", r.dh_s.cpu().numpy(), dh)
    assert_grad_close("dW_s", r.dW_s.cpu().numpy(), dW)


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("kind", ["fkl", "rkl", "tvd"])
def test_self_distillation_bitwise_zero(kind):
    """Student := teacher (P:64 self-distillation): identical GEMM paths ⇒ loss and gradients exactly 0."""
    inp = KI.self_distillation_twin(KI.make_config_inputs(KI.CONFIGS["tiny"]))
    r = run(inp, T=1.0, kind=kind, want_dW=True)
    assert np.all(r.loss.cpu().numpy() == 0)
    assert np.all(r.dh_s.cpu().numpy() == 0)
    assert np.all(r.dW_s.cpu().numpy() == 0)


def test_self_distillation_jsd_near_zero():
    inp = KI.self_distillation_twin(KI.make_config_inputs(KI.CONFIGS["tiny"]))
    r = run(inp, T=1.0, kind="jsd")
    assert np.abs(r.loss.cpu().numpy()).max() < 1e-6
    assert np.abs(r.dh_s.cpu().numpy()).max() < 1e-6


def test_masked_rows_never_read_bitwise():
    """NaN/Inf garbage in masked rows changes no output bit."""
    N, d_t, d_s, V = 400, 256, 128, 3000
    mask = (np.random.default_rng(3).random(N) > 0.4).astype(np.uint8)
    inp = KI.make_inputs(N, d_t, d_s, V, seed=9, mask=mask)
    r0 = run(inp, mask, T=2.0, kind="jsd", want_dW=True, chunk_tokens=128)
    bad_t, bad_s = inp.H_t.copy(), inp.H_s.copy()
    bad_t[mask == 0] = 0x7FC0  # bf16 NaN
    bad_s[mask == 0] = 0x7F80  # bf16 +Inf
    r1 = run(KI.KDInputs(bad_t, inp.W_t, bad_s, inp.W_s, mask), mask, T=2.0, kind="jsd", want_dW=True,
             chunk_tokens=128)
    for a, b in ((r0.loss, r1.loss), (r0.dh_s, r1.dh_s), (r0.dW_s, r1.dW_s)):
        assert torch.equal(a, b)


def test_deterministic_bitwise():
    inp = KI.make_inputs(700, 256, 128, 5000, seed=11)
    a = run(inp, T=1.0, kind="rkl", want_dW=True)
    b = run(inp, T=1.0, kind="rkl", want_dW=True)
    assert torch.equal(a.loss, b.loss) and torch.equal(a.dh_s, b.dh_s) and torch.equal(a.dW_s, b.dW_s)


def test_shift_invariance_constant_column():
    """Adding a constant to every logit of a row leaves the divergence unchanged.  The shift is
    built inside the GEMM: hidden column 1 set to 1 and head column 1 set to a constant c (exact in bf16)."""
    inp = KI.make_inputs(256, 256, 128, 2048, seed=12)
    Ht, Hs = KI.bf16_to_f32(inp.H_t).copy(), KI.bf16_to_f32(inp.H_s).copy()
    Wt, Ws = KI.bf16_to_f32(inp.W_t).copy(), KI.bf16_to_f32(inp.W_s).copy()
    Ht[:, 1] = 1.0
    Hs[:, 1] = 1.0
    Wt[:, 1] = 0.0
    Ws[:, 1] = 0.0
    base = KI.KDInputs(KI.bf16_bits(Ht), KI.bf16_bits(Wt), KI.bf16_bits(Hs), KI.bf16_bits(Ws), None)
    Wt[:, 1] = 8.0
    Ws[:, 1] = -4.0
    shifted = KI.KDInputs(base.H_t, KI.bf16_bits(Wt), base.H_s, KI.bf16_bits(Ws), None)
    r0 = run(base, T=1.0, kind="fkl")
    r1 = run(shifted, T=1.0, kind="fkl")
    assert_kd_close("shifted loss", r1.loss.cpu().numpy(), r0.loss.cpu().numpy().astype(np.float64), 1e-3, 2e-5)
    ref = oracle_run(base, T=1.0, kind="fkl")[0]
    assert_kd_close("loss vs oracle", r1.loss.cpu().numpy(), ref, LOSS_RTOL, LOSS_ATOL)


def test_worked_example_through_gpu():
    """SURVEY §8c golden example (V=4) embedded in a V=1024 problem via the bias column; other logits −1e4."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example_v4.json")))
    V, d = 1024, 64
    H = np.zeros((1, d), np.float32)
    H[0, 0] = 1.0
    Wt = np.zeros((V, d), np.float32)
    Ws = np.zeros((V, d), np.float32)
    Wt[:, 0] = -1e4
    Ws[:, 0] = -1e4
    Wt[:4, 0] = g["z_t"]
    Ws[:4, 0] = g["z_s"]
    for case in g["cases"]:
        inp = KI.KDInputs(KI.bf16_bits(H), KI.bf16_bits(Wt), KI.bf16_bits(H), KI.bf16_bits(Ws), None)
        r = run(inp, T=case["T"], kind=case["kind"], beta=g["beta"])
        assert abs(float(r.loss[0]) - case["loss"]) <= 1e-3 * case["loss"] + 1e-5, case
        # dh_s[0, 0] = Σ_v G_v · W_s[v, 0] with the golden gradient on v < 4 (others ~0)
        ref = float(np.dot(case["grad"], g["z_s"]))
        assert abs(float(r.dh_s[0, 0]) - ref) <= 2e-3 * abs(ref) + 1e-5, (case, float(r.dh_s[0, 0]), ref)


def test_nonfinite_counter():
    inp = KI.make_inputs(300, 128, 64, 700, seed=13)
    bad = inp.H_t.copy()
    bad[[5, 200]] = 0x7F80  # +Inf rows (unmasked) -> non-finite logits -> non-finite loss
    r = run(KI.KDInputs(bad, inp.W_t, inp.H_s, inp.W_s, None), T=1.0, kind="fkl")
    assert int(r.n_nonfinite.item()) == 2


def test_invalid_arguments_rejected():
    k = kd()
    inp = KI.make_inputs(8, 64, 64, 100, seed=1)
    args = [dev_bf16(x) for x in (inp.H_t, inp.W_t, inp.H_s, inp.W_s)]
    with pytest.raises(k.KDError) as e:
        k.fused_fwd_bwd(*args, T=0.0)
    assert e.value.status == 1
    with pytest.raises(k.KDError) as e:
        k.fused_fwd_bwd(*args, kind="jsd", beta=1.0)
    assert e.value.status == 1
    odd = KI.make_inputs(8, 96, 64, 100, seed=1)
    with pytest.raises(k.KDError) as e:
        k.fused_fwd_bwd(*[dev_bf16(x) for x in (odd.H_t, odd.W_t, odd.H_s, odd.W_s)])
    assert e.value.status == 2


# ------------------------------------------------------------------ vocab-sharded entry points (1 GPU, P shards)
@pytest.mark.parametrize("P,kind", [(2, "fkl"), (3, "rkl"), (8, "fkl")])
def test_vocab_sharded_equals_single(P, kind):
    """P vocab shards (128-row granules) run one after another on this GPU: records all-gathered, merged in
    rank order, partial dh (and FKL's partial loss) summed — equals the oracle (the exchange the multi-GPU path
    performs)."""
    from paper_2603_01875_b200.sharding import vocab_shard_bounds
    N, d_t, d_s, V = 520, 256, 128, 5000
    mask = (np.random.default_rng(P).random(N) > 0.2).astype(np.uint8)
    inp = KI.make_inputs(N, d_t, d_s, V, seed=20 + P, mask=mask)
    Ht, Hs, Wt, Ws = dev_bf16(inp.H_t), dev_bf16(inp.H_s), dev_bf16(inp.W_t), dev_bf16(inp.W_s)
    m = torch.from_numpy(mask).cuda()
    bounds = vocab_shard_bounds(V, P)
    recs = torch.stack([kd().vocab_stats(Ht, Wt[a:b], Hs, Ws[a:b], m, vocab=V, v_begin=a, T=1.5, kind=kind)
                        for a, b in bounds])
    dh = torch.zeros(N, d_s, device="cuda")
    dW = torch.zeros(V, d_s, device="cuda")
    losses = []
    for a, b in bounds:
        r = kd().vocab_backward(Ht, Wt[a:b], Hs, Ws[a:b], recs, m, vocab=V, v_begin=a, T=1.5, kind=kind,
                                want_dW=True)
        dh += r.dh_s
        dW[a:b] = r.dW_s
        losses.append(r.loss)
    torch.cuda.synchronize()
    if kind == "rkl":
        for l in losses[1:]:
            assert torch.equal(l, losses[0])  # every rank derives the same loss from the same merged records
        got_loss = losses[0]
    else:  # FKL: each shard returns its partial loss; the caller sums them (kdfused.h kd_vocab_backward)
        got_loss = sum(losses[1:], losses[0].clone())
        assert not torch.equal(losses[0], got_loss)
    loss, dh_ref, dW_ref = oracle_run(inp, T=1.5, kind=kind, want_dW=True)
    assert_kd_close("loss", got_loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", dh.cpu().numpy(), dh_ref)
    assert_grad_close("dW_s", dW.cpu().numpy(), dW_ref)


@pytest.mark.parametrize("P,kind,chunk", [(2, "jsd", 0), (3, "tvd", 0), (4, "jsd", 256)])
def test_vocab_sharded_jsd_tvd_equals_single(P, kind, chunk):
    """JSD/TVD vocab shards: per token chunk, records all-gathered -> kd_vocab_partials -> (K, J) partials
    all-gathered -> kd_vocab_finish (rank-order sums), partial dh summed; equals the oracle.  chunk=256 drives
    three token chunks (the per-chunk protocol sharding.py runs)."""
    from paper_2603_01875_b200.sharding import vocab_shard_bounds
    N, d_t, d_s, V = 520, 256, 128, 5000
    mask = (np.random.default_rng(P).random(N) > 0.2).astype(np.uint8)
    inp = KI.make_inputs(N, d_t, d_s, V, seed=40 + P, mask=mask)
    Ht, Hs, Wt, Ws = dev_bf16(inp.H_t), dev_bf16(inp.H_s), dev_bf16(inp.W_t), dev_bf16(inp.W_s)
    m = torch.from_numpy(mask).cuda()
    bounds = vocab_shard_bounds(V, P)
    step = chunk or N
    dh = torch.zeros(N, d_s, device="cuda")
    dW = torch.zeros(V, d_s, device="cuda")
    loss = torch.zeros(N, device="cuda")
    for t0 in range(0, N, step):
        t1 = min(N, t0 + step)
        sl = slice(t0, t1)
        recs = torch.stack([kd().vocab_stats(Ht[sl], Wt[a:b], Hs[sl], Ws[a:b], m[sl], vocab=V, v_begin=a, T=2.0,
                                             kind=kind, chunk_tokens=t1 - t0) for a, b in bounds])
        parts = [kd().vocab_partials(Ht[sl], Wt[a:b], Hs[sl], Ws[a:b], recs, m[sl], vocab=V, v_begin=a, T=2.0,
                                     kind=kind, beta=0.5, want_dW=True, accumulate_dW=t0 > 0)
                 for a, b in bounds]
        kj_all = torch.stack([kj for kj, _ in parts])
        losses = []
        for (a, b), (_, st) in zip(bounds, parts):
            r = kd().vocab_finish(st, Ht[sl], Wt[a:b], Hs[sl], Ws[a:b], kj_all, m[sl], dW_s=dW[a:b])
            dh[sl] += r.dh_s
            losses.append(r.loss)
        for l in losses[1:]:
            assert torch.equal(l, losses[0])  # every rank sums the same (K, J) partials in the same order
        loss[sl] = losses[0]
    torch.cuda.synchronize()
    loss_ref, dh_ref, dW_ref = oracle_run(inp, T=2.0, kind=kind, beta=0.5, want_dW=True)
    assert_kd_close("loss", loss.cpu().numpy(), loss_ref, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", dh.cpu().numpy(), dh_ref)
    assert_grad_close("dW_s", dW.cpu().numpy(), dW_ref)


@pytest.mark.parametrize("kind", ["fkl", "rkl", "jsd"])
def test_grad_precision_bf16_within_its_bound(kind):
    """KD_GRAD_BF16 (one bf16 G plane, kdfused.h): not parity-grade, so it is held to its own rounding bound.
    Each G entry is rounded once to bf16 (|δ_v| <= 2^-8 |g_v|, the unit roundoff; the residual fix restores the largest exactly),
    so |Δdh_j| <= 2^-8 (|G|·|W_s|)_j and |ΔdW_vj| <= 2^-8 (|G|ᵀ·|H_s|)_vj, plus the north-star terms.  The loss does
    not depend on G: it must stay within the north-star loss tolerance."""
    from oracle.kd_oracle import grad_student_logits, lm_head_logits
    cfg = KI.CONFIGS["c2"]
    W_t, W_s = heads(cfg.vocab, cfg.d_t, cfg.d_s)
    n = 256
    H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1011, head_seed=1000)
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, None)
    T = 2.0 if kind != "fkl" else 1.0
    r = run(inp, T=T, kind=kind, want_dW=True, grad_precision="bf16")
    loss, dh, dW = oracle_run(inp, T=T, kind=kind, want_dW=True)
    Ws64, Hs64 = f64(W_s), f64(H_s)
    G = grad_student_logits(kind, lm_head_logits(f64(H_t), f64(W_t)), lm_head_logits(Hs64, Ws64), T, 0.5)
    bh = 2.0 ** -8 * (np.abs(G) @ np.abs(Ws64))
    bW = 2.0 ** -8 * (np.abs(G).T @ np.abs(Hs64))
    assert_kd_close("loss (bf16 G)", r.loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    for name, got, ref, b in (("dh_s (bf16 G)", r.dh_s, dh, bh), ("dW_s (bf16 G)", r.dW_s, dW, bW)):
        got = got.cpu().numpy().astype(np.float64)
        d = np.abs(got - ref)
        tol = b + GRAD_ATOL + GRAD_RTOL * np.abs(ref)
        i = np.unravel_index(np.argmax(d / tol), d.shape)
        assert np.all(d <= tol), (name, float((d / tol).max()), i, float(got[i]), float(ref[i]), float(b[i]),
                                  int((d > tol).sum()))
    # and it is a real approximation: measurably worse than the split planes somewhere, never better by design
    r2 = run(inp, T=T, kind=kind, want_dW=True)
    e_fast = np.abs(r.dh_s.cpu().numpy() - dh).max()
    e_split = np.abs(r2.dh_s.cpu().numpy() - dh).max()
    assert e_fast >= e_split * 0.5
