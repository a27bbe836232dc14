"""Pins for the fp64 oracle (-m "not gpu").

Each test ties ``oracle/`` to something other than itself: a worked example computed
independently at 40 digits (tests/golden), central finite differences, closed forms,
bounds, identities, and an mpmath brute force with pure-Python loops.  Citations:
P:n = PAPER.md, S:n = SPEC.md, SURVEY §8c.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import kd_oracle as O
from oracle import kd_blockwise as B

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_example_v4.json")
KINDS3 = ("fkl", "rkl", "jsd")


def _rand(rng, *shape, scale=1.0):
    return rng.standard_normal(shape) * scale


# ---------------------------------------------------------------- worked example (golden)
def test_worked_example_golden():
    g = json.load(open(GOLDEN))
    zt = np.array([g["z_t"]])
    zs = np.array([g["z_s"]])
    for case in g["cases"]:
        loss, G = O.kd_loss_from_logits(zt, zs, T=case["T"], kind=case["kind"], beta=g["beta"])
        assert abs(loss[0] - case["loss"]) <= g["tolerance"], case
        np.testing.assert_allclose(G[0], case["grad"], rtol=0, atol=g["tolerance"])
        assert abs(G[0].sum()) < 1e-15


# ---------------------------------------------------------------- mpmath brute force
def _mp_case(zt, zs, T, kind, beta):
    """Independent 50-digit evaluation with Python loops (definitions)."""
    mpmath.mp.dps = 50
    a = [mpmath.mpf(float(x)) / T for x in zt]
    b = [mpmath.mpf(float(x)) / T for x in zs]
    Zp = mpmath.fsum(mpmath.e ** x for x in a)
    Zq = mpmath.fsum(mpmath.e ** x for x in b)
    p = [mpmath.e ** x / Zp for x in a]
    q = [mpmath.e ** x / Zq for x in b]
    if kind == "fkl":
        return mpmath.fsum(pi * mpmath.log(pi / qi) for pi, qi in zip(p, q))
    if kind == "rkl":
        return mpmath.fsum(qi * mpmath.log(qi / pi) for pi, qi in zip(p, q))
    if kind == "jsd":
        m = [beta * pi + (1 - beta) * qi for pi, qi in zip(p, q)]
        return beta * mpmath.fsum(pi * mpmath.log(pi / mi) for pi, mi in zip(p, m)) + \
            (1 - beta) * mpmath.fsum(qi * mpmath.log(qi / mi) for qi, mi in zip(q, m))
    return mpmath.fsum(abs(pi - qi) for pi, qi in zip(p, q)) / 2


@pytest.mark.parametrize("kind", O.KINDS)
def test_mpmath_bruteforce_through_lm_heads(kind):
    """Whole composition incl. the LM-head matmuls (catches transposed operands)."""
    rng = np.random.default_rng(11)
    N, dt, ds, V = 3, 5, 4, 7
    ht, hs = _rand(rng, N, dt), _rand(rng, N, ds)
    Wt, Ws = _rand(rng, V, dt), _rand(rng, V, ds)
    T, beta = 1.7, 0.3
    loss, _, _ = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, T=T, kind=kind, beta=beta)
    for n in range(N):
        zt = [sum(ht[n, k] * Wt[v, k] for k in range(dt)) for v in range(V)]
        zs = [sum(hs[n, k] * Ws[v, k] for k in range(ds)) for v in range(V)]
        ref = _mp_case(zt, zs, T, kind, beta)
        assert abs(loss[n] - float(ref)) <= 1e-13 * max(1.0, abs(float(ref)))


# ---------------------------------------------------------------- finite differences
@pytest.mark.parametrize("kind", O.KINDS)
@pytest.mark.parametrize("T", [0.5, 1.0, 2.0, 3.7])
def test_grad_logits_central_fd(kind, T):
    """∂ℓ/∂z_s vs central differences."""
    rng = np.random.default_rng(int(T * 10) + len(kind))
    for trial in range(4):
        V = int(rng.integers(2, 24))
        zt, zs = _rand(rng, 1, V, scale=2), _rand(rng, 1, V, scale=2)
        beta = float(rng.choice([0.2, 0.5, 0.8]))
        G = O.grad_student_logits(kind, zt, zs, T, beta)[0]
        h = 1e-6
        fd = np.zeros(V)
        for v in range(V):
            zp, zm = zs.copy(), zs.copy()
            zp[0, v] += h
            zm[0, v] -= h
            fd[v] = (O.divergence(kind, zt, zp, T, beta)[0] - O.divergence(kind, zt, zm, T, beta)[0]) / (2 * h)
        if kind == "tvd":  # skip kinks |p - q| ~ 0
            p = np.exp(O.log_softmax(zt, T))[0]
            q = np.exp(O.log_softmax(zs, T))[0]
            if np.min(np.abs(p - q)) < 1e-5:
                continue
        np.testing.assert_allclose(G, fd, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("kind", KINDS3 + ("tvd",))
def test_grad_hidden_and_head_central_fd(kind):
    """dL/dh_s and dL/dW_s through the LM head, L = loss_scale·Σ mask·ℓ."""
    rng = np.random.default_rng(5)
    N, dt, ds, V = 4, 6, 5, 9
    ht, hs = _rand(rng, N, dt), _rand(rng, N, ds)
    Wt, Ws = _rand(rng, V, dt), _rand(rng, V, ds)
    mask = np.array([1, 0, 1, 1], dtype=np.uint8)
    kw = dict(T=1.3, kind=kind, beta=0.4, loss_scale=0.7)
    _, dh, dW = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, mask, want_dW=True, **kw)

    def L(hs_, Ws_):
        loss, _, _ = O.kd_fused_fwd_bwd(ht, Wt, hs_, Ws_, mask, **kw)
        return kw["loss_scale"] * loss.sum()

    h = 1e-6
    fd_h = np.zeros_like(hs)
    for i in range(N):
        for j in range(ds):
            a, b = hs.copy(), hs.copy()
            a[i, j] += h
            b[i, j] -= h
            fd_h[i, j] = (L(a, Ws) - L(b, Ws)) / (2 * h)
    fd_W = np.zeros_like(Ws)
    for i in range(V):
        for j in range(ds):
            a, b = Ws.copy(), Ws.copy()
            a[i, j] += h
            b[i, j] -= h
            fd_W[i, j] = (L(hs, a) - L(hs, b)) / (2 * h)
    tol = dict(rtol=1e-5, atol=1e-7) if kind != "tvd" else dict(rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(dh, fd_h, **tol)
    np.testing.assert_allclose(dW, fd_W, **tol)
    assert np.all(dh[1] == 0.0)


# ---------------------------------------------------------------- identities, bounds, closed forms
@pytest.mark.parametrize("kind", O.KINDS)
def test_identical_logits_zero(kind):
    """KL(p‖p)=0 etc. and zero gradient (self-distillation P:64)."""
    rng = np.random.default_rng(3)
    z = _rand(rng, 5, 33, scale=3)
    loss, G = O.kd_loss_from_logits(z, z, T=1.5, kind=kind)
    assert np.all(np.abs(loss) < 1e-14)
    assert np.all(np.abs(G) < 1e-15)


@pytest.mark.parametrize("beta", [0.2, 0.5, 0.8])
def test_bounds_nonneg_jsd_tvd(beta):
    """ℓ ≥ 0; JSD_β ≤ H(β) (= ln 2 at ½); TVD ≤ 1."""
    rng = np.random.default_rng(4)
    zt, zs = _rand(rng, 200, 17, scale=6), _rand(rng, 200, 17, scale=6)
    hb = -beta * math.log(beta) - (1 - beta) * math.log(1 - beta)
    for kind in O.KINDS:
        l = O.divergence(kind, zt, zs, 1.0, beta)
        assert np.all(l >= -1e-15)
    assert np.all(O.divergence("jsd", zt, zs, 1.0, beta) <= hb + 1e-15)
    assert np.all(O.divergence("tvd", zt, zs, 1.0) <= 1 + 1e-15)


def test_v2_saturation():
    """V=2, logits (±30, ∓30): JSD → ln 2, TVD → 1 within 1e-4; general β → H(β)."""
    zt = np.array([[30.0, -30.0]])
    zs = np.array([[-30.0, 30.0]])
    assert abs(O.divergence("jsd", zt, zs, 1.0, 0.5)[0] - math.log(2)) < 1e-4
    assert abs(O.divergence("tvd", zt, zs, 1.0)[0] - 1.0) < 1e-4
    b = 0.2
    assert abs(O.divergence("jsd", zt, zs, 1.0, b)[0] - (-b * math.log(b) - (1 - b) * math.log(1 - b))) < 1e-4


def test_uniform_teacher_closed_form():
    """H_t = 0 ⇒ p uniform ⇒ FKL = −ln V − (1/V) Σ_v ln q_v."""
    rng = np.random.default_rng(8)
    N, dt, ds, V = 6, 8, 7, 50
    ht = np.zeros((N, dt))
    hs, Wt, Ws = _rand(rng, N, ds), _rand(rng, V, dt), _rand(rng, V, ds)
    T = 1.6
    loss, _, _ = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, T=T, kind="fkl")
    zs = hs @ Ws.T / T
    lq = zs - np.log(np.exp(zs).sum(axis=1, keepdims=True))  # tiny |z|, no max shift needed
    ref = -math.log(V) - lq.mean(axis=1)
    np.testing.assert_allclose(loss, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("kind", O.KINDS)
def test_shift_and_temperature_identities(kind):
    """Shift invariance and softmax(z, T) = softmax(z/T, 1)."""
    rng = np.random.default_rng(9)
    zt, zs = _rand(rng, 4, 19, scale=2), _rand(rng, 4, 19, scale=2)
    c = rng.standard_normal((4, 1)) * 50
    l0 = O.divergence(kind, zt, zs, 1.3)
    np.testing.assert_allclose(O.divergence(kind, zt + c, zs - c, 1.3), l0, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(O.divergence(kind, zt / 1.3, zs / 1.3, 1.0), l0, rtol=1e-12, atol=1e-14)
    with pytest.raises(ValueError):
        O.divergence(kind, zt, zs, 0.0)


def test_gradient_rowsum_and_constant_column():
    """Σ_v ∂ℓ/∂z_v = 0 ⇒ a constant column j of W_s gives dh[:, j] = 0 and Σ_v dW[v,:] = 0."""
    rng = np.random.default_rng(10)
    N, dt, ds, V = 8, 6, 5, 40
    ht, hs, Wt, Ws = _rand(rng, N, dt), _rand(rng, N, ds), _rand(rng, V, dt), _rand(rng, V, ds)
    Ws[:, 2] = 0.37
    for kind in O.KINDS:
        _, dh, dW = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, T=1.1, kind=kind, want_dW=True)
        assert np.max(np.abs(dh[:, 2])) < 1e-14
        assert np.max(np.abs(dW.sum(axis=0))) < 1e-13


def test_mask_rows_never_read():
    """Masked rows: loss 0, gradient rows exactly 0, and NaN garbage there changes nothing
    (S:248-251)."""
    rng = np.random.default_rng(12)
    N, dt, ds, V = 7, 6, 5, 30
    ht, hs, Wt, Ws = _rand(rng, N, dt), _rand(rng, N, ds), _rand(rng, V, dt), _rand(rng, V, ds)
    mask = np.array([1, 0, 1, 0, 0, 1, 1], dtype=np.uint8)
    out0 = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, mask, kind="rkl", want_dW=True)
    ht2, hs2 = ht.copy(), hs.copy()
    ht2[mask == 0] = np.nan
    hs2[mask == 0] = np.inf
    out1 = O.kd_fused_fwd_bwd(ht2, Wt, hs2, Ws, mask, kind="rkl", want_dW=True)
    for a, b in zip(out0, out1):
        assert np.array_equal(a, b)
    assert np.all(out0[0][mask == 0] == 0) and np.all(out0[1][mask == 0] == 0)


def test_mean_reduction_matches_spec():
    """loss_scale = 1/max(1, Σmask) gives the SPEC's mean-over-unmasked scalar."""
    rng = np.random.default_rng(13)
    N, d, V = 6, 5, 11
    ht, hs, Wt, Ws = _rand(rng, N, d), _rand(rng, N, d), _rand(rng, V, d), _rand(rng, V, d)
    mask = np.array([1, 1, 0, 1, 0, 1], dtype=np.uint8)
    loss, dh, _ = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, mask, loss_scale=1 / 4)
    zt, zs = ht @ Wt.T, hs @ Ws.T
    l_all, G = O.kd_loss_from_logits(zt, zs, mask, loss_scale=1 / 4)
    assert abs(loss.sum() / 4 - l_all.sum() / 4) < 1e-15
    np.testing.assert_allclose(dh, G @ Ws, rtol=1e-13, atol=1e-16)
    # FKL gradient = (q − p)/N_unmasked
    p = np.exp(O.log_softmax(zt, 1.0))
    q = np.exp(O.log_softmax(zs, 1.0))
    np.testing.assert_allclose(G, (q - p) / 4 * mask[:, None], rtol=1e-12, atol=1e-16)


# ---------------------------------------------------------------- dense ≡ blockwise ≡ sharded
@pytest.mark.parametrize("kind", O.KINDS)
@pytest.mark.parametrize("shards,n_split,order", [(1, 1, "sequential"), (1, 5, "tree"),
                                                  (2, 3, "sequential"), (3, 1, "tree"),
                                                  (8, 2, "sequential")])
def test_dense_equals_blockwise(kind, shards, n_split, order):
    """Online-LSE records + merge operator reproduce the dense definition (P:136 equivalence)."""
    rng = np.random.default_rng(shards * 10 + n_split)
    N, dt, ds, V = 9, 12, 8, 250
    ht, hs = _rand(rng, N, dt, scale=1.5), _rand(rng, N, ds, scale=1.5)
    Wt, Ws = _rand(rng, V, dt), _rand(rng, V, ds)
    ht[:, 0] = 1.0
    hs[:, 0] = 1.0
    Wt[:, 0] += 25.0  # shared large offset: stresses cancellation in the merge
    Ws[:, 0] += 25.0
    mask = (rng.random(N) > 0.3).astype(np.uint8)
    kw = dict(T=1.7, kind=kind, beta=0.35, loss_scale=0.9, want_dW=True)
    d = O.kd_fused_fwd_bwd(ht, Wt, hs, Ws, mask, **kw)
    b = B.kd_blockwise(ht, Wt, hs, Ws, mask, n_shards=shards, n_split=n_split, granule=8,
                       merge_order=order, **kw)
    for x, y in zip(d, b):
        np.testing.assert_allclose(y, x, rtol=1e-12, atol=1e-13)


def test_merge_identity_and_order():
    rng = np.random.default_rng(14)
    a, b = _rand(rng, 3, 40), _rand(rng, 3, 40)
    R = B.block_record(a, b)
    assert B.merge(B.EMPTY, R) is R and B.merge(R, B.EMPTY) is R
    assert B.block_record(a[:, :0], b[:, :0]) is B.EMPTY
    parts = [B.block_record(a[:, i:i + 7], b[:, i:i + 7]) for i in range(0, 40, 7)]
    fwd = parts[0]
    for p in parts[1:]:
        fwd = B.merge(fwd, p)
    rev = parts[-1]
    for p in parts[-2::-1]:
        rev = B.merge(p, rev)
    for x, y, z in zip(fwd, rev, R):
        np.testing.assert_allclose(x, z, rtol=1e-13)
        np.testing.assert_allclose(y, z, rtol=1e-13)


def test_vocab_bounds_granules():
    """V = 151936 = 128·1187 splits into 128-row granules at P = 2/4/8 (SURVEY finding 8)."""
    V = 151936
    for P in (2, 4, 8):
        b = B.vocab_bounds(V, P, 128)
        assert b[0][0] == 0 and b[-1][1] == V
        assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
        assert all(v0 % 128 == 0 for v0, _ in b)
        sizes = [v1 - v0 for v0, v1 in b]
        assert max(sizes) - min(sizes) <= 128


def test_comm_volume_footnote():
    """P:37 footnote: 128 × 4096 × 151936 × 2 bytes ≈ 160 GB (decimal)."""
    from kd_inputs import comm_volume_bytes
    v = comm_volume_bytes(128, 4096)
    assert v == 159_316_443_136
    assert round(v / 1e9) == 159 and abs(v / 1e9 - 160) < 1
    assert abs(151936 / 4096 - 37.09) < 0.01  # P:133 "4096 vs 151936"


# ---------------------------------------------------------------- teacher_stats (the per-row (max, LSE) record)
@pytest.mark.parametrize("T", [0.5, 1.0, 2.0])
def test_teacher_stats_mpmath_bruteforce(T):
    """oracle.teacher_stats against an independent 50-digit evaluation with Python loops: the dot products
    h·W[v] (catches a transposed operand), the max of z/T and ln Σ_v e^{z_v/T} (the record the
    vocab-sharded exchange and kd_teacher_lse carry)."""
    rng = np.random.default_rng(int(T * 10))
    N, d, V = 3, 5, 7
    h = _rand(rng, N, d)
    W = _rand(rng, V, d, scale=2.0)
    m, lse = O.teacher_stats(h, W, T)
    mpmath.mp.dps = 50
    for n in range(N):
        z = [mpmath.fsum(mpmath.mpf(float(h[n, k])) * mpmath.mpf(float(W[v, k])) for k in range(d)) / T
             for v in range(V)]
        zmax = max(z)
        ref = zmax + mpmath.log(mpmath.fsum(mpmath.e ** (x - zmax) for x in z))
        assert abs(m[n] - float(zmax)) <= 1e-14 * max(1.0, abs(float(zmax)))
        assert abs(lse[n] - float(ref)) <= 1e-13 * max(1.0, abs(float(ref)))


def test_teacher_stats_closed_forms():
    """Zero hidden row: every logit 0, so max = 0 and LSE = ln V at any T.  One-hot h = e_j with a head column
    holding k copies of c and the rest −∞-like: LSE = c/T + ln k.  LSE − max lies in [0, ln V]."""
    V, d = 1000, 8
    W = np.random.default_rng(3).standard_normal((V, d))
    for T in (0.5, 1.0, 3.0):
        m, lse = O.teacher_stats(np.zeros((2, d)), W, T)
        np.testing.assert_array_equal(m, 0.0)
        np.testing.assert_allclose(lse, math.log(V), rtol=0, atol=1e-12)
    W2 = np.full((V, d), -1e4)
    W2[:13, 2] = 3.0
    h = np.zeros((1, d))
    h[0, 2] = 1.0
    m, lse = O.teacher_stats(h, W2, 2.0)
    assert m[0] == 1.5
    assert abs(lse[0] - (1.5 + math.log(13))) < 1e-12
    rng = np.random.default_rng(4)
    m, lse = O.teacher_stats(rng.standard_normal((20, d)), W * 5, 0.7)
    assert np.all(lse >= m) and np.all(lse - m <= math.log(V) + 1e-12)
