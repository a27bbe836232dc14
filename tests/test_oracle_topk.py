"""Pins of the top-k teacher baseline oracle (oracle/kd_topk.py).

Each pin is fixed by something other than the oracle's own formula: the k = V identity with the full-logit
oracle, the k = 1 closed form (p̂ one-hot ⇒ FKL_topk = −ln q_argmax), SPEC's worked examples,
hand-written two-entry softmax on a tiny case, central finite differences of the gradient, and brute-force
sorting for the selection."""
import math

import numpy as np
import pytest

from oracle.kd_oracle import divergence, log_softmax
from oracle.kd_topk import fkl_topk_support, kd_loss_topk, kd_topk_fwd_bwd, teacher_topk


def _rng(s):
    return np.random.default_rng(s)


@pytest.mark.parametrize("kind", ["fkl", "rkl", "jsd", "tvd"])
@pytest.mark.parametrize("T", [1.0, 2.0])
def test_k_equals_V_is_full_logit_kd(kind, T):
    """S:272 "k = V → bitwise equal to kd_loss" (reading: to rounding, 1e-13)."""
    r = _rng(1)
    z_t, z_s = r.normal(0, 3, (6, 37)), r.normal(0, 3, (6, 37))
    np.testing.assert_allclose(kd_loss_topk(kind, z_t, 37, z_s, T=T, beta=0.3), divergence(kind, z_t, z_s, T, 0.3),
                               rtol=1e-13, atol=1e-14)


def test_k1_closed_form():
    """k = 1: p̂ is one-hot at the teacher argmax, so FKL_topk = −ln q_argmax and G = (q − e_argmax)/T."""
    r = _rng(2)
    z_t, z_s = r.normal(0, 2, (5, 50)), r.normal(0, 2, (5, 50))
    T = 1.7
    am = z_t.argmax(axis=1)
    lq = log_softmax(z_s, T)
    np.testing.assert_allclose(kd_loss_topk("fkl", z_t, 1, z_s, T=T), -lq[np.arange(5), am], rtol=1e-13)
    idx, val = teacher_topk(z_t, 1)
    _, g = fkl_topk_support(idx, val, z_s, T)
    want = np.exp(lq)
    want[np.arange(5), am] -= 1.0
    np.testing.assert_allclose(g, want / T, rtol=1e-13, atol=1e-15)


def test_spec_peaked_teacher_k1():
    """k = 1 with a greedy-peaked teacher (one logit +20) → FKL_topk ≈ FKL_full within 1e-3."""
    r = _rng(3)
    z_t = r.normal(0, 1, (8, 200))
    z_t[np.arange(8), r.integers(0, 200, 8)] += 20.0
    z_s = r.normal(0, 1, (8, 200))
    full = divergence("fkl", z_t, z_s, 1.0)
    top = kd_loss_topk("fkl", z_t, 1, z_s, T=1.0)
    assert np.all(np.abs(top - full) < 1e-3)


def test_spec_sweep_breaks_equivalence_and_shrinks_with_k():
    """random logits, V = 64: |FKL_topk(k=8) − FKL_full| > 0, and the mean gap over 100 seeds is
    non-increasing in k (the equivalence P:37 / P:130 says top-k transfer loses)."""
    gaps = {k: [] for k in (1, 2, 4, 8, 16, 32, 64)}
    for s in range(100):
        r = _rng(100 + s)
        z_t, z_s = r.normal(0, 2, (1, 64)), r.normal(0, 2, (1, 64))
        full = divergence("fkl", z_t, z_s, 1.0)[0]
        for k in gaps:
            gaps[k].append(abs(kd_loss_topk("fkl", z_t, k, z_s)[0] - full))
    assert min(gaps[8]) > 0
    means = [np.mean(gaps[k]) for k in sorted(gaps)]
    assert all(a >= b for a, b in zip(means, means[1:]))
    assert means[-1] < 1e-13


def test_two_entry_support_by_hand():
    """V = 5, k = 2, written out with math.exp: p̂ = (e^{a/T}, e^{b/T}) / (e^{a/T} + e^{b/T})."""
    z_t = np.array([[0.3, 2.0, -1.0, 1.5, 0.0]])
    z_s = np.array([[1.0, 0.5, 0.2, -0.3, 0.9]])
    T = 1.3
    ea, eb = math.exp(2.0 / T), math.exp(1.5 / T)
    p1, p3 = ea / (ea + eb), eb / (ea + eb)
    Zs = sum(math.exp(x / T) for x in z_s[0])
    q = [math.exp(x / T) / Zs for x in z_s[0]]
    want = p1 * math.log(p1 / q[1]) + p3 * math.log(p3 / q[3])
    assert abs(kd_loss_topk("fkl", z_t, 2, z_s, T=T)[0] - want) < 1e-14
    idx, _ = teacher_topk(z_t, 2)
    assert idx.tolist() == [[1, 3]]


def test_selection_brute_force_and_ties():
    r = _rng(4)
    z = np.round(r.normal(0, 1, (20, 30)), 1)  # many exact ties
    idx, val = teacher_topk(z, 7)
    for n in range(20):
        want = sorted(range(30), key=lambda v: (-z[n, v], v))[:7]
        assert idx[n].tolist() == want
        assert val[n].tolist() == [z[n, v] for v in want]


def test_gradient_central_differences():
    r = _rng(5)
    z_t, z_s = r.normal(0, 2, (3, 12)), r.normal(0, 2, (3, 12))
    T = 0.8
    idx, val = teacher_topk(z_t, 4)
    _, g = fkl_topk_support(idx, val, z_s, T)
    h = 1e-6
    fd = np.zeros_like(z_s)
    for n in range(3):
        for v in range(12):
            zp, zm = z_s.copy(), z_s.copy()
            zp[n, v] += h
            zm[n, v] -= h
            fd[n, v] = (fkl_topk_support(idx, val, zp, T)[0][n] - fkl_topk_support(idx, val, zm, T)[0][n]) / (2 * h)
    np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-9)


def test_student_side_fd_through_the_head():
    """kd_topk_fwd_bwd: dh_s and dW_s are the derivatives of Σ_n mask_n FKL_topk through z_s = h_s·W_sᵀ."""
    r = _rng(6)
    N, d, V = 4, 5, 9
    h_s, W_s = r.normal(0, 1, (N, d)), r.normal(0, 1, (V, d))
    z_t = r.normal(0, 2, (N, V))
    idx, val = teacher_topk(z_t, 3)
    mask = np.array([1, 0, 1, 1], np.uint8)
    T = 1.4
    loss, dh, dW = kd_topk_fwd_bwd(h_s, W_s, idx, val, mask, T=T, want_dW=True)
    assert loss[1] == 0 and np.all(dh[1] == 0)

    def total(hs, Ws):
        return kd_topk_fwd_bwd(hs, Ws, idx, val, mask, T=T)[0].sum()
    eps = 1e-6
    for (n, j) in [(0, 0), (2, 3), (3, 4)]:
        hp, hm = h_s.copy(), h_s.copy()
        hp[n, j] += eps
        hm[n, j] -= eps
        assert abs((total(hp, W_s) - total(hm, W_s)) / (2 * eps) - dh[n, j]) < 1e-7
    for (v, j) in [(0, 1), (4, 2), (8, 0)]:
        wp, wm = W_s.copy(), W_s.copy()
        wp[v, j] += eps
        wm[v, j] -= eps
        assert abs((total(h_s, wp) - total(h_s, wm)) / (2 * eps) - dW[v, j]) < 1e-7


def test_rkl_topk_is_infinite_off_support():
    """Why the GPU builds FKL only (reading R17): RKL against a truncated teacher is +inf for k < V."""
    r = _rng(7)
    z_t, z_s = r.normal(0, 1, (2, 20)), r.normal(0, 1, (2, 20))
    assert np.all(np.isinf(kd_loss_topk("rkl", z_t, 5, z_s)))
