"""Dense fp64 oracle for the KDFlow student-side hot path.  TEST INFRASTRUCTURE ONLY.

The method (§3.2): the teacher ships only its final hidden states
``H_t``; the student recomputes the full teacher logits with the teacher's LM head
 and computes the KD divergence against its own logits.  The paper states that
this is "mathematically equivalent" to full-logit KD, so the oracle
is that plain full-logit definition written out:

    Z_t = H_t · W_tᵀ ,  Z_s = H_s · W_sᵀ                      (S:159-167 apply_lm_head)
    ln p = logsoftmax(Z_t / T) ,  ln q = logsoftmax(Z_s / T)
    FKL = Σ p (ln p − ln q)   RKL = Σ q (ln q − ln p)           (P:153 names them; S:260 defines)
    JSD_β = β KL(p‖m) + (1−β) KL(q‖m),  m = βp + (1−β)q         (reading R4)
    TVD = ½ Σ |p − q|
    loss_n = mask_n ℓ_n ;  G = loss_scale · mask_n · ∂ℓ_n/∂z_s  (reading R3)
    dL/dh_s = G · W_s ;  dL/dW_s = Gᵀ · H_s                      ("backward passes")

Gradients w.r.t. the student logits (teacher constant) are the analytic forms
derived in DESIGN.md "Readings" R5 (softmax chain rule  ∂ℓ/∂b_v = q_v (g_v − Σ_u q_u g_u),
g = ∂ℓ/∂q, b = z_s/T):

    FKL: (q − p)/T            RKL: q (ln q − ln p − RKL)/T
    JSD: (1−β) q (ln q − ln m − KL(q‖m))/T      TVD: ½ q (s − Σ q s)/T,  s = sign(q − p)

Everything is numpy float64; natural logs; no T² factor (reading R2).  Matrices are
row-major with heads in ``nn.Linear`` layout ``[V, d]`` (reading R7).  Masked rows are
never read (reading R9).
"""
from __future__ import annotations

import numpy as np

KINDS = ("fkl", "rkl", "jsd", "tvd")


# ----------------------------------------------------------------------------- primitives
def lm_head_logits(h: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Z = h · Wᵀ in fp64.  P:135 ("recomputes the full logit distributions using the
    teacher's language model head").  h: [N, d], W: [V, d] -> Z: [N, V]."""
    return np.asarray(h, dtype=np.float64) @ np.asarray(W, dtype=np.float64).T


def log_softmax(z: np.ndarray, T: float) -> np.ndarray:
    """Row-wise ln softmax(z / T), max-subtracted."""
    if not T > 0:
        raise ValueError("temperature must be > 0 (S:261)")
    a = np.asarray(z, dtype=np.float64) / T
    m = a.max(axis=-1, keepdims=True)
    return a - m - np.log(np.exp(a - m).sum(axis=-1, keepdims=True))


def _log_mixture(lp: np.ndarray, lq: np.ndarray, beta: float) -> np.ndarray:
    """ln m with m = βp + (1−β)q, evaluated as logaddexp(ln β + ln p, ln(1−β) + ln q)."""
    return np.logaddexp(np.log(beta) + lp, np.log1p(-beta) + lq)


def _check_beta(beta: float):
    if not (0.0 < beta < 1.0):
        raise ValueError("jsd_beta must lie in (0, 1) (reading R4)")


def divergence(kind: str, z_t: np.ndarray, z_s: np.ndarray, T: float, beta: float = 0.5) -> np.ndarray:
    """Per-row divergence ℓ_n in nats.  P:153 names FKL/RKL/JSD/TVD; S:260 definitions."""
    lp, lq = log_softmax(z_t, T), log_softmax(z_s, T)
    p, q = np.exp(lp), np.exp(lq)
    if kind == "fkl":
        return (p * (lp - lq)).sum(axis=-1)
    if kind == "rkl":
        return (q * (lq - lp)).sum(axis=-1)
    if kind == "jsd":
        _check_beta(beta)
        lm = _log_mixture(lp, lq, beta)
        return beta * (p * (lp - lm)).sum(axis=-1) + (1.0 - beta) * (q * (lq - lm)).sum(axis=-1)
    if kind == "tvd":
        return 0.5 * np.abs(p - q).sum(axis=-1)
    raise ValueError(f"unknown divergence kind {kind!r}")


def grad_student_logits(kind: str, z_t: np.ndarray, z_s: np.ndarray, T: float,
                        beta: float = 0.5) -> np.ndarray:
    """∂ℓ_n/∂z_s[n, v] (teacher constant; FKL form S:265; others reading R5)."""
    lp, lq = log_softmax(z_t, T), log_softmax(z_s, T)
    p, q = np.exp(lp), np.exp(lq)
    if kind == "fkl":
        return (q - p) / T
    if kind == "rkl":
        rkl = (q * (lq - lp)).sum(axis=-1, keepdims=True)
        return q * (lq - lp - rkl) / T
    if kind == "jsd":
        _check_beta(beta)
        lm = _log_mixture(lp, lq, beta)
        K = (q * (lq - lm)).sum(axis=-1, keepdims=True)          # KL(q‖m)
        return (1.0 - beta) * q * (lq - lm - K) / T
    if kind == "tvd":
        s = np.sign(q - p)
        return 0.5 * q * (s - (q * s).sum(axis=-1, keepdims=True)) / T
    raise ValueError(f"unknown divergence kind {kind!r}")


# ----------------------------------------------------------------------------- fused composition
def kd_fused_fwd_bwd(h_t, W_t, h_s, W_s, mask=None, *, T: float = 1.0, kind: str = "fkl",
                     beta: float = 0.5, loss_scale: float = 1.0, want_dW: bool = False,
                     row_batch: int = 64):
    """The whole hot path, plain definition (no vocabulary chunking, fp64).

    Inputs are float arrays (the exact values of the bf16 inputs).  Returns
    ``(loss [N], dh_s [N, d_s], dW_s [V, d_s] or None)`` with
    ``loss_n = mask_n ℓ_n``, ``dh_s = G · W_s``, ``dW_s = Gᵀ · H_s``,
    ``G = loss_scale · mask_n · ∂ℓ_n/∂z_s``.

    Rows with mask 0 are never read.  Token rows are processed ``row_batch`` at a time only to
    bound memory; each row is independent, and dW_s sums the per-batch products in row order.
    """
    if not T > 0:
        raise ValueError("temperature must be > 0 (S:261)")
    if kind not in KINDS:
        raise ValueError(f"unknown divergence kind {kind!r}")
    N = h_t.shape[0]
    if h_s.shape[0] != N or W_t.shape[0] != W_s.shape[0] or h_t.shape[1] != W_t.shape[1] \
            or h_s.shape[1] != W_s.shape[1]:
        raise ValueError("shape mismatch (S:261)")
    V, d_s = W_s.shape
    W_t64 = np.asarray(W_t, dtype=np.float64)
    W_s64 = np.asarray(W_s, dtype=np.float64)
    rows = np.arange(N) if mask is None else np.flatnonzero(np.asarray(mask) != 0)
    loss = np.zeros(N, dtype=np.float64)
    dh = np.zeros((N, d_s), dtype=np.float64)
    dW = np.zeros((V, d_s), dtype=np.float64) if want_dW else None
    for i in range(0, rows.size, row_batch):
        r = rows[i:i + row_batch]
        hs = np.asarray(h_s[r], dtype=np.float64)
        z_t = lm_head_logits(h_t[r], W_t64)
        z_s = lm_head_logits(hs, W_s64)
        loss[r] = divergence(kind, z_t, z_s, T, beta)
        G = loss_scale * grad_student_logits(kind, z_t, z_s, T, beta)
        dh[r] = G @ W_s64
        if want_dW:
            dW += G.T @ hs
    return loss, dh, dW


def kd_loss_from_logits(z_t, z_s, mask=None, *, T=1.0, kind="fkl", beta=0.5, loss_scale=1.0):
    """Full-logit KD (S:256-265 kd_loss): per-row loss and G = loss_scale·mask·∂ℓ/∂z_s."""
    z_t = np.asarray(z_t, dtype=np.float64)
    z_s = np.asarray(z_s, dtype=np.float64)
    m = np.ones(z_t.shape[0]) if mask is None else np.asarray(mask, dtype=np.float64)
    loss = m * divergence(kind, z_t, z_s, T, beta)
    G = loss_scale * m[:, None] * grad_student_logits(kind, z_t, z_s, T, beta)
    return loss, G


def teacher_stats(h_t, W_t, T: float):
    """Per-row (max, LSE) of Z_t/T — the quantities a vocab-sharded exchange carries."""
    a = lm_head_logits(h_t, W_t) / T
    m = a.max(axis=-1)
    return m, m + np.log(np.exp(a - m[:, None]).sum(axis=-1))
