"""Top-k teacher transfer — the prior-art baseline KDFlow argues against.  TEST INFRASTRUCTURE ONLY.

PAPER.md P:37 "only transferring the top-k logits breaks the mathematical equivalence of the loss
function"; "only transferring the top-k logits saves bandwidth but inevitably undermines the
mathematical equivalence of distillation"; Table 1 lists "top-k" for two of the compared
frameworks.  SPEC S:267-271 (``kd_loss_topk``) fixes the construction this oracle writes out:

    K_n   = the k vocabulary indices of the largest teacher logits of row n
            (ties: the lower index first — reading R17)
    p̂_v  = exp(z_t,v / T) / Σ_{u ∈ K_n} exp(z_t,u / T)   for v ∈ K_n,   0 otherwise
            ("renormalized over the k support; off-support teacher mass treated as 0")
    q     = softmax(z_s / T) over the FULL vocabulary (the student's own head, nothing truncated)
    FKL_topk = Σ_{v ∈ K_n} p̂_v (ln p̂_v − ln q_v)                     ("same loss formulas")
    ∂FKL_topk/∂z_s = (q − p̂)/T                                        (Σ p̂ = 1; the FKL form of S:265)

Only FKL is built on the GPU (kd_topk_fwd_bwd, reading R17): RKL = Σ q ln(q/p̂) is +∞ whenever the
student puts mass off the support (p̂ = 0 there), for any k < V.  The oracle still evaluates every kind
(``divergence`` of kd_oracle on the rebuilt p̂) so the SPEC examples can be pinned.

Plain fp64 numpy, one row at a time where it matters; shares nothing with the CUDA path.
"""
from __future__ import annotations

import numpy as np

from .kd_oracle import lm_head_logits, log_softmax


def teacher_topk(z_t: np.ndarray, k: int):
    """Row-wise top-k of the teacher logits: (idx [N, k] int64, val [N, k] fp64), largest first.

    Ties broken toward the lower vocabulary index (a stable sort of −z)."""
    z_t = np.asarray(z_t, dtype=np.float64)
    V = z_t.shape[-1]
    if not 1 <= k <= V:
        raise ValueError("need 1 <= k <= V (S:268)")
    order = np.argsort(-z_t, axis=-1, kind="stable")[:, :k]
    return order, np.take_along_axis(z_t, order, axis=-1)


def topk_teacher_logprobs(idx: np.ndarray, val: np.ndarray, V: int, T: float) -> np.ndarray:
    """ln p̂ over the full vocabulary: log-softmax of val/T on the support, −inf elsewhere."""
    if not T > 0:
        raise ValueError("temperature must be > 0 (S:261)")
    a = np.asarray(val, dtype=np.float64) / T
    m = a.max(axis=-1, keepdims=True)
    lp_k = a - m - np.log(np.exp(a - m).sum(axis=-1, keepdims=True))
    lp = np.full((a.shape[0], V), -np.inf)
    np.put_along_axis(lp, np.asarray(idx), lp_k, axis=-1)
    return lp


def fkl_topk_support(idx, val, z_s, T: float):
    """FKL_topk per row and its gradient (q − p̂)/T for a GIVEN support (idx, teacher logits val)."""
    z_s = np.asarray(z_s, dtype=np.float64)
    lq = log_softmax(z_s, T)
    lp = topk_teacher_logprobs(idx, val, z_s.shape[-1], T)
    p = np.exp(lp)  # exactly 0 off the support
    on = np.isfinite(lp)
    loss = np.where(on, p * (np.where(on, lp, 0.0) - lq), 0.0).sum(axis=-1)
    return loss, (np.exp(lq) - p) / T


def kd_loss_topk(kind: str, z_t, k: int, z_s, mask=None, *, T: float = 1.0, beta: float = 0.5):
    """SPEC S:267-271 ``kd_loss_topk``: the divergence of the rebuilt teacher p̂ against the full student q."""
    from .kd_oracle import _log_mixture
    z_t = np.asarray(z_t, dtype=np.float64)
    idx, val = teacher_topk(z_t, k)
    lp = topk_teacher_logprobs(idx, val, z_t.shape[-1], T)
    lq = log_softmax(z_s, T)
    p, q = np.exp(lp), np.exp(lq)
    on = p > 0
    lp0 = np.where(on, lp, 0.0)
    if kind == "fkl":
        ell = np.where(on, p * (lp0 - lq), 0.0).sum(axis=-1)
    elif kind == "rkl":
        with np.errstate(invalid="ignore"):
            ell = (q * (lq - lp)).sum(axis=-1)  # +inf as soon as q > 0 off the support
    elif kind == "jsd":
        lm = _log_mixture(lp, lq, beta)
        ell = beta * np.where(on, p * (lp0 - lm), 0.0).sum(axis=-1) + (1 - beta) * (q * (lq - lm)).sum(axis=-1)
    elif kind == "tvd":
        ell = 0.5 * np.abs(p - q).sum(axis=-1)
    else:
        raise ValueError(f"unknown divergence kind {kind!r}")
    m = np.ones(z_t.shape[0]) if mask is None else np.asarray(mask, dtype=np.float64)
    return m * ell


def kd_topk_fwd_bwd(h_s, W_s, idx, val, mask=None, *, T: float = 1.0, loss_scale: float = 1.0,
                    want_dW: bool = False, row_batch: int = 64):
    """The student side of top-k KD (FKL), plain definition: the teacher shipped (idx, val) per row; the student
    computes z_s = h_s·W_sᵀ, FKL_topk and G = loss_scale·mask·(q − p̂)/T; dh_s = G·W_s, dW_s = Gᵀ·h_s
    ("backward passes").  Rows with mask 0 are never read.  Returns (loss [N], dh_s [N, d_s], dW_s or None)."""
    N = h_s.shape[0]
    V, d_s = W_s.shape
    W64 = np.asarray(W_s, dtype=np.float64)
    rows = np.arange(N) if mask is None else np.flatnonzero(np.asarray(mask) != 0)
    loss = np.zeros(N)
    dh = np.zeros((N, d_s))
    dW = np.zeros((V, d_s)) if want_dW else None
    for i in range(0, rows.size, row_batch):
        r = rows[i:i + row_batch]
        hs = np.asarray(h_s[r], dtype=np.float64)
        ell, g = fkl_topk_support(np.asarray(idx)[r], np.asarray(val)[r], lm_head_logits(hs, W64), T)
        loss[r] = ell
        G = loss_scale * g
        dh[r] = G @ W64
        if want_dW:
            dW += G.T @ hs
    return loss, dh, dW
