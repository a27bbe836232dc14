"""Vocabulary-chunked formulation (online log-sum-exp records).  TEST INFRASTRUCTURE ONLY.

This is the "second opinion" formulation of the same quantity ``kd_oracle``
defines.  It is NOT the reference: tests pin it to ``kd_oracle.kd_fused_fwd_bwd`` to
<= 1e-12, which checks, on CPU, the algebra that a vocabulary-sharded implementation must
use to combine per-shard partial statistics (north star: "chunked over the vocabulary
with an online log-sum-exp"; P:135-136 equivalence).  It shares no code with the CUDA
path (which works in base 2 and fp32; this works in base e and fp64).

Record of a vocabulary range R for one row, with a = z_t/T, b = z_s/T (FKL roles):
    m_t = max_R a,  m_s = max_R b,  S_t = Σ_R e^{a−m_t},  S_s = Σ_R e^{b−m_s},
    U   = Σ_R e^{a−m_t} ((a − m_t) − (b − m_s))
Then FKL = U/S_t − ln S_t + ln S_s.  For RKL the roles of (a, b) are swapped.
Merge A ⊕ B (reading R10): M = max of maxima, δ = M − m^R per record,
    S += e^{−δ} S^R,   U += e^{−δ_t} (U^R − (δ_t − δ_s) S_t^R)
with the empty record (−∞, −∞, 0, 0, 0) as identity (skipped explicitly).
"""
from __future__ import annotations

import numpy as np

from .kd_oracle import KINDS, lm_head_logits, _check_beta

EMPTY = None  # the identity record


def block_record(a: np.ndarray, b: np.ndarray):
    """Record (m_t, m_s, S_t, S_s, U) of one vocabulary block; a, b: [N, Vb] scaled logits."""
    if a.shape[1] == 0:
        return EMPTY
    m_t = a.max(axis=1)
    m_s = b.max(axis=1)
    xt = a - m_t[:, None]
    xs = b - m_s[:, None]
    et = np.exp(xt)
    return (m_t, m_s, et.sum(axis=1), np.exp(xs).sum(axis=1), (et * (xt - xs)).sum(axis=1))


def merge(A, B):
    """Pairwise merge operator; EMPTY is the identity."""
    if A is EMPTY:
        return B
    if B is EMPTY:
        return A
    M_t = np.maximum(A[0], B[0])
    M_s = np.maximum(A[1], B[1])
    S_t = np.zeros_like(M_t)
    S_s = np.zeros_like(M_t)
    U = np.zeros_like(M_t)
    for R in (A, B):
        dt = M_t - R[0]
        ds = M_s - R[1]
        ft = np.exp(-dt)
        S_t += ft * R[2]
        S_s += np.exp(-ds) * R[3]
        U += ft * (R[4] - (dt - ds) * R[2])
    return (M_t, M_s, S_t, S_s, U)


def vocab_bounds(V: int, n_parts: int, granule: int = 1):
    """Split [0, V) into n_parts contiguous ranges of whole granules, as evenly as possible."""
    n_gran = -(-V // granule)
    edges = [min(V, (n_gran * i // n_parts) * granule) for i in range(n_parts + 1)]
    return [(edges[i], edges[i + 1]) for i in range(n_parts)]


def kd_blockwise(h_t, W_t, h_s, W_s, mask=None, *, T=1.0, kind="fkl", beta=0.5,
                 loss_scale=1.0, want_dW=False, n_shards=1, n_split=1, granule=1,
                 merge_order="sequential"):
    """Simulated vocab-sharded hot path.

    Pass 1: per (shard, split) block record -> merge (sequential in block order, or a
    pairwise tree) -> per-row LSEs and FKL/RKL loss.  Pass 2: per block, the logit
    gradient from the merged LSEs (JSD/TVD: per-block partial K = Σ q·ℓ_v, summed across
    blocks, then G = c (G_a − K G_b)); per-shard partial dh summed over shards (the
    all-reduce); dW rows are shard-local.
    """
    if kind not in KINDS:
        raise ValueError(kind)
    if kind == "jsd":
        _check_beta(beta)
    N = h_t.shape[0]
    V, d_s = W_s.shape
    rows = np.arange(N) if mask is None else np.flatnonzero(np.asarray(mask) != 0)
    ht = np.asarray(h_t, np.float64)[rows]
    hs = np.asarray(h_s, np.float64)[rows]
    Wt = np.asarray(W_t, np.float64)
    Ws = np.asarray(W_s, np.float64)
    blocks = []
    for (s0, s1) in vocab_bounds(V, n_shards, granule):
        sub = vocab_bounds(s1 - s0, n_split, 1)
        blocks.append([(s0 + b0, s0 + b1) for (b0, b1) in sub])
    flat = [b for shard in blocks for b in shard]
    swap = kind == "rkl"

    # ---- pass 1
    recs = []
    for (v0, v1) in flat:
        a = lm_head_logits(ht, Wt[v0:v1]) / T
        b = lm_head_logits(hs, Ws[v0:v1]) / T
        recs.append(block_record(b, a) if swap else block_record(a, b))
    if merge_order == "sequential":
        R = EMPTY
        for r in recs:
            R = merge(R, r)
    elif merge_order == "tree":
        level = list(recs)
        while len(level) > 1:
            level = [merge(level[i], level[i + 1]) if i + 1 < len(level) else level[i]
                     for i in range(0, len(level), 2)]
        R = level[0]
    else:
        raise ValueError(merge_order)
    m_p, m_q, S_p, S_q, U = R  # primary / secondary roles
    lse_p = m_p + np.log(S_p)
    lse_q = m_q + np.log(S_q)
    if swap:
        lse_t, lse_s = lse_q, lse_p
    else:
        lse_t, lse_s = lse_p, lse_q
    ell = U / S_p - np.log(S_p) + np.log(S_q)  # FKL (or RKL with swapped roles)

    # ---- pass 2
    c = loss_scale / T
    Ks = np.zeros(rows.size)
    Js = np.zeros(rows.size)
    Ga_blocks, Gb_blocks = [], []
    for (v0, v1) in flat:
        lp = lm_head_logits(ht, Wt[v0:v1]) / T - lse_t[:, None]
        lq = lm_head_logits(hs, Ws[v0:v1]) / T - lse_s[:, None]
        p, q = np.exp(lp), np.exp(lq)
        if kind == "fkl":
            Ga_blocks.append(c * (q - p)); Gb_blocks.append(None)
        elif kind == "rkl":
            Ga_blocks.append(c * q * (lq - lp - ell[:, None])); Gb_blocks.append(None)
        elif kind == "jsd":
            lm = np.logaddexp(np.log(beta) + lp, np.log1p(-beta) + lq)
            lv = lq - lm
            Ks += (q * lv).sum(axis=1)
            Js += beta * (p * (lp - lm)).sum(axis=1)
            Ga_blocks.append(q * lv); Gb_blocks.append(q)
        else:  # tvd
            s = np.sign(q - p)
            Ks += (q * s).sum(axis=1)
            Js += 0.5 * np.abs(p - q).sum(axis=1)
            Ga_blocks.append(q * s); Gb_blocks.append(q)
    if kind == "jsd":
        ell = Js + (1.0 - beta) * Ks
        scale = c * (1.0 - beta)
        Ga_blocks = [scale * (ga - Ks[:, None] * gb) for ga, gb in zip(Ga_blocks, Gb_blocks)]
    elif kind == "tvd":
        ell = Js
        Ga_blocks = [0.5 * c * (ga - Ks[:, None] * gb) for ga, gb in zip(Ga_blocks, Gb_blocks)]

    loss = np.zeros(N)
    loss[rows] = ell
    dh_rows = np.zeros((rows.size, d_s))
    dW = np.zeros((V, d_s)) if want_dW else None
    i = 0
    for shard in blocks:
        dh_part = np.zeros((rows.size, d_s))   # this shard's partial dh (before all-reduce)
        for (v0, v1) in shard:
            G = Ga_blocks[i]
            i += 1
            dh_part += G @ Ws[v0:v1]
            if want_dW:
                dW[v0:v1] = G.T @ hs
        dh_rows += dh_part
    dh = np.zeros((N, d_s))
    dh[rows] = dh_rows
    return loss, dh, dW
