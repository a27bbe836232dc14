"""Shared helpers for the parity tests: upload generator bit patterns, run the oracle, compare."""
from __future__ import annotations

import os

import numpy as np
import torch

import kd_inputs as KI

# BASELINE.json north_star tolerances (+ the absolute floor of DESIGN.md reading R13)
LOSS_RTOL, LOSS_ATOL = 1e-3, 1e-5
GRAD_RTOL, GRAD_ATOL = 2e-3, 1e-5


def dev_bf16(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device).view(torch.bfloat16)


def f64(bits: np.ndarray) -> np.ndarray:
    return KI.bf16_to_f64(bits)


def oracle_run(inp: KI.KDInputs, *, T, kind, beta=0.5, loss_scale=1.0, want_dW=False, rows=None):
    from oracle.kd_oracle import kd_fused_fwd_bwd
    ht, hs = f64(inp.H_t), f64(inp.H_s)
    mask = inp.mask
    if rows is not None:  # per-token outputs depend only on that row (+ the heads)
        ht, hs = ht[rows], hs[rows]
        mask = None if mask is None else mask[rows]
    return kd_fused_fwd_bwd(ht, f64(inp.W_t), hs, f64(inp.W_s), mask, T=T, kind=kind, beta=beta,
                            loss_scale=loss_scale, want_dW=want_dW)


def _parity_log(name, got, ref, strict_tol, floor_used, n_strict):
    """KD_PARITY_LOG=path: append one JSON line per comparison (summarised in profiles/r01_parity.md)."""
    path = os.environ.get("KD_PARITY_LOG")
    if not path or got.size == 0:
        return
    import json
    d = np.abs(got - ref)
    rec = {"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "name": name, "n": int(got.size),
           "max_abs_err": float(d.max()), "max_err_over_strict_tol": float((d / strict_tol).max()),
           "strict_violations": int(n_strict), "floor_used": bool(floor_used)}
    with open(path, "a") as fh:
        fh.write(json.dumps(rec) + "\n")


def assert_kd_close(name, got, ref, rtol, atol, max_report=5):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    _parity_log(name, got, ref, atol + rtol * np.abs(ref), False,
                int((np.abs(got - ref) > atol + rtol * np.abs(ref)).sum()))
    bad = ~(np.abs(got - ref) <= atol + rtol * np.abs(ref))
    if bad.any():
        idx = np.argwhere(bad)[:max_report]
        details = [(tuple(i), float(got[tuple(i)]), float(ref[tuple(i)])) for i in idx]
        raise AssertionError(f"{name}: {bad.sum()} / {bad.size} elements outside |d| <= {atol} + {rtol}|ref|; "
                             f"max|d| = {np.abs(got - ref).max():.3e}; first: {details}")


def assert_grad_close(name, got, ref, rtol=GRAD_RTOL, atol=GRAD_ATOL, allow=0, max_ratio=1.0):
    """Gradient parity at the BASELINE.json north_star tolerance, element by element: |Δ| <= rtol·|ref| + atol.

    Fails closed.  ``allow`` / ``max_ratio`` name, per test, the ONLY exception DESIGN.md reading R14 admits: at most
    ``allow`` elements may exceed the bound, each by at most ``max_ratio`` × (rtol·|ref| + atol).  They are the
    ill-conditioned elements (results ~100x smaller than their terms, e.g. the Zipf-bias column of dh_s) where the
    prescribed arithmetic — bf16 tensor-core GEMMs with fp32 accumulation over K = d_t = 4096 — is itself outside the
    bound (scripts/probe_parity_src.py: tcgen05 logit error up to 1.7e-4 at K = 4096, proportional to the steps per
    accumulator).  Every such element is printed and logged (KD_PARITY_LOG); the default (allow = 0) is strict.
    Returns the number of elements beyond the plain bound."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    d = np.abs(got - ref)
    tol = atol + rtol * np.abs(ref)
    ratio = d / tol
    bad = ~(ratio <= 1.0)  # NaN counts as a violation
    _parity_log(name, got, ref, tol, False, int(bad.sum()))
    if bad.any():
        idx = np.argwhere(bad)
        order = np.argsort(-np.nan_to_num(ratio[bad], nan=np.inf))
        listed = [(tuple(int(x) for x in idx[i]), float(got[tuple(idx[i])]), float(ref[tuple(idx[i])]),
                   float(ratio[tuple(idx[i])])) for i in order[:20]]
        print(f"[parity] {name}: {int(bad.sum())} element(s) beyond |d| <= {atol} + {rtol}|ref| "
              f"(allowed {allow} up to {max_ratio}x): {listed}")
        worst = float(np.nan_to_num(ratio, nan=np.inf).max())
        assert int(bad.sum()) <= allow and worst <= max_ratio, (
            f"{name}: {int(bad.sum())} / {bad.size} elements outside |d| <= {atol} + {rtol}|ref| "
            f"(worst {worst:.3f}x; allowed {allow} element(s) up to {max_ratio}x); worst first: {listed[:5]}")
    return int(bad.sum())
