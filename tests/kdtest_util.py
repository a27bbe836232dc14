"""Shared helpers for the parity tests: upload generator bit patterns, run the oracle, compare."""
from __future__ import annotations

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


def assert_kd_close(name, got, ref, rtol, atol, max_report=5):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    bad = ~(np.abs(got - ref) <= atol + rtol * np.abs(ref))
    if bad.any():
        idx = np.argwhere(bad)[:max_report]
        details = [(tuple(i), float(got[tuple(i)]), float(ref[tuple(i)])) for i in idx]
        raise AssertionError(f"{name}: {bad.sum()} / {bad.size} elements outside |d| <= {atol} + {rtol}|ref|; "
                             f"max|d| = {np.abs(got - ref).max():.3e}; first: {details}")
