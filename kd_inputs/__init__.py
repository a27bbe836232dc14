"""Seeded synthetic inputs for the KD hot path — shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no logits, softmax, divergence or
gradient).  It only draws random numbers, rounds them to bf16 (round-to-nearest-even)
and returns the bf16 bit patterns as ``uint16`` arrays, so the fp64 oracle and the
bf16 CUDA kernels consume identical inputs.

Recipe (calibrated to LLM-like rows):

* LM heads in ``nn.Linear`` layout ``[V, d]``.  ``W_t ~ N(0, σ_t²)``, ``σ = 1.28/√d``
  (0.02 at d=4096, logit std ≈ 1.3).  ``W_s = W_t[:, :d_s]·√(d_t/d_s) + 0.5·σ_s·noise``.
* Zipf bias column: column 0 of both heads is ``−ln(rank_v)`` centred, ``rank`` a random
  permutation of 1..V; every hidden row has ``h[0] = 1`` so the bias lives inside the GEMM.
* Hidden rows: ``h[1:] = RMS-normalise(α·e_y + √(1−α²)·n)`` with ``e_y`` the direction of
  ``W[y, 1:]`` for a target ``y`` drawn from the Zipf prior (P(y) ∝ 1/rank_y) and ``n`` a
  random unit direction; ``α = min(0.9, 0.12·√(4096/d))`` (target logit spike ≈ 10).
  The student's target equals the teacher's with probability 0.9.
* Masks: config 3 — per 4096-token sequence a prompt prefix L_p ~ U[64,512] and padding
  beyond L ~ U[2048,4096] are masked; config 5 — ragged sequences L ~ U[256,8192] with a
  masked prompt L_p ~ U[32, min(512, L/2)], packed back to back.
* Seeds: heads 1000, hidden 1001, masks/lengths 1002 (parity runs also use other seeds).

Shapes are BASELINE.json's configs (Qwen3 vocabulary V = 151936, ``P:37``, ``P:133``).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

V_QWEN3 = 151936  # P:37 footnote


@dataclass(frozen=True)
class KDConfig:
    """One BASELINE.json workload (configs[0..4])."""
    name: str
    n_seq: int
    seq_len: int
    d_t: int
    d_s: int
    vocab: int
    kind: str = "fkl"
    temperature: float = 1.0
    jsd_beta: float = 0.5
    mask: str = "none"          # "none" | "prompt_pad" (config 3) | "ragged" (config 5)
    want_dW: bool = False
    notes: str = ""

    @property
    def n_tokens(self) -> int:
        return self.n_seq * self.seq_len


CONFIGS = {
    # configs[0]: tiny fp32 check (CPU oracle in seconds)
    "tiny": KDConfig("tiny", 1, 64, 256, 256, 1024, "fkl", 1.0,
                     notes="BASELINE.json configs[0]"),
    # configs[1]: Qwen3-8B (d=4096) -> Qwen3-1.7B (d=2048), 8 x 4096 tokens, FKL, 1 B200
    "c2": KDConfig("c2", 8, 4096, 4096, 2048, V_QWEN3, "fkl", 1.0,
                   notes="BASELINE.json configs[1] (the metric's workload)"),
    # configs[2]: same shapes, RKL / JSD(0.5) at T=2 with prompt/padding mask
    "c3_rkl": KDConfig("c3_rkl", 8, 4096, 4096, 2048, V_QWEN3, "rkl", 2.0, mask="prompt_pad",
                       notes="BASELINE.json configs[2], RKL"),
    "c3_jsd": KDConfig("c3_jsd", 8, 4096, 4096, 2048, V_QWEN3, "jsd", 2.0, 0.5, mask="prompt_pad",
                       notes="BASELINE.json configs[2], JSD(beta=0.5)"),
    # configs[3]: Qwen3-30B-A3B (d=2048) -> Qwen3-0.6B (d=1024), 128 x 4096 tokens (8-GPU scale)
    "c4": KDConfig("c4", 128, 4096, 2048, 1024, V_QWEN3, "fkl", 1.0,
                   notes="BASELINE.json configs[3]; 8-GPU scale, per-GPU slice is 16 seqs"),
    # configs[4]: on-policy ragged 256..8192, RKL, dW_s accumulation
    "c5": KDConfig("c5", 8, 4096, 4096, 2048, V_QWEN3, "rkl", 1.0, mask="ragged", want_dW=True,
                   notes="BASELINE.json configs[4]; 32k-token packed step"),
}


# ----------------------------------------------------------------------------- bf16 helpers
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round-to-nearest-even (finite inputs)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit pattern (uint16) -> exact fp32 values."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_to_f64(b: np.ndarray) -> np.ndarray:
    return bf16_to_f32(b).astype(np.float64)


# ----------------------------------------------------------------------------- generators
def _sigma(d: int) -> float:
    return 1.28 / math.sqrt(d)


def _alpha(d: int) -> float:
    return min(0.9, 0.12 * math.sqrt(4096.0 / d))


def zipf_ranks(vocab: int, seed: int = 1000) -> np.ndarray:
    """rank[v] in 1..V, a random permutation (seed shared with the heads)."""
    rng = np.random.Generator(np.random.PCG64([seed, 7]))
    return rng.permutation(vocab).astype(np.int64) + 1


def _normal_rows(seed: int, stream: int, rows: int, cols: int, block: int = 2048) -> np.ndarray:
    """Standard-normal fp32 [rows, cols]; row blocks use independent PCG64 streams
    (SeedSequence([seed, stream, block_index])) and are filled by a thread pool, so the
    result depends only on (seed, stream, shape), never on the thread count."""
    out = np.empty((rows, cols), dtype=np.float32)
    starts = list(range(0, rows, block))

    def fill(i):
        r0 = starts[i]
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, i])))
        g.standard_normal(out=out[r0:r0 + block], dtype=np.float32)

    workers = max(1, min(len(starts), len(os.sched_getaffinity(0))))
    if workers == 1:
        for i in range(len(starts)):
            fill(i)
    else:
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(fill, range(len(starts))))
    return out


def _bf16_bits_par(x: np.ndarray, block: int = 4096) -> np.ndarray:
    out = np.empty(x.shape, dtype=np.uint16)
    starts = list(range(0, x.shape[0], block))

    def conv(r0):
        out[r0:r0 + block] = bf16_bits(x[r0:r0 + block])

    with ThreadPoolExecutor(max(1, len(os.sched_getaffinity(0)))) as ex:
        list(ex.map(conv, starts))
    return out


def make_heads(vocab: int, d_t: int, d_s: int, seed: int = 1000):
    """Return (W_t, W_s) as bf16 bit patterns, shapes [V, d_t] and [V, d_s]."""
    ranks = zipf_ranks(vocab, seed)
    bias = -np.log(ranks.astype(np.float64))
    bias = (bias - bias.mean()).astype(np.float32)
    st, ss = _sigma(d_t), _sigma(d_s)
    W_t = _normal_rows(seed, 1, vocab, d_t)
    W_t *= np.float32(st)
    W_t[:, 0] = bias
    W_s = _normal_rows(seed, 2, vocab, d_s)
    W_s *= np.float32(0.5 * ss)
    k = min(d_t, d_s)
    W_s[:, :k] += W_t[:, :k] * np.float32(math.sqrt(d_t / d_s))
    W_s[:, 0] = bias
    return _bf16_bits_par(W_t), _bf16_bits_par(W_s)


def _hidden_rows(seed: int, stream: int, W_bits: np.ndarray, targets: np.ndarray) -> np.ndarray:
    n, d = targets.shape[0], W_bits.shape[1]
    alpha = _alpha(d)
    dirs = bf16_to_f32(W_bits[targets, 1:])
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True) + np.float32(1e-30)
    noise = _normal_rows(seed, stream, n, d - 1)
    noise /= np.linalg.norm(noise, axis=1, keepdims=True) + np.float32(1e-30)
    h = np.float32(alpha) * dirs + np.float32(math.sqrt(1 - alpha * alpha)) * noise
    h *= (np.float32(math.sqrt(d - 1)) / (np.linalg.norm(h, axis=1, keepdims=True) + np.float32(1e-30)))
    out = np.empty((n, d), dtype=np.float32)
    out[:, 0] = 1.0
    out[:, 1:] = h
    return bf16_bits(out)


def make_hidden(n_tokens: int, W_t_bits: np.ndarray, W_s_bits: np.ndarray, seed: int = 1001,
                head_seed: int = 1000, p_same: float = 0.9):
    """Return (H_t, H_s) as bf16 bit patterns, shapes [N, d_t] and [N, d_s]."""
    vocab = W_t_bits.shape[0]
    rng = np.random.Generator(np.random.PCG64(seed))
    ranks = zipf_ranks(vocab, head_seed)
    prior = 1.0 / ranks.astype(np.float64)
    prior /= prior.sum()
    cdf = np.cumsum(prior)
    y_t = np.minimum(np.searchsorted(cdf, rng.random(n_tokens)), vocab - 1)
    other = np.minimum(np.searchsorted(cdf, rng.random(n_tokens)), vocab - 1)
    y_s = np.where(rng.random(n_tokens) < p_same, y_t, other)
    H_t = _hidden_rows(seed, 1, W_t_bits, y_t)
    H_s = _hidden_rows(seed, 2, W_s_bits, y_s)
    return H_t, H_s


def make_mask(cfg: KDConfig, seed: int = 1002) -> np.ndarray | None:
    """uint8 [N] loss mask (1 = loss-bearing) or None for an all-ones mask."""
    if cfg.mask == "none":
        return None
    rng = np.random.Generator(np.random.PCG64(seed))
    n = cfg.n_tokens
    m = np.zeros(n, dtype=np.uint8)
    if cfg.mask == "prompt_pad":
        for s in range(cfg.n_seq):
            lp = int(rng.integers(64, 513))
            ln = int(rng.integers(2048, 4097))
            lo = s * cfg.seq_len
            m[lo + lp: lo + min(ln, cfg.seq_len)] = 1
        return m
    if cfg.mask == "ragged":
        pos = 0
        while pos < n:
            ln = int(rng.integers(256, 8193))
            lp = int(rng.integers(32, min(512, ln // 2) + 1))
            end = min(pos + ln, n)
            m[min(pos + lp, end):end] = 1
            pos = end
        return m
    raise ValueError(f"unknown mask recipe {cfg.mask!r}")


@dataclass
class KDInputs:
    """bf16 bit patterns + mask for one problem instance."""
    H_t: np.ndarray
    W_t: np.ndarray
    H_s: np.ndarray
    W_s: np.ndarray
    mask: np.ndarray | None
    meta: dict = field(default_factory=dict)


def make_inputs(n_tokens: int, d_t: int, d_s: int, vocab: int, *, seed: int = 0,
                mask: np.ndarray | None = None, heads=None) -> KDInputs:
    """Instance of arbitrary shape; ``seed`` offsets the canonical seeds 1000/1001."""
    W_t, W_s = heads if heads is not None else make_heads(vocab, d_t, d_s, seed=1000 + seed)
    H_t, H_s = make_hidden(n_tokens, W_t, W_s, seed=1001 + seed, head_seed=1000 + seed)
    return KDInputs(H_t, W_t, H_s, W_s, mask,
                    dict(n_tokens=n_tokens, d_t=d_t, d_s=d_s, vocab=vocab, seed=seed))


def make_config_inputs(cfg: KDConfig, n_tokens: int | None = None, seed: int = 0) -> KDInputs:
    """Inputs for a named config (optionally truncated to the first ``n_tokens`` rows)."""
    n = cfg.n_tokens if n_tokens is None else n_tokens
    mask = make_mask(cfg, seed=1002 + seed)
    if mask is not None:
        mask = mask[:n]
    return make_inputs(n, cfg.d_t, cfg.d_s, cfg.vocab, seed=seed, mask=mask)


def self_distillation_twin(inp: KDInputs) -> KDInputs:
    """Student := teacher (A18 self-distillation).  Requires d_t == d_s."""
    assert inp.H_t.shape[1] == inp.H_s.shape[1]
    return KDInputs(inp.H_t, inp.W_t, inp.H_t.copy(), inp.W_t.copy(), inp.mask, dict(inp.meta))


def comm_volume_bytes(n_seq: int, seq_len: int, vocab: int = V_QWEN3, bytes_per: int = 2) -> int:
    """Full-logit transfer volume of P:37's footnote: B·T·V·2 bytes (an integer, not arithmetic of
    the method)."""
    return n_seq * seq_len * vocab * bytes_per
