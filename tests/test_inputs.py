"""The seeded input generator (shared by oracle and CUDA path; holds no method arithmetic)."""
import numpy as np
import torch

import kd_inputs as KI


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10,
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -0.0, 0.0, 65504.0], np.float32)])
    ours = KI.bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(KI.bf16_bits(KI.bf16_to_f32(ours)), ours)  # projection idempotent


def test_generator_deterministic_and_shapes():
    a = KI.make_inputs(16, 128, 64, 512, seed=3)
    b = KI.make_inputs(16, 128, 64, 512, seed=3)
    for x, y in zip((a.H_t, a.W_t, a.H_s, a.W_s), (b.H_t, b.W_t, b.H_s, b.W_s)):
        assert np.array_equal(x, y)
    assert a.H_t.shape == (16, 128) and a.W_t.shape == (512, 128)
    assert a.H_s.shape == (16, 64) and a.W_s.shape == (512, 64)
    assert np.all(KI.bf16_to_f32(a.H_t[:, 0]) == 1.0)


def test_masks():
    m = KI.make_mask(KI.CONFIGS["c3_rkl"])
    assert m.shape == (32768,) and m.dtype == np.uint8
    frac = m.mean()
    assert 0.45 < frac < 0.85
    for s in range(8):
        seg = m[s * 4096:(s + 1) * 4096]
        assert seg[:64].sum() == 0
    r = KI.make_mask(KI.CONFIGS["c5"])
    assert r.shape == (32768,) and 0.6 < r.mean() < 0.99
    assert KI.make_mask(KI.CONFIGS["c2"]) is None


def test_calibration_llm_like_rows():
    """Peaked teacher rows at T=1 (SURVEY §8d calibration): large max logit, p_max mostly high."""
    inp = KI.make_inputs(64, 1024, 512, 8192, seed=0)
    ht = KI.bf16_to_f64(inp.H_t)
    Wt = KI.bf16_to_f64(inp.W_t)
    z = ht @ Wt.T
    zmax = z.max(axis=1)
    p = np.exp(z - zmax[:, None])
    p /= p.sum(axis=1, keepdims=True)
    assert np.median(zmax) > 12
    assert np.median(p.max(axis=1)) > 0.3
