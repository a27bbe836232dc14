"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on identical bf16 inputs.

Tolerances (BASELINE.json north_star; R13/R14): per-token loss |Δ| <= 1e-3|ref| + 1e-5 element by
element; gradients |Δ| <= 2e-3|ref| + 1e-5 element by element (here, at these sizes, with no conditioning
floor at all; the full-size tests add the oracle's sensitivity to the measured tcgen05 logit error).
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
    import paper_2603_01875_b200 as kd
    kd.lib()  # fails loudly if the extension is missing


def _kd():
    import paper_2603_01875_b200 as kd
    return kd


# ------------------------------------------------------------------ building block: the tcgen05 GEMM
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_block_vs_matmul(a_mn, b_mn):
    """Operand majors used by the backward GEMMs (K-major and MN-major UMMA descriptors)."""
    kd = _kd()
    torch.manual_seed(0)
    M, N, K = 392, 512, 704   # ragged M tile, two N tiles, 11 K blocks
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    ref = A.double() @ B.double().T
    A_in = A.T.contiguous() if a_mn else A
    B_in = B.T.contiguous() if b_mn else B
    D = kd.gemm_bf16_f32(A_in, B_in, M=M, N=N, K=K, a_mn_major=a_mn, b_mn_major=b_mn)
    torch.cuda.synchronize()
    err = (D.double() - ref).abs().max().item()
    assert err < 1e-3 * ref.abs().max().item(), err


# ------------------------------------------------------------------ configs[0]: the tiny fp32 check
def test_tiny_config_parity():
    cfg = KI.CONFIGS["tiny"]
    inp = KI.make_config_inputs(cfg)
    kd = _kd()
    r = kd.fused_fwd_bwd(dev_bf16(inp.H_t), dev_bf16(inp.W_t), dev_bf16(inp.H_s), dev_bf16(inp.W_s),
                         T=cfg.temperature, kind=cfg.kind, want_dW=True)
    torch.cuda.synchronize()
    loss, dh, dW = oracle_run(inp, T=cfg.temperature, kind=cfg.kind, want_dW=True)
    assert_kd_close("loss", r.loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", r.dh_s.cpu().numpy(), dh)
    assert_grad_close("dW_s", r.dW_s.cpu().numpy(), dW)
    assert int(r.n_nonfinite.item()) == 0


# ------------------------------------------------------------------ all kinds, ragged shapes, masks
@pytest.mark.parametrize("kind", ["fkl", "rkl", "jsd", "tvd"])
@pytest.mark.parametrize("T", [1.0, 2.0])
@pytest.mark.parametrize("masked", [False, True])
def test_small_parity(kind, T, masked):
    """N = 300 (ragged token tile), V = 1000 (ragged vocab tile and chunk), d_t != d_s, chunked at 128."""
    N, d_t, d_s, V = 300, 256, 128, 1000
    rng = np.random.default_rng(7)
    mask = (rng.random(N) > 0.35).astype(np.uint8) if masked else None
    inp = KI.make_inputs(N, d_t, d_s, V, seed=3, mask=mask)
    kd = _kd()
    m_t = None if mask is None else torch.from_numpy(mask).cuda()
    r = kd.fused_fwd_bwd(dev_bf16(inp.H_t), dev_bf16(inp.W_t), dev_bf16(inp.H_s), dev_bf16(inp.W_s), m_t,
                         T=T, kind=kind, beta=0.5, loss_scale=1.0, want_dW=True, chunk_tokens=128)
    torch.cuda.synchronize()
    loss, dh, dW = oracle_run(inp, T=T, kind=kind, want_dW=True)
    assert_kd_close("loss", r.loss.cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s", r.dh_s.cpu().numpy(), dh)
    assert_grad_close("dW_s", r.dW_s.cpu().numpy(), dW)
    if mask is not None:
        assert np.all(r.loss.cpu().numpy()[mask == 0] == 0)
        assert np.all(r.dh_s.cpu().numpy()[mask == 0] == 0)
