"""The library's calls are capturable into a CUDA graph (no host syncs, no allocation inside a call, every launch on
the caller's stream): one captured step replayed on new inputs equals the eager call bit for bit."""
import numpy as np
import pytest
import torch

import kd_inputs as KI
from tests.kdtest_util import dev_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("stage", [False, True])
@pytest.mark.parametrize("kind", ["fkl", "jsd"])
def test_graph_replay_equals_eager(kind, stage):
    import paper_2603_01875_b200 as kd
    N, d_t, d_s, V = 640, 256, 128, 3000
    a = KI.make_inputs(N, d_t, d_s, V, seed=61)
    b = KI.make_inputs(N, d_t, d_s, V, seed=62)
    Wt, Ws = dev_bf16(a.W_t), dev_bf16(a.W_s)
    ht, hs = dev_bf16(a.H_t), dev_bf16(a.H_s)
    mask = torch.from_numpy((np.arange(N) % 9 != 4).astype(np.uint8)).cuda()
    kw = dict(T=1.2, kind=kind, want_dW=True, chunk_tokens=256, stage_logits=stage)
    out = kd.KDResult(torch.empty(N, device="cuda"), torch.empty(N, d_s, device="cuda"), None,
                      torch.zeros(1, dtype=torch.int64, device="cuda"))
    dW = torch.empty(V, d_s, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        kd.fused_fwd_bwd(ht, Wt, hs, Ws, mask, dW_s=dW, out=out, **kw)  # warm-up: workspace, smem opt-ins
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        kd.fused_fwd_bwd(ht, Wt, hs, Ws, mask, dW_s=dW, out=out, **kw)
    # new batch into the captured input buffers, replay
    ht.copy_(dev_bf16(b.H_t))
    hs.copy_(dev_bf16(b.H_s))
    g.replay()
    torch.cuda.synchronize()
    ref = kd.fused_fwd_bwd(dev_bf16(b.H_t), Wt, dev_bf16(b.H_s), Ws, mask, **kw)
    torch.cuda.synchronize()
    assert torch.equal(out.loss, ref.loss)
    assert torch.equal(out.dh_s, ref.dh_s)
    assert torch.equal(dW, ref.dW_s)
