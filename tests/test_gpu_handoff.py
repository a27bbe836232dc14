"""the hidden-state hand-off teacher process -> student process (kd_handoff_*, kdfused.h).

KDFlow's teacher ships only H_t; the student recomputes the teacher logits with the teacher's LM head.
Here a teacher PROCESS uploads H_t and exports it; the student process maps it (CUDA IPC) and (1) reads exactly the
teacher's bytes, (2) runs kd_fused_fwd_bwd on the mapped H_t in place — bit-identical to the same call on its own
copy — and (3) pulls it into its own buffer with one device-to-device copy.
"""
import ctypes
import multiprocessing as mp

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


SHAPE = dict(n_tokens=700, d_t=512, d_s=256, vocab=5000)


def _teacher(conn, seed):
    """Teacher side: upload H_t (the generator's bit pattern), export it, keep it alive until told to exit."""
    import paper_2603_01875_b200 as kd
    torch.cuda.set_device(0)
    inp = KI.make_inputs(SHAPE["n_tokens"], SHAPE["d_t"], SHAPE["d_s"], SHAPE["vocab"], seed=seed)
    ht = dev_bf16(inp.H_t)
    torch.cuda.synchronize()
    conn.send((kd.handoff_export(ht), tuple(ht.shape)))
    conn.recv()


def test_hidden_state_handoff_between_processes():
    import paper_2603_01875_b200 as kd
    ctx = mp.get_context("spawn")
    parent, child = ctx.Pipe()
    proc = ctx.Process(target=_teacher, args=(child, 7))
    proc.start()
    try:
        handle, shape = parent.recv()
        assert len(handle) == 96
        inp = KI.make_inputs(SHAPE["n_tokens"], SHAPE["d_t"], SHAPE["d_s"], SHAPE["vocab"], seed=7)
        ht_local = dev_bf16(inp.H_t)
        with pytest.raises(ValueError):
            kd.HandoffTensor(handle, (shape[0] + 1, shape[1]), torch.bfloat16)
        h = kd.HandoffTensor(handle, shape, torch.bfloat16)
        ht_mapped = h.tensor
        assert ht_mapped.dtype == torch.bfloat16 and tuple(ht_mapped.shape) == shape
        assert torch.equal(ht_mapped, ht_local)  # (1) the teacher's bytes
        Wt, hs, Ws = dev_bf16(inp.W_t), dev_bf16(inp.H_s), dev_bf16(inp.W_s)
        mask = torch.from_numpy((np.arange(shape[0]) % 5 != 0).astype(np.uint8)).cuda()
        kw = dict(T=1.0, kind="fkl", want_dW=True, chunk_tokens=256)
        a = kd.fused_fwd_bwd(ht_mapped, Wt, hs, Ws, mask, **kw)  # (2) in place, zero copy
        b = kd.fused_fwd_bwd(ht_local, Wt, hs, Ws, mask, **kw)
        pulled = torch.empty_like(ht_local)
        pulled.copy_(ht_mapped)  # (3) one D2D pull
        torch.cuda.synchronize()
        assert torch.equal(a.loss, b.loss) and torch.equal(a.dh_s, b.dh_s) and torch.equal(a.dW_s, b.dW_s)
        assert torch.equal(pulled, ht_local)
        h_ptr = h.ptr
        h.close()
        with pytest.raises(kd.KDError, match="not from kd_handoff_open"):
            kd.kdfused._check(kd.lib().kd_handoff_close(ctypes.c_void_p(h_ptr)))  # already closed
    finally:
        parent.send("done")
        proc.join(timeout=60)
    assert proc.exitcode == 0
