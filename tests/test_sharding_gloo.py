"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic.

The CUDA kernels cannot run here, so the two kernel-side callables of ``vocab_sharded_fwd_bwd`` are
replaced by CPU stand-ins built from the oracle's blockwise formulation (test code only).  What is under
test is the exchange the product performs: record all-gather in rank order, merge, partial-dh all-reduce,
shard bounds, and the token-sharded dW reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_01875_b200.sharding import (token_shard_bounds, token_sharded_dW_reduce, vocab_shard_bounds,
                                            vocab_sharded_fwd_bwd)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---------------------------------------------------------------- CPU stand-ins for the two kernel calls
def _stats_standin(h_t, Wt, h_s, Ws, mask, *, vocab, v_begin, T, kind, chunk_tokens):
    from oracle.kd_blockwise import block_record
    ht, hs = h_t.double().numpy(), h_s.double().numpy()
    a = ht @ Wt.double().numpy().T / T
    b = hs @ Ws.double().numpy().T / T
    rec = block_record(b, a) if kind == "rkl" else block_record(a, b)
    out = torch.tensor(np.stack(rec))
    if kind == "fkl":  # FKL records carry no cross term (the kernels' decoupled pass 1)
        out[4] = 0.0
    if mask is not None:
        out[:, mask == 0] = 0.0
    return out


class _R:
    def __init__(self, loss, dh, dW):
        self.loss, self.dh_s, self.dW_s = loss, dh, dW


def _backward_standin(h_t, Wt, h_s, Ws, recs, mask, *, vocab, v_begin, T, kind, loss_scale, want_dW,
                      accumulate_dW, dW_s, chunk_tokens):
    from oracle.kd_blockwise import merge
    R = None
    for r in recs:  # rank order
        rr = tuple(x.numpy() for x in r)
        if np.all(rr[2] == 0):
            continue
        R = rr if R is None else merge(R, rr)
    m = np.ones(recs.shape[-1]) if mask is None else mask.numpy().astype(np.float64)
    live = m > 0
    m_p, m_q, S_p, S_q, U = (np.where(live, x, 1.0) for x in R)  # masked rows: inert placeholder record
    lse_p, lse_q = m_p + np.log(S_p), m_q + np.log(S_q)
    lse_t, lse_s = (lse_q, lse_p) if kind == "rkl" else (lse_p, lse_q)
    ell = U / S_p - np.log(S_p) + np.log(S_q)
    lp = h_t.double().numpy() @ Wt.double().numpy().T / T - lse_t[:, None]
    lq = h_s.double().numpy() @ Ws.double().numpy().T / T - lse_s[:, None]
    p, q = np.exp(lp), np.exp(lq)
    G = loss_scale / T * ((q - p) if kind == "fkl" else q * (lq - lp - ell[:, None]))
    G = np.where(live[:, None], G, 0.0)
    if kind == "fkl":  # this shard's partial loss, global LSEs; the caller sums over shards
        ell = (p * (lp - lq)).sum(1)
    ell = np.where(live, ell, 0.0)
    dh = torch.tensor(G @ Ws.double().numpy())
    dW = torch.tensor(G.T @ h_s.double().numpy()) if want_dW else None
    if want_dW and accumulate_dW and dW_s is not None:  # the kernels accumulate into the caller's dW_s
        dW = dW_s + dW
    return _R(torch.tensor(ell), dh, dW)


class _FixState:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _probs(h_t, Wt, h_s, Ws, recs, mask, T, kind):
    from oracle.kd_blockwise import merge
    R = None
    for r in recs:  # rank order
        rr = tuple(x.numpy() for x in r)
        if np.all(rr[2] == 0):
            continue
        R = rr if R is None else merge(R, rr)
    m = np.ones(recs.shape[-1]) if mask is None else mask.numpy().astype(np.float64)
    live = m > 0
    m_p, m_q, S_p, S_q, _ = (np.where(live, x, 1.0) for x in R)
    lse_t, lse_s = m_p + np.log(S_p), m_q + np.log(S_q)
    lp = h_t.double().numpy() @ Wt.double().numpy().T / T - lse_t[:, None]
    lq = h_s.double().numpy() @ Ws.double().numpy().T / T - lse_s[:, None]
    return live, lp, lq


def _partials_standin(h_t, Wt, h_s, Ws, recs, mask, *, vocab, v_begin, T, kind, beta, loss_scale, want_dW,
                      accumulate_dW, chunk_tokens):
    live, lp, lq = _probs(h_t, Wt, h_s, Ws, recs, mask, T, kind)
    p, q = np.exp(lp), np.exp(lq)
    if kind == "jsd":
        lm = np.log(beta * p + (1 - beta) * q)
        K = (q * (lq - lm)).sum(1) / np.log(2)   # bits, like the kernels
        J = (p * (lp - lm)).sum(1) / np.log(2)
    else:
        s = np.sign(q - p)
        K = (q * s).sum(1)
        J = np.abs(q - p).sum(1)
    kj = torch.tensor(np.stack([np.where(live, K, 0.0), np.where(live, J, 0.0)]))
    st = _FixState(live=live, p=p, q=q, lp=lp, lq=lq, beta=beta, T=T, kind=kind, loss_scale=loss_scale,
                   want_dW=want_dW, accumulate_dW=accumulate_dW)
    return kj, st


def _finish_standin(st, h_t, Wt, h_s, Ws, kj_all, mask, *, dW_s=None):
    K = kj_all[:, 0].numpy().sum(0)   # rank order
    J = kj_all[:, 1].numpy().sum(0)
    c = st.loss_scale / st.T
    if st.kind == "jsd":
        lm = np.log(st.beta * st.p + (1 - st.beta) * st.q)
        G = c * (1 - st.beta) * st.q * ((st.lq - lm) - K[:, None] * np.log(2))
        ell = np.log(2) * (st.beta * J + (1 - st.beta) * K)
    else:
        G = 0.5 * c * st.q * (np.sign(st.q - st.p) - K[:, None])
        ell = 0.5 * J
    G = np.where(st.live[:, None], G, 0.0)
    ell = np.where(st.live, ell, 0.0)
    dh = torch.tensor(G @ Ws.double().numpy())
    dW = None
    if st.want_dW:
        dW = torch.tensor(G.T @ h_s.double().numpy())
        if st.accumulate_dW and dW_s is not None:
            dW = dW_s + dW
    return _R(torch.tensor(ell), dh, dW)


def _worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import kd_inputs as KI
        N, d_t, d_s, V = 40, 32, 24, 300
        mask = (np.arange(N) % 7 != 3).astype(np.uint8)
        inp = KI.make_inputs(N, d_t, d_s, V, seed=4, mask=mask)
        ht = torch.tensor(KI.bf16_to_f64(inp.H_t))
        hs = torch.tensor(KI.bf16_to_f64(inp.H_s))
        Wt = torch.tensor(KI.bf16_to_f64(inp.W_t))
        Ws = torch.tensor(KI.bf16_to_f64(inp.W_s))
        a, b = vocab_shard_bounds(V, world, granule=16)[rank]
        # exchange_chunk=16 drives three pipelined token chunks: records all-gather (and for JSD/TVD the (K, J)
        # all-gather) of chunk c+1 in flight while chunk c's partial dh all-reduce is still pending
        r = vocab_sharded_fwd_bwd(ht, Wt[a:b], hs, Ws[a:b], torch.tensor(mask), vocab=V, v_begin=a, T=1.3,
                                  kind=kind, beta=0.3, want_dW=True, exchange_chunk=16, stats_fn=_stats_standin,
                                  backward_fn=_backward_standin, partials_fn=_partials_standin,
                                  finish_fn=_finish_standin)
        # token-sharded dW: each rank's partial sum over its tokens, reduced
        t0, t1 = token_shard_bounds(N, world)[rank]
        from oracle.kd_oracle import kd_fused_fwd_bwd
        sl = slice(t0, t1)
        _, _, dW_part = kd_fused_fwd_bwd(ht.numpy()[sl], Wt.numpy(), hs.numpy()[sl], Ws.numpy(), mask[sl],
                                         T=1.3, kind=kind, beta=0.3, want_dW=True)
        dW_tok = token_sharded_dW_reduce(torch.tensor(dW_part))
        # dh_reduce="scatter": the reduce-scatter of the same exchange, this rank's token slice only
        rs = vocab_sharded_fwd_bwd(ht, Wt[a:b], hs, Ws[a:b], torch.tensor(mask), vocab=V, v_begin=a, T=1.3,
                                   kind=kind, beta=0.3, exchange_chunk=16, stats_fn=_stats_standin,
                                   backward_fn=_backward_standin, partials_fn=_partials_standin,
                                   finish_fn=_finish_standin, dh_reduce="scatter")
        q.put((rank, r.loss.numpy(), r.dh_s.numpy(), (a, b, r.dW_s.numpy()), dW_tok.numpy(),
               (rs.loss.numpy(), rs.dh_s.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["fkl", "rkl", "jsd", "tvd"])
def test_vocab_and_token_sharding_world2(kind):
    import kd_inputs as KI
    from oracle.kd_oracle import kd_fused_fwd_bwd
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, d_t, d_s, V = 40, 32, 24, 300
    mask = (np.arange(N) % 7 != 3).astype(np.uint8)
    inp = KI.make_inputs(N, d_t, d_s, V, seed=4, mask=mask)
    f = KI.bf16_to_f64
    loss, dh, dW = kd_fused_fwd_bwd(f(inp.H_t), f(inp.W_t), f(inp.H_s), f(inp.W_s), mask, T=1.3, kind=kind,
                                    beta=0.3, want_dW=True)
    dW_cat = np.zeros_like(dW)
    for rank, l, d, (a, b, dws), dW_tok, (ls, ds) in res:
        own = slice(rank * N // world, (rank + 1) * N // world)
        np.testing.assert_allclose(ls, loss[own], rtol=1e-12, atol=1e-13)  # reduce-scatter: own tokens only
        np.testing.assert_allclose(ds, dh[own], rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(l, loss, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(d, dh, rtol=1e-11, atol=1e-13)   # all-reduced dh on every rank
        np.testing.assert_allclose(dW_tok, dW, rtol=1e-11, atol=1e-13)
        dW_cat[a:b] = dws
    np.testing.assert_allclose(dW_cat, dW, rtol=1e-11, atol=1e-13)  # local dW rows tile the full dW


def test_bounds():
    b = vocab_shard_bounds(151936, 8)
    assert b[0][0] == 0 and b[-1][1] == 151936 and all(x[0] % 128 == 0 for x in b)
    assert sorted({y - x for x, y in b}) == [18944, 19072]   # 148 / 149 granules
    assert vocab_shard_bounds(100, 3, granule=128) == [(0, 0), (0, 0), (0, 100)]
    assert token_shard_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]


@pytest.mark.parametrize("kind", ["fkl", "jsd"])
def test_one_rank_without_process_group(kind):
    """A one-rank job (bench.py --shard vocab at N=1) runs the same protocol with identity exchanges."""
    import kd_inputs as KI
    from oracle.kd_oracle import kd_fused_fwd_bwd
    assert not dist.is_initialized()
    N, d_t, d_s, V = 24, 32, 16, 200
    inp = KI.make_inputs(N, d_t, d_s, V, seed=6)
    f = KI.bf16_to_f64
    ht, hs, Wt, Ws = (torch.tensor(f(x)) for x in (inp.H_t, inp.H_s, inp.W_t, inp.W_s))
    r = vocab_sharded_fwd_bwd(ht, Wt, hs, Ws, None, vocab=V, v_begin=0, T=1.1, kind=kind, beta=0.5, want_dW=True,
                              exchange_chunk=16, stats_fn=_stats_standin, backward_fn=_backward_standin,
                              partials_fn=_partials_standin, finish_fn=_finish_standin)
    loss, dh, dW = kd_fused_fwd_bwd(f(inp.H_t), f(inp.W_t), f(inp.H_s), f(inp.W_s), None, T=1.1, kind=kind,
                                    beta=0.5, want_dW=True)
    np.testing.assert_allclose(r.loss.numpy(), loss, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(r.dh_s.numpy(), dh, rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(r.dW_s.numpy(), dW, rtol=1e-11, atol=1e-13)
