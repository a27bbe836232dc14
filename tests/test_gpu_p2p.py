"""Peer-memory exchange of the vocab-sharded step (FKL / RKL / JSD / TVD) (kdfused.h kd_p2p) on one GPU.

P ranks run in one process against P local arenas (sharding.vocab_sharded_p2p_one_gpu): the same kernels, slot
addressing, counters and slot-set rotation as the multi-GPU path, launched in an order where no kernel waits on a
later launch.  Checked: every rank's dh_s (and FKL loss) equals, bit for bit, the rank-order sum of the shards'
partials from kd_vocab_backward (the NCCL path's inputs); the loss / dh_s / dW_s equal the fp64 oracle within the
north-star tolerances; two consecutive steps on the same arenas (counter continuity); exchange chunks smaller than
P rows (owners with no rows)."""
import numpy as np
import pytest
import torch

import kd_inputs as KI
from tests.kdtest_util import (LOSS_ATOL, LOSS_RTOL, assert_grad_close, assert_kd_close, dev_bf16, oracle_run)

pytestmark = pytest.mark.gpu


def kd():
    import paper_2603_01875_b200 as m
    return m


def _reference(Ht, Wt, Hs, Ws, m, spans, bounds, *, V, T, kind, beta=0.5, want_dW=True):
    """The NCCL path's arithmetic: per exchange chunk, each shard's partial dh_s / loss from kd_vocab_backward, summed
    over shards in rank order in fp32 (what the owner's combine does)."""
    N, d_s = Hs.shape[0], Ws.shape[1]
    dh = torch.zeros(N, d_s, device="cuda")
    loss = torch.zeros(N, device="cuda")
    dW = [None] * len(bounds)
    for i, (a, b) in enumerate(spans):
        m_c = None if m is None else m[a:b]
        fix = kind in ("jsd", "tvd")
        recs = torch.stack([kd().vocab_stats(Ht[a:b], Wt[v0:v1], Hs[a:b], Ws[v0:v1], m_c, vocab=V, v_begin=v0, T=T,
                                             kind=kind, chunk_tokens=(b - a) if fix else 0) for v0, v1 in bounds])
        acc_dh = torch.zeros(b - a, d_s, device="cuda")
        acc_l = torch.zeros(b - a, device="cuda")
        if fix:
            parts = [kd().vocab_partials(Ht[a:b], Wt[v0:v1], Hs[a:b], Ws[v0:v1], recs, m_c, vocab=V, v_begin=v0, T=T,
                                         kind=kind, beta=beta, want_dW=want_dW, accumulate_dW=i > 0)
                     for v0, v1 in bounds]
            kj_all = torch.stack([kj for kj, _ in parts])
        for r, (v0, v1) in enumerate(bounds):
            if fix:
                res = kd().vocab_finish(parts[r][1], Ht[a:b], Wt[v0:v1], Hs[a:b], Ws[v0:v1], kj_all, m_c, dW_s=dW[r])
            else:
                res = kd().vocab_backward(Ht[a:b], Wt[v0:v1], Hs[a:b], Ws[v0:v1], recs, m_c, vocab=V, v_begin=v0,
                                          T=T, kind=kind, want_dW=want_dW, accumulate_dW=i > 0, dW_s=dW[r])
            dW[r] = res.dW_s
            acc_dh = acc_dh + res.dh_s
            acc_l = acc_l + res.loss if kind == "fkl" else res.loss
        dh[a:b] = acc_dh
        loss[a:b] = acc_l
    return loss, dh, dW


@pytest.mark.parametrize("P,kind,N,chunk", [(2, "fkl", 520, 128), (3, "rkl", 520, 128), (8, "fkl", 517, 128),
                                            (4, "rkl", 300, 0), (2, "jsd", 520, 128), (3, "tvd", 517, 256)])
def test_p2p_exchange_equals_rank_order_sum(P, kind, N, chunk):
    from paper_2603_01875_b200.sharding import P2PExchange, vocab_shard_bounds, vocab_sharded_p2p_one_gpu
    d_t, d_s, V, T = 256, 128, 5000, 1.5
    mask = (np.random.default_rng(P).random(N) > 0.2).astype(np.uint8)
    inp = KI.make_inputs(N, d_t, d_s, V, seed=70 + P, mask=mask)
    Ht, Hs, Wt, Ws = dev_bf16(inp.H_t), dev_bf16(inp.H_s), dev_bf16(inp.W_t), dev_bf16(inp.W_s)
    m = torch.from_numpy(mask).cuda()
    bounds = vocab_shard_bounds(V, P)
    c = chunk if chunk > 0 else N
    spans = [(a, min(N, a + c)) for a in range(0, N, c)]
    exs = P2PExchange.local_group(P, d_s, max_rows=c, max_tokens=N)
    beta = 0.3
    ref_loss, ref_dh, ref_dW = _reference(Ht, Wt, Hs, Ws, m, spans, bounds, V=V, T=T, kind=kind, beta=beta)
    for step in range(2):  # the second step reuses the arenas: counters continue, slot sets keep rotating
        out = vocab_sharded_p2p_one_gpu(Ht, Wt, Hs, Ws, m, exchanges=exs, T=T, kind=kind, beta=beta, want_dW=True,
                                        exchange_chunk=c)
        torch.cuda.synchronize()
        assert all(ex.chunks == (step + 1) * len(spans) for ex in exs)
        for r, (loss, dh, dW) in enumerate(out):
            assert torch.equal(dh, ref_dh), f"rank {r} step {step}: dh_s differs from the rank-order sum"
            assert torch.equal(loss, ref_loss), f"rank {r} step {step}: loss differs"
            assert torch.equal(dW, ref_dW[r]), f"rank {r} step {step}: dW_s rows differ"
    loss, dh_ref, dW_ref = oracle_run(inp, T=T, kind=kind, beta=beta, want_dW=True)
    assert_kd_close("loss (p2p)", out[0][0].cpu().numpy(), loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s (p2p)", out[0][1].cpu().numpy(), dh_ref)
    dW = torch.cat([o[2] for o in out]).cpu().numpy()
    assert_grad_close("dW_s (p2p)", dW, dW_ref)
    assert (out[0][1][torch.from_numpy(mask == 0).cuda()] == 0).all()  # masked rows: exact zeros from the owner


def test_p2p_argument_errors():
    from paper_2603_01875_b200 import kdfused as K
    from paper_2603_01875_b200.sharding import P2PExchange
    ex = P2PExchange.local_group(2, 128, max_rows=64, max_tokens=64)[0]
    with pytest.raises(K.KDError) as e:
        K.p2p_combine(ex.x, 3, 64, 0, with_loss=True, target=2)   # set outside [0, 3)
    assert e.value.status == 1
    with pytest.raises(K.KDError) as e:
        K.p2p_combine(ex.x, 0, 65, 0, with_loss=True, target=2)   # more rows than the arena holds
    assert e.value.status == 2
    bad = K.make_p2p(2, 2, 128, 64, 64, [ex.own.data_ptr()] * 2)  # rank outside [0, world)
    with pytest.raises(K.KDError) as e:
        K.p2p_wait(bad, 0)
    assert e.value.status == 1


@pytest.mark.parametrize("name,P", [("c2", 8), ("c3_jsd", 4)])
def test_p2p_full_vocab_sampled(name, P):
    """BASELINE config shapes (d_t 4096, d_s 2048, V = 151936; c3: T = 2, prompt/padding mask), 8192 tokens in
    2048-token exchange chunks, P emulated ranks: the p2p result equals the rank-order sum of the shards' partials bit
    for bit on every rank, and 48 sampled tokens match the fp64 oracle."""
    from paper_2603_01875_b200.sharding import P2PExchange, vocab_shard_bounds, vocab_sharded_p2p_one_gpu
    cfg = KI.CONFIGS[name]
    N, c = 8192, 2048
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
    H_t, H_s = KI.make_hidden(N, W_t, W_s, seed=1001, head_seed=1000)
    mask = KI.make_mask(KI.KDConfig(**{**cfg.__dict__, "n_seq": N // cfg.seq_len})) if cfg.mask != "none" else None
    inp = KI.KDInputs(H_t, W_t, H_s, W_s, mask)
    Ht, Hs, Wt, Ws = dev_bf16(H_t), dev_bf16(H_s), dev_bf16(W_t), dev_bf16(W_s)
    m = None if mask is None else torch.from_numpy(mask).cuda()
    bounds = vocab_shard_bounds(cfg.vocab, P)
    spans = [(a, min(N, a + c)) for a in range(0, N, c)]
    ref_loss, ref_dh, _ = _reference(Ht, Wt, Hs, Ws, m, spans, bounds, V=cfg.vocab, T=cfg.temperature, kind=cfg.kind,
                                     beta=cfg.jsd_beta, want_dW=False)
    exs = P2PExchange.local_group(P, cfg.d_s, max_rows=c, max_tokens=N)
    out = vocab_sharded_p2p_one_gpu(Ht, Wt, Hs, Ws, m, exchanges=exs, T=cfg.temperature, kind=cfg.kind,
                                    beta=cfg.jsd_beta, exchange_chunk=c)
    torch.cuda.synchronize()
    for r, (loss, dh, _) in enumerate(out):
        assert torch.equal(dh, ref_dh), f"rank {r}: dh_s differs from the rank-order sum"
        assert torch.equal(loss, ref_loss), f"rank {r}: loss differs"
    live = np.arange(N) if mask is None else np.flatnonzero(mask)
    rows = np.sort(np.random.default_rng(3).choice(live, 48, replace=False))
    loss, dh, _ = oracle_run(inp, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, rows=rows)
    assert_kd_close("loss (p2p, full V)", out[0][0].cpu().numpy()[rows], loss, LOSS_RTOL, LOSS_ATOL)
    assert_grad_close("dh_s (p2p, full V)", out[0][1].cpu().numpy()[rows], dh)
