"""Multi-process (world_size 2, gloo, CPU) test of the host protocol of the peer-memory exchange
(sharding.vocab_sharded_fwd_bwd(exchange=P2PExchange), kdfused.h kd_p2p).

The CUDA kernels and peer mappings cannot run here, so the kernel-side callables are CPU stand-ins over
shared-memory "arenas" created by the parent: the stats stand-in writes its record into every rank's record set and
raises their record counters; the backward stand-in waits for the P records and writes each partial dh_s / loss row into its
owner's receive slot (owner = row // R, R = ceil(n / P)) of the chunk's slot set and then raises its arrival
counter; the combine stand-in polls the arrivals, sums the slots in rank order, stores the sum into every rank's
dh_out / loss_out and raises the done counters; the wait stand-in polls the done counters.  Every counter entry
is written by one process only (a per-source entry, as in the arena's counter block), so the stand-ins need no
atomics, and a wait needs every source at the chunk (an early version summed the sources: a rank running a chunk
ahead satisfied the sum — this test caught it).  What is under test is the
product's protocol: slot-set rotation over five exchange chunks, the set-reuse waits, the deferred combine, the
counter targets across two steps, and the result, against the fp64 oracle."""
import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.test_sharding_gloo import _backward_standin, _finish_standin, _partials_standin, _stats_standin

N, D_T, D_S, V, CHUNK, WORLD = 40, 32, 24, 300, 8, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _arena(world, max_rows, max_tokens, d_s):
    R = -(-max_rows // world)
    return dict(arr=torch.zeros(world, dtype=torch.int64).share_memory_(),    # [src]: chunks src pushed here
                done=torch.zeros(world, dtype=torch.int64).share_memory_(),   # [owner]: chunks owner combined
                nrec=torch.zeros(world, dtype=torch.int64).share_memory_(),   # [src]: records src wrote here
                nkj=torch.zeros(world, dtype=torch.int64).share_memory_(),    # [src]: (K, J) src wrote here
                recs=torch.zeros(3, world, 5, max_rows, dtype=torch.float64).share_memory_(),
                kj=torch.zeros(3, world, 2, max_rows, dtype=torch.float64).share_memory_(),
                slots=torch.zeros(3, world, R, d_s, dtype=torch.float64).share_memory_(),
                lslots=torch.zeros(3, world, R, dtype=torch.float64).share_memory_(),
                dh=torch.zeros(max_tokens, d_s, dtype=torch.float64).share_memory_(),
                loss=torch.zeros(max_tokens, dtype=torch.float64).share_memory_())


class _X:
    """Stand-in for the kd_p2p view: this rank and every rank's arena."""

    def __init__(self, rank, arenas):
        self.rank, self.arenas, self.world = rank, arenas, len(arenas)


def _poll(fn, what):
    t0 = time.time()
    while not fn():
        if time.time() - t0 > 60:
            raise TimeoutError(what)
        time.sleep(0.001)


def _stats_p2p_standin(h_t, Wt, h_s, Ws, mask, *, x, set, vocab, v_begin, T, kind, chunk_tokens):
    time.sleep(0.004 * (x.world - 1 - x.rank))  # skew: rank 0 lags in its stats, rank 1 in its backward
    rec = _stats_standin(h_t, Wt, h_s, Ws, mask, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                         chunk_tokens=chunk_tokens)
    n = h_t.shape[0]
    for a in x.arenas:  # the all-gather: this rank's record into slot [rank] of every rank's record set
        a["recs"][set, x.rank, :, :n] = rec
    for a in x.arenas:
        a["nrec"][x.rank] += 1


def _backward_p2p_standin(h_t, Wt, h_s, Ws, recs, mask, *, x, set, vocab, v_begin, T, kind, loss_scale, want_dW,
                          accumulate_dW, dW_s, chunk_tokens, records_target):
    me = x.arenas[x.rank]
    n = h_t.shape[0]
    time.sleep(0.004 * x.rank)
    assert recs is None  # the product path reads the records from the arena
    _poll(lambda: int(me["nrec"].min()) >= records_target, f"records {records_target}")
    recs = me["recs"][set, :, :, :n].clone()
    r = _backward_standin(h_t, Wt, h_s, Ws, recs, mask, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                          loss_scale=loss_scale, want_dW=want_dW, accumulate_dW=accumulate_dW, dW_s=dW_s,
                          chunk_tokens=chunk_tokens)
    _push_rows(x, set, n, mask, r.dh_s, r.loss)
    r.dh_s = None
    if kind != "rkl":
        r.loss = None
    return r


def _push_rows(x, set, n, mask, dh, loss):
    R = -(-n // x.world)
    for row in range(n):  # masked rows are not pushed (the owner writes their zeros)
        if mask is not None and mask[row] == 0:
            continue
        j = row // R
        x.arenas[j]["slots"][set, x.rank, row - j * R] = dh[row]
        if loss is not None:
            x.arenas[j]["lslots"][set, x.rank, row - j * R] = loss[row]
    for a in x.arenas:
        a["arr"][x.rank] += 1


def _partials_p2p_standin(h_t, Wt, h_s, Ws, mask, *, x, set, vocab, v_begin, T, kind, beta, loss_scale, want_dW,
                          accumulate_dW, records_target):
    me = x.arenas[x.rank]
    n = h_t.shape[0]
    time.sleep(0.004 * x.rank)
    _poll(lambda: int(me["nrec"].min()) >= records_target, f"records {records_target}")
    kj, st = _partials_standin(h_t, Wt, h_s, Ws, me["recs"][set, :, :, :n].clone(), mask, vocab=vocab,
                               v_begin=v_begin, T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                               accumulate_dW=accumulate_dW, chunk_tokens=n)
    for a in x.arenas:  # the (K, J) all-gather through the arenas
        a["kj"][set, x.rank, :, :n] = kj
    for a in x.arenas:
        a["nkj"][x.rank] += 1
    return st


def _finish_p2p_standin(st, h_t, Wt, h_s, Ws, mask, *, x, set, kj_target, dW_s=None):
    me = x.arenas[x.rank]
    n = h_t.shape[0]
    _poll(lambda: int(me["nkj"].min()) >= kj_target, f"kj {kj_target}")
    r = _finish_standin(st, h_t, Wt, h_s, Ws, me["kj"][set, :, :, :n].clone(), mask, dW_s=dW_s)
    _push_rows(x, set, n, mask, r.dh_s, None)
    r.dh_s = None
    return r


def _combine_standin(x, set, n_rows, row0, mask, *, with_loss, target):
    me = x.arenas[x.rank]
    _poll(lambda: int(me["arr"].min()) >= target, f"arrivals {target}")
    R = -(-n_rows // x.world)
    r0 = x.rank * R
    for i in range(max(0, min(n_rows, r0 + R) - r0)):
        live = mask is None or mask[r0 + i] != 0
        acc = torch.zeros(me["slots"].shape[-1], dtype=torch.float64)
        lacc = torch.zeros((), dtype=torch.float64)
        if live:
            for src in range(x.world):  # rank order
                acc = acc + me["slots"][set, src, i]
                lacc = lacc + me["lslots"][set, src, i]
        for a in x.arenas:
            a["dh"][row0 + r0 + i] = acc
            if with_loss:
                a["loss"][row0 + r0 + i] = lacc
    for a in x.arenas:
        a["done"][x.rank] += 1


def _wait_standin(x, target):
    me = x.arenas[x.rank]
    _poll(lambda: int(me["done"].min()) >= target, f"done {target}")


def _worker(rank, world, port, kind, arenas, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import kd_inputs as KI
        from paper_2603_01875_b200.sharding import P2PExchange, vocab_shard_bounds, vocab_sharded_fwd_bwd
        mask = (np.arange(N) % 7 != 3).astype(np.uint8)
        inp = KI.make_inputs(N, D_T, D_S, V, seed=4, mask=mask)
        ht, hs, Wt, Ws = (torch.tensor(KI.bf16_to_f64(t)) for t in (inp.H_t, inp.H_s, inp.W_t, inp.W_s))
        a, b = vocab_shard_bounds(V, world, granule=16)[rank]
        ex = P2PExchange(world, rank, D_S, CHUNK, N, [0] * world, own=None)
        ex.x = _X(rank, arenas)
        fns = dict(stats=_stats_p2p_standin, backward=_backward_p2p_standin, partials=_partials_p2p_standin,
                   finish=_finish_p2p_standin, combine=_combine_standin, wait=_wait_standin,
                   outputs=lambda e, n: (e.x.arenas[e.rank]["dh"][:n].clone(), e.x.arenas[e.rank]["loss"][:n].clone()))
        outs = []
        for step in range(2):  # counters and slot sets carry over into the second step
            r = vocab_sharded_fwd_bwd(ht, Wt[a:b], hs, Ws[a:b], torch.tensor(mask), vocab=V, v_begin=a, T=1.3,
                                      kind=kind, beta=0.3, want_dW=True, exchange_chunk=CHUNK, exchange=ex,
                                      p2p_fns=fns)
            outs.append((r.loss.numpy().copy(), r.dh_s.numpy().copy(), r.dW_s.numpy().copy()))
            dist.barrier()  # the next step overwrites dh_out: both ranks have read this one
        q.put((rank, (a, b), ex.chunks, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["fkl", "rkl", "jsd", "tvd"])
def test_p2p_exchange_protocol_world2(kind):
    import kd_inputs as KI
    from oracle.kd_oracle import kd_fused_fwd_bwd
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    arenas = [_arena(WORLD, CHUNK, N, D_S) for _ in range(WORLD)]
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, kind, arenas, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(WORLD)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mask = (np.arange(N) % 7 != 3).astype(np.uint8)
    inp = KI.make_inputs(N, D_T, D_S, V, seed=4, mask=mask)
    f = KI.bf16_to_f64
    loss, dh, dW = kd_fused_fwd_bwd(f(inp.H_t), f(inp.W_t), f(inp.H_s), f(inp.W_s), mask, T=1.3, kind=kind,
                                    beta=0.3, want_dW=True)
    dW_cat = np.zeros_like(dW)
    n_chunks = -(-N // CHUNK)
    for rank, (a, b), chunks, outs in res:
        assert chunks == 2 * n_chunks
        for l, d, dws in outs:
            np.testing.assert_allclose(l, loss, rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(d, dh, rtol=1e-11, atol=1e-13)
            dW_cat[a:b] = dws
    np.testing.assert_allclose(dW_cat, dW, rtol=1e-11, atol=1e-13)
    for a in arenas:  # every owner combined every chunk of both steps for every rank
        assert int(a["done"].sum()) == WORLD * 2 * n_chunks and int(a["arr"].sum()) == WORLD * 2 * n_chunks
        assert int(a["nrec"].sum()) == WORLD * 2 * n_chunks
        assert int(a["nkj"].sum()) == (WORLD * 2 * n_chunks if kind in ("jsd", "tvd") else 0)
