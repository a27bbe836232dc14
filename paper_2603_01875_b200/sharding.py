"""Multi-GPU host logic: how the hot path is partitioned across ranks (one process per GPU).

Two layouts (BASELINE.json north_star: "vocabulary sharding of W_t/W_s ... token sharding is reported
alongside"):

* token sharding — rank r owns tokens [t0, t1) and full heads.  Per-token outputs need no exchange at
  all (the path is data-parallel); only dW_s (if requested) is a sum over ranks.
* vocabulary sharding — rank r owns LM-head rows [v0, v1) (128-row granules; V = 151936 = 128·1187) and
  every token.  Exchanges: (1) all-gather of the per-token pass-1 records (20 B/token/rank), merged in rank
  order by the kernels (deterministic); (2) all-reduce SUM of the partial dL/dh_s (FKL: and of the partial
  per-token loss, 4 B/token).  dW_s rows stay local.
  JSD/TVD add (1b): all-gather of the per-token (K, J) partials (8 B/token/rank) between the shards'
  pass 2 and the gradient fix-up, token chunk by token chunk.

The collectives go through ``torch.distributed`` (NCCL over NVLink on the GPU box; gloo in the CPU tests);
the kernels on either side are the library's (``kd_vocab_stats`` / ``kd_vocab_backward``, and for JSD/TVD
``kd_vocab_partials`` / ``kd_vocab_finish``).
"""
from __future__ import annotations

import os

from typing import Callable

import torch
import torch.distributed as dist

GRANULE = 128


def vocab_shard_bounds(vocab: int, world: int, granule: int = GRANULE) -> list[tuple[int, int]]:
    """Contiguous vocabulary ranges of whole granules, as even as possible (rank order)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    n_gran = -(-vocab // granule)
    edges = [min(vocab, (n_gran * i // world) * granule) for i in range(world + 1)]
    return [(edges[i], edges[i + 1]) for i in range(world)]


def token_shard_bounds(n_tokens: int, world: int) -> list[tuple[int, int]]:
    edges = [n_tokens * i // world for i in range(world + 1)]
    return [(edges[i], edges[i + 1]) for i in range(world)]


def _distributed() -> bool:
    """False when no process group exists: a one-rank job runs the same protocol with identity exchanges."""
    return dist.is_available() and dist.is_initialized()


def gather_records(rec: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather this rank's [5, N] record into [P, 5, N] in rank order."""
    if not _distributed():
        return rec.contiguous()[None]
    world = dist.get_world_size(group)
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec.contiguous(), group=group)
    return torch.stack(out)


def gather_kj(kj: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather this rank's [2, n] (K, J) partials into [P, 2, n] in rank order."""
    if not _distributed():
        return kj.contiguous()[None]
    world = dist.get_world_size(group)
    out = [torch.empty_like(kj) for _ in range(world)]
    dist.all_gather(out, kj.contiguous(), group=group)
    return torch.stack(out)


def _all_reduce_sum(t: torch.Tensor, group=None):
    if _distributed():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _reduce_scatter_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum over the group of [N, ...] and keep this rank's row slice (rows j·N/P .. (j+1)·N/P, rank order): the
    gradient / loss of the rank's own tokens when the group's tokens are its members' slices concatenated."""
    if not _distributed():
        return t
    world = dist.get_world_size(group)
    if t.shape[0] % world:
        raise ValueError(f"dh_reduce='scatter' needs the group's {t.shape[0]} tokens divisible by {world} ranks")
    if dist.get_backend(group) == "gloo":  # gloo has no reduce-scatter: all-reduce, keep the own rows
        t = t.contiguous()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return _own_rows(t, group)
    out = torch.empty((t.shape[0] // world,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.reduce_scatter_tensor(out, t.contiguous(), op=dist.ReduceOp.SUM, group=group)
    return out


def _own_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    if not _distributed():
        return t
    world, j = dist.get_world_size(group), dist.get_rank(group)
    n = t.shape[0] // world
    return t[j * n:(j + 1) * n]


class _Result:
    def __init__(self, loss, dh_s, dW_s):
        self.loss, self.dh_s, self.dW_s = loss, dh_s, dW_s


class _Done:
    """Stand-in for a finished collective (no process group: identity exchange)."""

    def wait(self):
        return None


def _all_gather_async(t: torch.Tensor, group=None):
    """Start the all-gather of this rank's [..] tensor into [P, ..] (rank order); returns (out, work).

    NCCL: the collective is enqueued behind the current stream's work and runs on NCCL's stream, so the caller
    keeps launching kernels; ``work.wait()`` makes the current stream (not the host) wait for it."""
    if not _distributed():
        return t.contiguous()[None], _Done()
    world = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "gloo":
        parts = [torch.empty_like(t) for _ in range(world)]
        work = dist.all_gather(parts, t, group=group, async_op=True)
        return parts, work
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    work = dist.all_gather_into_tensor(out, t, group=group, async_op=True)
    return out, work


def _gathered(out):
    return torch.stack(out) if isinstance(out, list) else out


def _all_reduce_async(t: torch.Tensor, group=None):
    if not _distributed():
        return _Done()
    return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=True)


def library_chunk(d_t: int, d_s: int) -> int:
    """The library's default token chunk (kd_api.cu make_plan: ~36 MiB of H_t|H_s rows in [1024, 4096], rounded up to
    the 256-row pair tile) — mirrored here so FKL/RKL exchange chunks hold whole library chunks."""
    nc = (36 << 20) // (2 * (d_t + d_s))
    nc = min(4096, max(1024, nc))
    return -(-nc // 256) * 256


def default_exchange_chunk(n_tokens: int, v_rows: int, kind: str, d_t: int = 0, d_s: int = 0) -> int:
    """Tokens per pipelined exchange chunk of the vocab-sharded step.

    Each chunk's pass 1 runs while the previous chunk's records are all-gathered, and each chunk's partial-dh
    all-reduce runs under the next chunk's kernels, so only the last chunk's all-reduce is exposed; more chunks
    overlap more but shorten each launch.  JSD/TVD keep the chunk's G planes (12 B per (token, v)) between their two
    calls, so their chunk is bounded to ~5 GB of planes: 8192 tokens at P = 8, at most 5376 at P = 2, balanced over the chunks (measured on one GPU
    simulating rank 0, c3 JSD: per-GPU efficiency at P = 8 0.67 with 2048-token chunks -> 0.85 with 8192;
    scripts/gpu/simv_jsd*.sh).  FKL/RKL: 8192 tokens (four exchange chunks at config 2).  KD_VOCAB_FIX_CHUNK
    overrides."""
    if "KD_VOCAB_FIX_CHUNK" in os.environ:
        return max(1, int(os.environ["KD_VOCAB_FIX_CHUNK"]))
    cap = 8192
    if kind in ("jsd", "tvd"):
        cap = max(4096, min(8192, int(5e9 / (12 * max(1, v_rows))) // 256 * 256))
    if n_tokens <= cap:
        return max(1, n_tokens)
    # FKL/RKL with the widths given: whole library chunks per exchange chunk (c2: 3 x 3072 = 9216 instead of 8192 =
    # 3072 + 3072 + 2048; simulated P = 8 rank step 17.38 -> 17.09 ms, profiles/r02_ab.md)
    if kind not in ("jsd", "tvd") and d_t > 0 and d_s > 0:
        lc = library_chunk(d_t, d_s)
        per = -(-cap // lc)                       # library chunks per exchange chunk
        return min(n_tokens, per * lc)
    # balance the chunks: a ragged tail of a few hundred tokens fills a fraction of a wave of output tiles (c3 JSD at
    # P = 2: 5376-token chunks left a 512-token tail, per-rank efficiency 0.86)
    n_chunks = -(-n_tokens // cap)
    return min(cap, -(-(-(-n_tokens // n_chunks)) // 256) * 256)


class P2PExchange:
    """One rank's end of the peer-memory exchange of the vocab-sharded step (kdfused.h kd_p2p).

    Each rank owns an arena (receive slots, counters, the step's dh_out / loss_out) and maps every peer's arena:
    the library's kernels then push the partial dh_s rows straight from the dh reduction into their owners' slots
    (NVLink peer stores) and the owners store the rank-order sums into every rank's dh_out — no NCCL call on the
    data path.  ``create`` builds it over a process group (CUDA IPC handles exchanged with all_gather_object);
    ``local_group`` builds P of them inside one process on one device (the one-GPU emulation the tests use).
    ``chunks`` counts the exchange chunks completed, from which every counter target follows (kdfused.h)."""

    def __init__(self, world: int, rank: int, d_s: int, max_rows: int, max_tokens: int, arenas, own: torch.Tensor,
                 mapped=()):
        from . import kdfused
        self.world, self.rank, self.d_s = world, rank, d_s
        self.max_rows, self.max_tokens = max_rows, max_tokens
        self.own = own              # keeps this rank's arena alive
        self.mapped = list(mapped)  # HandoffTensor views of the peers' arenas (closed by close())
        self.x = kdfused.make_p2p(world, rank, d_s, max_rows, max_tokens, arenas)
        self.chunks = 0

    @staticmethod
    def _alloc(world, d_s, max_rows, max_tokens, device) -> torch.Tensor:
        from . import kdfused
        n = kdfused.p2p_arena_bytes(world, max_rows, max_tokens, d_s)
        return torch.zeros(n, dtype=torch.uint8, device=device)  # counters start at 0

    @classmethod
    def local_group(cls, world: int, d_s: int, max_rows: int, max_tokens: int, device="cuda") -> list:
        """P exchanges sharing one process and device (every 'peer' arena is a local allocation)."""
        arenas = [cls._alloc(world, d_s, max_rows, max_tokens, device) for _ in range(world)]
        ptrs = [a.data_ptr() for a in arenas]
        return [cls(world, r, d_s, max_rows, max_tokens, ptrs, arenas[r]) for r in range(world)]

    @classmethod
    def create(cls, group, d_s: int, max_rows: int, max_tokens: int, device=None):
        """Collective over ``group``: allocate and zero this rank's arena, exchange CUDA IPC handles, map the peers."""
        from . import kdfused
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        own = cls._alloc(world, d_s, max_rows, max_tokens, dev)
        torch.cuda.synchronize(dev)
        shape = (d_s, max_rows, max_tokens, own.numel())
        handles = [None] * world
        dist.all_gather_object(handles, (shape, kdfused.handoff_export(own)), group=group)
        if any(sh != shape for sh, _ in handles):  # every rank's kernels address the peers' arenas with ITS layout
            raise ValueError(f"P2PExchange.create: ranks disagree on (d_s, max_rows, max_tokens, arena bytes): "
                             f"{[sh for sh, _ in handles]}")
        handles = [h for _, h in handles]
        ptrs, mapped = [], []
        for j, h in enumerate(handles):
            if j == rank:
                ptrs.append(own.data_ptr())
            else:
                m = kdfused.HandoffTensor(h, (own.numel(),), torch.uint8, device=dev)
                mapped.append(m)
                ptrs.append(m.ptr)
        dist.barrier(group=group)
        return cls(world, rank, d_s, max_rows, max_tokens, ptrs, own, mapped)

    def set_of(self, chunk: int) -> int:
        return chunk % 3

    # every counter is per source rank (kdfused.h): after chunk g, each source has raised its counter g + 1 times
    def arrivals_target(self, chunk: int) -> int:
        return chunk + 1

    def done_target(self, chunk: int) -> int:
        return chunk + 1

    def records_target(self, chunk: int) -> int:
        return chunk + 1

    def close(self):
        for m in self.mapped:
            m.close()
        self.mapped = []


def _p2p_step(ex: P2PExchange, spans, stats_p2p, backward_p2p, combine, wait, outputs, *, mask, kind, N, device):
    """The per-rank p2p pipeline of one step — no NCCL call on the data path:

        stats_p2p(0)
        per chunk i:  stats_p2p(i+1)  [records into every rank's arena]
                      [wait done(i-3)]  backward_p2p(i)  [waits for the P records of i; partial rows -> owners]
                      combine(i-1)  (deferred behind chunk i's kernels: the P arrivals of i-1 are long there)
        end:          combine(last) ; wait done(all)

    Chunk g (counted over the exchange's life) uses set g % 3 of the dh slots and of the records.  Reusing a dh slot
    set needs every owner's combine of chunk g - 3 (a done target); a record set is rewritten by stats_p2p(g) only
    after this rank ran combine(g - 3), which waited for every rank's backward of g - 3 (the set's last reader).
    The previous step ended waiting for all of its chunks."""
    base = ex.chunks
    n = len(spans)
    loss_rkl = None
    dW = None

    def do_combine(i):
        a, b = spans[i]
        g = base + i
        combine(ex, ex.set_of(g), b - a, a, None if mask is None else mask[a:b], with_loss=(kind == "fkl"),
                target=ex.arrivals_target(g))

    if n:
        stats_p2p(0, ex.set_of(base))
    for i, (a, b) in enumerate(spans):
        g = base + i
        if i + 1 < n:
            stats_p2p(i + 1, ex.set_of(g + 1))
        if i >= 3:
            wait(ex, ex.done_target(g - 3))
        r = backward_p2p(i, ex.set_of(g), dW, ex.records_target(g))
        if kind != "fkl":  # RKL / JSD / TVD: every rank derives the full loss itself
            if loss_rkl is None:  # the kernels' dtype (fp32; the CPU test stand-ins return fp64)
                loss_rkl = torch.zeros(N, dtype=r.loss.dtype, device=r.loss.device)
            loss_rkl[a:b] = r.loss
        if r.dW_s is not None:
            dW = r.dW_s
        if i >= 1:
            do_combine(i - 1)
    if n:
        do_combine(n - 1)
        wait(ex, ex.done_target(base + n - 1))
    ex.chunks = base + n
    dh_out, loss_out = outputs(ex, N)
    if kind != "fkl" and loss_rkl is None:  # no tokens
        loss_rkl = torch.zeros(0, dtype=torch.float32, device=device)
    return _Result(loss_rkl if kind != "fkl" else loss_out, dh_out, dW)


def vocab_sharded_fwd_bwd(h_t, W_t_shard, h_s, W_s_shard, mask=None, *, vocab: int, v_begin: int, group=None,
                          T=1.0, kind="fkl", beta=0.5, loss_scale=1.0, want_dW=False, accumulate_dW=False,
                          dW_s=None, chunk_tokens=0, exchange_chunk=0, stats_fn: Callable | None = None,
                          backward_fn: Callable | None = None, partials_fn: Callable | None = None,
                          finish_fn: Callable | None = None, dh_reduce: str = "all",
                          exchange: "P2PExchange | None" = None, p2p_fns: dict | None = None):
    """One vocab-sharded step on this rank; every rank of ``group`` holds the same tokens and its own
    LM-head rows [v_begin, v_begin + V_r).  Returns a result whose dh_s is the full gradient (all-reduced) and whose
    dW_s holds this rank's rows.

    Pipelined over exchange chunks of ``exchange_chunk`` tokens (default: ``default_exchange_chunk``):

        FKL / RKL   stats(c+1) ‖ all-gather records(c) ;  backward(c) ‖ all-reduce partial dh(c-1) (+ FKL loss)
        JSD / TVD   stats(c+1) ‖ all-gather records(c) ;  partials(c) -> all-gather (K, J)(c) -> finish(c)
                    ‖ all-reduce partial dh(c-1)

    (‖ = concurrent: NCCL runs the collective on its own stream while this stream launches the next kernels; the
    kernels merge records and (K, J) partials in rank order, so the result is deterministic for a fixed P.)

    dh_reduce="scatter": when the group's tokens are its members' equal slices concatenated in rank order (each rank
    contributes its own batch, bench.py's 2-D grid), every rank keeps dh_s / loss of its own slice only: one
    reduce-scatter at the end instead of the per-chunk all-reduces.

    ``exchange`` (a P2PExchange, dh_reduce="all"): records (and JSD/TVD's (K, J) partials) are all-gathered and the
    partial dh_s / FKL loss leave the library's dh
    reduction straight into their owners' slots in peer memory and the owners' rank-order sums land in every rank's
    arena (kdfused.h kd_p2p) — no NCCL call for the dh exchange; the returned dh_s / loss are views of the arena,
    valid until the next step on it.  ``p2p_fns`` substitutes {stats, backward, partials, finish, combine, wait, outputs}
    (CPU stand-ins).

    ``chunk_tokens`` is the library's internal token chunk (kd_problem.chunk_tokens, 0 = its default).  The
    kernel-side callables default to the CUDA entry points; tests substitute CPU stand-ins to exercise this exchange
    logic under gloo.
    """
    if dh_reduce not in ("all", "scatter"):
        raise ValueError(f"dh_reduce must be 'all' or 'scatter' (got {dh_reduce!r})")
    fix = kind in ("jsd", "tvd")
    if stats_fn is None or (fix and (partials_fn is None or finish_fn is None)) or (not fix and backward_fn is None):
        from . import kdfused
        stats_fn = stats_fn or kdfused.vocab_stats
        backward_fn = backward_fn or kdfused.vocab_backward
        partials_fn = partials_fn or kdfused.vocab_partials
        finish_fn = finish_fn or kdfused.vocab_finish
    N = h_t.shape[0]
    d_s = W_s_shard.shape[1]
    chunk = exchange_chunk if exchange_chunk > 0 else default_exchange_chunk(N, W_s_shard.shape[0], kind,
                                                                             W_t_shard.shape[1], d_s)
    if fix and chunk_tokens > 0:
        chunk = min(chunk, chunk_tokens)  # the JSD/TVD pair runs one library chunk per call
    spans = [(a, min(N, a + chunk)) for a in range(0, N, chunk)]
    per_chunk = dh_reduce == "all"
    loss = dh = None
    pending = []  # per-chunk all-reduces in flight

    def stats(i):
        a, b = spans[i]
        m_c = None if mask is None else mask[a:b]
        rec = stats_fn(h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, m_c, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                       chunk_tokens=(b - a) if fix else chunk_tokens)
        return _all_gather_async(rec, group)

    if exchange is not None:
        if dh_reduce != "all":
            raise ValueError("the peer exchange serves dh_reduce='all'")
        if N > exchange.max_tokens or chunk > exchange.max_rows:
            raise ValueError(f"step of {N} tokens / exchange chunk {chunk} exceeds the arena "
                             f"({exchange.max_tokens} / {exchange.max_rows})")
        from . import kdfused
        f = dict(stats=kdfused.vocab_stats_p2p, backward=kdfused.vocab_backward_p2p,
                 partials=kdfused.vocab_partials_p2p, finish=kdfused.vocab_finish_p2p, combine=kdfused.p2p_combine,
                 wait=kdfused.p2p_wait, outputs=lambda ex, n: kdfused.p2p_outputs(ex.x, h_t.device, n, d_s))
        f.update(p2p_fns or {})

        def stats_p2p(i, set_):
            a, b = spans[i]
            f["stats"](h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, None if mask is None else mask[a:b], x=exchange.x,
                       set=set_, vocab=vocab, v_begin=v_begin, T=T, kind=kind, chunk_tokens=chunk_tokens)

        def backward_p2p(i, set_, dW_cur, rec_target):
            a, b = spans[i]
            m_c = None if mask is None else mask[a:b]
            acc = accumulate_dW or i > 0
            if fix:  # JSD/TVD: (K, J) partials all-gathered through the arena between the two calls
                st = f["partials"](h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, m_c, x=exchange.x, set=set_, vocab=vocab,
                                   v_begin=v_begin, T=T, kind=kind, beta=beta, loss_scale=loss_scale,
                                   want_dW=want_dW, accumulate_dW=acc, records_target=rec_target)
                return f["finish"](st, h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, m_c, x=exchange.x, set=set_,
                                   kj_target=rec_target, dW_s=dW_cur if i > 0 else dW_s)
            return f["backward"](h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, None,
                                 None if mask is None else mask[a:b], x=exchange.x, set=set_, vocab=vocab,
                                 v_begin=v_begin, T=T, kind=kind, loss_scale=loss_scale, want_dW=want_dW,
                                 accumulate_dW=accumulate_dW or i > 0, dW_s=dW_cur if i > 0 else dW_s,
                                 chunk_tokens=chunk_tokens, records_target=rec_target)

        def combine(ex, set_, n_rows, row0, m, *, with_loss, target):
            f["combine"](ex.x, set_, n_rows, row0, m, with_loss=with_loss, target=target)

        def wait(ex, target):
            f["wait"](ex.x, target)

        r = _p2p_step(exchange, spans, stats_p2p, backward_p2p, combine, wait, f["outputs"], mask=mask, kind=kind,
                      N=N, device=h_t.device)
        return _Result(r.loss, r.dh_s, r.dW_s if want_dW else None)

    nxt = stats(0) if spans else None
    for i, (a, b) in enumerate(spans):
        recs_out, work = nxt
        if i + 1 < len(spans):
            nxt = stats(i + 1)  # next chunk's pass 1 runs while this chunk's records travel
        work.wait()
        recs = _gathered(recs_out)
        m_c = None if mask is None else mask[a:b]
        acc = accumulate_dW or i > 0  # later chunks add into the first chunk's dW_s
        if fix:
            kj, state = partials_fn(h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, recs, m_c, vocab=vocab,
                                    v_begin=v_begin, T=T, kind=kind, beta=beta, loss_scale=loss_scale,
                                    want_dW=want_dW, accumulate_dW=acc, chunk_tokens=b - a)
            kj_out, kw = _all_gather_async(kj, group)
            kw.wait()
            r = finish_fn(state, h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, _gathered(kj_out), m_c, dW_s=dW_s)
        else:
            r = backward_fn(h_t[a:b], W_t_shard, h_s[a:b], W_s_shard, recs, m_c, vocab=vocab, v_begin=v_begin, T=T,
                            kind=kind, loss_scale=loss_scale, want_dW=want_dW, accumulate_dW=acc, dW_s=dW_s,
                            chunk_tokens=chunk_tokens)
        if loss is None:  # outputs in the kernels' dtype (fp32; the CPU test stand-ins return fp64)
            loss = torch.zeros(N, dtype=r.loss.dtype, device=r.loss.device)
            dh = torch.zeros(N, d_s, dtype=r.dh_s.dtype, device=r.dh_s.device)
        loss[a:b] = r.loss
        dh[a:b] = r.dh_s
        if want_dW:
            dW_s = r.dW_s
        if per_chunk:
            # partial dh (and FKL's partial loss: each shard's Σ over its rows) summed over the group under the
            # next chunk's kernels
            pending.append(_all_reduce_async(dh[a:b], group))
            if kind == "fkl":
                pending.append(_all_reduce_async(loss[a:b], group))
    for w in pending:
        w.wait()
    if dh is None:  # no tokens
        loss = torch.zeros(0, dtype=torch.float32, device=h_t.device)
        dh = torch.zeros(0, d_s, dtype=torch.float32, device=h_t.device)
    if not per_chunk:
        # FKL: each shard returns its partial loss (kdfused.h kd_vocab_backward), reduced like dh; the others are
        # already the full per-token loss on every rank
        loss = _reduce_scatter_rows(loss, group) if kind == "fkl" else _own_rows(loss, group)
        dh = _reduce_scatter_rows(dh, group)
    return _Result(loss, dh, dW_s if want_dW else None)


def token_sharded_dW_reduce(dW_s: torch.Tensor, group=None) -> torch.Tensor:
    """Token sharding with dW_s: the only exchange is the sum of the per-rank dW_s."""
    _all_reduce_sum(dW_s, group)
    return dW_s


def vocab_sharded_p2p_one_gpu(h_t, W_t, h_s, W_s, mask=None, *, exchanges, T=1.0, kind="fkl", beta=0.5,
                              loss_scale=1.0, want_dW=False, chunk_tokens=0, exchange_chunk=0):
    """One-GPU emulation of the P-rank p2p step (tests, ``bench.py --sim-p2p``): the P ranks' kernels run in one
    stream in an order where every counter a kernel waits on was raised by an EARLIER launch (per exchange chunk: all
    ranks' stats_p2p, then all ranks' backward_p2p — JSD/TVD: all partials_p2p, then all finish_p2p — then all owners'
    combine) — no kernel waits on one launched after it, so nothing depends on two launches running concurrently.
    The kernels, slot addressing, counters and set rotation are the multi-GPU ones; the 'peer' arenas are local
    allocations (``P2PExchange.local_group``).

    Returns per rank (loss, dh_s view, dW_s rows)."""
    from . import kdfused
    P = len(exchanges)
    V = W_t.shape[0]
    bounds = vocab_shard_bounds(V, P)
    N = h_t.shape[0]
    d_s = W_s.shape[1]
    fix = kind in ("jsd", "tvd")
    chunk = exchange_chunk if exchange_chunk > 0 else default_exchange_chunk(N, -(-V // P), kind, W_t.shape[1], d_s)
    spans = [(a, min(N, a + chunk)) for a in range(0, N, chunk)]
    base = exchanges[0].chunks
    dW = [None] * P
    loss_loc = [torch.zeros(N, dtype=torch.float32, device=h_t.device) for _ in range(P)] if kind != "fkl" else None
    for i, (a, b) in enumerate(spans):
        m_c = None if mask is None else mask[a:b]
        g = base + i
        for r, (v0, v1) in enumerate(bounds):  # every rank's record into every rank's arena
            kdfused.vocab_stats_p2p(h_t[a:b], W_t[v0:v1], h_s[a:b], W_s[v0:v1], m_c, x=exchanges[r].x,
                                    set=exchanges[r].set_of(g), vocab=V, v_begin=v0, T=T, kind=kind,
                                    chunk_tokens=(b - a) if fix else chunk_tokens)
        for r, (v0, v1) in enumerate(bounds):
            if i >= 3:
                kdfused.p2p_wait(exchanges[r].x, exchanges[r].done_target(g - 3))
        states = []
        if fix:
            for r, (v0, v1) in enumerate(bounds):
                ex = exchanges[r]
                states.append(kdfused.vocab_partials_p2p(h_t[a:b], W_t[v0:v1], h_s[a:b], W_s[v0:v1], m_c, x=ex.x,
                                                         set=ex.set_of(g), vocab=V, v_begin=v0, T=T, kind=kind,
                                                         beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                                                         accumulate_dW=i > 0, records_target=ex.records_target(g)))
        for r, (v0, v1) in enumerate(bounds):
            ex = exchanges[r]
            if fix:
                res = kdfused.vocab_finish_p2p(states[r], h_t[a:b], W_t[v0:v1], h_s[a:b], W_s[v0:v1], m_c, x=ex.x,
                                               set=ex.set_of(g), kj_target=ex.records_target(g), dW_s=dW[r])
            else:
                res = kdfused.vocab_backward_p2p(h_t[a:b], W_t[v0:v1], h_s[a:b], W_s[v0:v1], None, m_c, x=ex.x,
                                                 set=ex.set_of(g), vocab=V, v_begin=v0, T=T, kind=kind,
                                                 loss_scale=loss_scale, want_dW=want_dW, accumulate_dW=i > 0,
                                                 dW_s=dW[r], chunk_tokens=chunk_tokens,
                                                 records_target=ex.records_target(g))
            if want_dW:
                dW[r] = res.dW_s
            if kind != "fkl":
                loss_loc[r][a:b] = res.loss
        for r in range(P):
            ex = exchanges[r]
            kdfused.p2p_combine(ex.x, ex.set_of(g), b - a, a, m_c, with_loss=(kind == "fkl"),
                                target=ex.arrivals_target(g))
    out = []
    for r, ex in enumerate(exchanges):
        if spans:
            kdfused.p2p_wait(ex.x, ex.done_target(base + len(spans) - 1))
        ex.chunks = base + len(spans)
        dh, ls = kdfused.p2p_outputs(ex.x, h_t.device, N, d_s)
        out.append((loss_loc[r] if kind != "fkl" else ls, dh, dW[r]))
    return out
