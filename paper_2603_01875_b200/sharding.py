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
    if t.is_cuda and dist.get_backend(group) == "gloo":  # gloo has no CUDA reduce-scatter (one-GPU rank tests)
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


def _vocab_sharded_fix(h_t, W_t_shard, h_s, W_s_shard, mask, *, vocab, v_begin, group, T, kind, beta, loss_scale,
                       want_dW, accumulate_dW, dW_s, chunk_tokens, stats_fn, partials_fn, finish_fn, dh_reduce):
    """JSD/TVD: per token chunk, records all-gather -> partials -> (K, J) all-gather -> finish."""
    N = h_t.shape[0]
    d_s = W_s_shard.shape[1]
    # token chunk of the (K, J) exchange: a narrow vocab shard makes a 2048-token chunk's launches short (the dh GEMM
    # over K = V_r runs in 1-2 unbalanced waves; three prologues per chunk), so the chunk grows as the shard narrows,
    # keeping the chunk's G planes (12 B per (token, v)) near 5 GB, at least 4096 tokens: 8192 at P = 8, 5376 at
    # P = 2 (measured on one GPU simulating rank 0, c3 JSD: per-GPU efficiency at P = 8 0.67 with 2048-token chunks
    # -> 0.85 with 8192; at P = 2 0.79 with 2560 -> 0.84 with 4096; scripts/gpu/simv_jsd*.sh).
    # KD_VOCAB_FIX_CHUNK overrides.
    v_r = max(1, W_s_shard.shape[0])
    auto = max(4096, min(8192, int(5e9 / (12 * v_r)) // 256 * 256))
    chunk = chunk_tokens if chunk_tokens > 0 else int(os.environ.get("KD_VOCAB_FIX_CHUNK", str(auto)))
    loss = dh = None
    for a in range(0, N, chunk):
        b = min(N, a + chunk)
        ht_c, hs_c = h_t[a:b], h_s[a:b]
        m_c = None if mask is None else mask[a:b]
        rec = stats_fn(ht_c, W_t_shard, hs_c, W_s_shard, m_c, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                       chunk_tokens=b - a)
        recs = gather_records(rec, group)
        acc = accumulate_dW or a > 0  # later chunks add into the first chunk's dW_s
        kj, state = partials_fn(ht_c, W_t_shard, hs_c, W_s_shard, recs, m_c, vocab=vocab, v_begin=v_begin, T=T,
                                kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW, accumulate_dW=acc,
                                chunk_tokens=b - a)
        kj_all = gather_kj(kj, group)
        r = finish_fn(state, ht_c, W_t_shard, hs_c, W_s_shard, kj_all, m_c, dW_s=dW_s)
        if loss is None:  # outputs in the kernels' dtype (fp32; the CPU test stand-ins return fp64)
            loss = torch.zeros(N, dtype=r.loss.dtype, device=r.loss.device)
            dh = torch.zeros(N, d_s, dtype=r.dh_s.dtype, device=r.dh_s.device)
        loss[a:b] = r.loss
        dh[a:b] = r.dh_s
        if want_dW:
            dW_s = r.dW_s
    if dh is None:  # no tokens
        loss = torch.zeros(0, dtype=torch.float32, device=h_t.device)
        dh = torch.zeros(0, d_s, dtype=torch.float32, device=h_t.device)
    if dh_reduce == "scatter":
        return _Result(_own_rows(loss, group), _reduce_scatter_rows(dh, group), dW_s if want_dW else None)
    _all_reduce_sum(dh, group)
    return _Result(loss, dh, dW_s if want_dW else None)


def vocab_sharded_fwd_bwd(h_t, W_t_shard, h_s, W_s_shard, mask=None, *, vocab: int, v_begin: int, group=None,
                          T=1.0, kind="fkl", beta=0.5, loss_scale=1.0, want_dW=False, accumulate_dW=False,
                          dW_s=None, chunk_tokens=0, stats_fn: Callable | None = None,
                          backward_fn: Callable | None = None, partials_fn: Callable | None = None,
                          finish_fn: Callable | None = None, dh_reduce: str = "all"):
    """One vocab-sharded step on this rank; returns a KDResult whose dh_s is the full (all-reduced) gradient.

    dh_reduce="scatter": when the group's tokens are its members' equal slices concatenated in rank order (each rank
    contributes its own batch), every rank only needs dh_s / loss for its own slice: the dh exchange becomes a
    reduce-scatter (half the bytes of the all-reduce) and the result rows are this rank's slice.

    The kernel-side callables default to the CUDA entry points; tests substitute CPU stand-ins to
    exercise this exchange logic under gloo.
    """
    if kind in ("jsd", "tvd"):
        if stats_fn is None or partials_fn is None or finish_fn is None:
            from . import kdfused
            stats_fn = stats_fn or kdfused.vocab_stats
            partials_fn = partials_fn or kdfused.vocab_partials
            finish_fn = finish_fn or kdfused.vocab_finish
        return _vocab_sharded_fix(h_t, W_t_shard, h_s, W_s_shard, mask, vocab=vocab, v_begin=v_begin, group=group,
                                  T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                                  accumulate_dW=accumulate_dW, dW_s=dW_s, chunk_tokens=chunk_tokens,
                                  stats_fn=stats_fn, partials_fn=partials_fn, finish_fn=finish_fn,
                                  dh_reduce=dh_reduce)
    if stats_fn is None or backward_fn is None:
        from . import kdfused
        stats_fn = stats_fn or kdfused.vocab_stats
        backward_fn = backward_fn or kdfused.vocab_backward
    rec = stats_fn(h_t, W_t_shard, h_s, W_s_shard, mask, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                   chunk_tokens=chunk_tokens)
    recs = gather_records(rec, group)
    r = backward_fn(h_t, W_t_shard, h_s, W_s_shard, recs, mask, vocab=vocab, v_begin=v_begin, T=T, kind=kind,
                    loss_scale=loss_scale, want_dW=want_dW, accumulate_dW=accumulate_dW, dW_s=dW_s,
                    chunk_tokens=chunk_tokens)
    if dh_reduce not in ("all", "scatter"):
        raise ValueError(f"dh_reduce must be 'all' or 'scatter' (got {dh_reduce!r})")
    if dh_reduce == "scatter":
        # FKL: each shard returns its partial loss (kdfused.h kd_vocab_backward), reduced like dh; RKL: already full
        loss = _reduce_scatter_rows(r.loss, group) if kind == "fkl" else _own_rows(r.loss, group)
        return _Result(loss, _reduce_scatter_rows(r.dh_s, group), r.dW_s)
    _all_reduce_sum(r.dh_s, group)
    if kind == "fkl":  # FKL: each shard returns its partial loss (kdfused.h kd_vocab_backward)
        _all_reduce_sum(r.loss, group)
    return r


def token_sharded_dW_reduce(dW_s: torch.Tensor, group=None) -> torch.Tensor:
    """Token sharding with dW_s: the only exchange is the sum of the per-rank dW_s."""
    _all_reduce_sum(dW_s, group)
    return dW_s
