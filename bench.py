#!/usr/bin/env python
"""bench.py — KD tokens/s of the fused KD hot path (BASELINE.json metric) on N B200s.

One step = one pass of the whole hot path over one batch: recompute the teacher logits from H_t (V = 151936), the
student logits, the divergence, the per-token loss and dL/dh_s (BASELINE.json configs[1] by default: Qwen3-8B
d_t=4096 -> Qwen3-1.7B d_s=2048, 8 x 4096 tokens, FKL, T = 1).

    python bench.py [--gpus N --steps K --warmup W] [--config c2|c3_rkl|c3_jsd|c4|c5] [--dW]
    python bench.py --impl reference ...      # the fp64 CPU oracle on this box's host cores

N = 1: the step is one ``kd_fused_fwd_bwd`` call (the C ABI); the vocabulary-sharded driver is timed alongside with
P = 1 (identity exchanges), so the N > 1 headline's code path is exercised at every N.
N > 1 (torchrun): the headline is the north star's VOCABULARY SHARDING at fixed N (strong scaling): every rank holds
the same tokens and 1/P of both LM heads' rows (128-row granules); per exchange chunk the ranks all-gather the 20 B/token
records (and for JSD/TVD the 8 B/token (K, J) partials) and all-reduce the partial dh over NCCL, pipelined under the
next chunk's kernels (``sharding.vocab_sharded_fwd_bwd``).  Token sharding (each rank its own tokens, full heads, no
data-path collective, weak scaling) is measured in the same run and reported alongside (``--shard token`` swaps them).
Timing: W warm-up steps, then K steps with a CUDA event at every step boundary on the launching stream (barrier +
synchronize on both sides); ``ms_per_step`` is the median step (max over ranks), ``value`` = tokens of the job per
median step.  The library's per-launch event brackets (roofline) are recorded in a separate profiled pass, never
inside the headline timing.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import kd_inputs as KI  # noqa: E402

METRIC = "KD tokens/s (fwd+bwd, V=151936)"
UNIT = "tokens/s"
L2_BYTES = 126 * 2 ** 20
GUIDE_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kd", choices=["kd", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(KI.CONFIGS))
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per GPU (default: the config's)")
    ap.add_argument("--dW", action="store_true", help="also compute dL/dW_s")
    ap.add_argument("--grad-precision", default="split", choices=["split", "bf16"],
                    help="G fed to the backward GEMMs: split hi+lo bf16 (parity-grade, default) or one bf16 plane "
                         "(KD_GRAD_BF16, fast, not within the north-star gradient tolerance)")
    ap.add_argument("--shard", default="vocab", choices=["token", "vocab"],
                    help="layout of the headline value at N>1: vocab sharding (default, the north star: every rank "
                         "the same tokens and 1/P of the LM-head rows, strong scaling; records all-gather + partial "
                         "dh all-reduce over NCCL, pipelined) or token sharding (each rank its own tokens, full heads, "
                         "no data-path collective, weak scaling).  At N>1 the other layout is reported alongside.")
    ap.add_argument("--teacher-lse", action="store_true",
                    help="SURVEY §8(f) NEXT-2(i): the teacher ships its per-token LSE record with H_t (computed once by "
                         "kd_teacher_lse outside the timed region, as the teacher side would); the timed step is "
                         "kd_fused_fwd_bwd_lse, whose pass 1 sweeps the student head only (FKL/JSD/TVD)")
    ap.add_argument("--vocab-ranks", type=int, default=0,
                    help="vocab-sharded leg on a 2-D grid: ranks per vocab group (P_voc; default all ranks). "
                         "world / P_voc token groups (BASELINE config 4: 8x1, 4x2, 2x4, 1x8)")
    ap.add_argument("--sim-vocab-shards", type=int, default=0,
                    help="1 GPU: time rank 0's share of a P-way vocab-sharded strong-scaling step (all tokens, its "
                         "V/P head rows; compute only, identity exchanges) and report the projected efficiency")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 vocab-sharded step: the partial-dh exchange over NCCL (default) or the library's "
                         "peer-memory exchange (kd_vocab_backward_p2p: dh rows stored from the dh reduction straight "
                         "into the owners' slots over NVLink, owners' rank-order sums stored into every rank; CUDA IPC "
                         "arenas mapped once before the timing)")
    ap.add_argument("--sim-p2p", type=int, default=0,
                    help="1 GPU: run the P-rank peer-exchange step emulated on this GPU (every rank's kernels in one "
                         "stream, local arenas as the peers) and report its time and kernel split alongside")
    ap.add_argument("--topk", type=int, default=0,
                    help="SURVEY §8(f) NEXT-3 negative control: the prior-art top-k teacher transfer (k <= 32).  The "
                         "teacher's (idx, logit) top-k is produced once by kd_teacher_topk outside the timed region; "
                         "the timed step is kd_topk_fwd_bwd (student head only, FKL against the truncated teacher)")
    ap.add_argument("--stage", action="store_true",
                    help="staged variant (kd_problem.stage_logits, SURVEY §8(f) NEXT-2(ii)): pass 1 writes the token "
                         "chunk's fp32 logits, an HBM-bound kernel forms G from them (no second tensor sweep)")
    ap.add_argument("--no-variants", action="store_true", help="skip the staged-variant leg of the default run")
    ap.add_argument("--graph", action="store_true", help="also time the step captured into a CUDA graph")
    ap.add_argument("--handoff-peer", type=int, default=-1,
                    help="with --handoff: the teacher process owns H_t on this GPU (another device of the node: the "
                         "student maps it over NVLink; -1 = the student's own GPU)")
    ap.add_argument("--handoff", action="store_true",
                    help="add the hidden-state hand-off leg (SURVEY NEXT-4): teacher process -> student via CUDA IPC")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=256)
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(GUIDE_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


def workload_desc(cfg: KI.KDConfig, n_tok: int, want_dW: bool, world: int, grad_precision: str = "split",
                  teacher_lse: bool = False, topk: int = 0, stage: bool = False):
    mask_desc = {"none": "all ones", "prompt_pad": "prompt L_p~U[64,512] + padding beyond L~U[2048,4096] masked",
                 "ragged": "ragged L~U[256,8192], prompt L_p~U[32,min(512,L/2)] masked"}[cfg.mask]
    heads_b = cfg.vocab * (cfg.d_t + cfg.d_s) * 2
    return {
        "workload": f"{cfg.name}: d_t={cfg.d_t} -> d_s={cfg.d_s}, V={cfg.vocab}, {n_tok} tokens/GPU, "
                    f"{cfg.kind.upper()} T={cfg.temperature:g}" + (" +dW_s" if want_dW else "")
                    + (" [G: one bf16 plane]" if grad_precision == "bf16" else "")
                    + (" [teacher-shipped LSE record: pass 1 sweeps W_s only]" if teacher_lse else "")
                    + (f" [NEGATIVE CONTROL: top-{topk} teacher transfer, student head only]" if topk else "")
                    + (" [staged: pass 1 writes the token chunk's fp32 logits, G from them, no pass-2 sweep]"
                       if stage else ""),
        "baseline_config": cfg.notes,
        "tokens_per_gpu": n_tok, "d_t": cfg.d_t, "d_s": cfg.d_s, "vocab": cfg.vocab, "kind": cfg.kind,
        "temperature": cfg.temperature, "jsd_beta": cfg.jsd_beta if cfg.kind == "jsd" else None,
        "want_dW": want_dW, "mask": mask_desc, "grad_precision": grad_precision, "stage_logits": stage,
        "parallelism": f"token-sharded x{world} (no data-path collective)" if world > 1 else "1 GPU",
        "l2": f"no flush: resident inputs {heads_b / 1e9:.2f} GB heads + {n_tok * (cfg.d_t + cfg.d_s) * 2 / 1e9:.2f} GB "
              f"hidden > {L2_BYTES / 2 ** 20:.0f} MiB L2",
    }


# ------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(gpu_index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "power_w_median": statistics.median(power) if power else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------------- oracle timing
def oracle_tokens_per_s(cfg: KI.KDConfig, n_sample: int, want_dW: bool, seed: int = 0):
    """Time the fp64 CPU oracle (as it stands) on a bounded token sample at the full config shapes."""
    from oracle.kd_oracle import kd_fused_fwd_bwd
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000 + seed)
    H_t, H_s = KI.make_hidden(n_sample, W_t, W_s, seed=1001 + seed, head_seed=1000 + seed)
    Wt, Ws = KI.bf16_to_f64(W_t), KI.bf16_to_f64(W_s)
    ht, hs = KI.bf16_to_f64(H_t), KI.bf16_to_f64(H_s)
    del W_t, W_s
    t0 = time.perf_counter()
    kd_fused_fwd_bwd(ht, Wt, hs, Ws, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, want_dW=want_dW)
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    return n_sample / dt, dt, cores


def run_reference(args):
    """--impl reference: the oracle on the host cores, rank 0 only (other ranks exit 0 without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = KI.CONFIGS[args.config]
    n_sample = max(1, args.cpu_sample_tokens // 2)
    from oracle.kd_oracle import kd_fused_fwd_bwd
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
    Wt, Ws = KI.bf16_to_f64(W_t), KI.bf16_to_f64(W_s)
    times = []
    for step in range(args.warmup + args.steps):
        H_t, H_s = KI.make_hidden(n_sample, W_t, W_s, seed=1001 + step, head_seed=1000)
        ht, hs = KI.bf16_to_f64(H_t), KI.bf16_to_f64(H_s)
        t0 = time.perf_counter()
        kd_fused_fwd_bwd(ht, Wt, hs, Ws, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, want_dW=args.dW)
        if step >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n_sample * len(times) / total
    cores = len(os.sched_getaffinity(0))
    sample = (f"{n_sample} tokens per step at full {cfg.name} shapes (V={cfg.vocab}, d_t={cfg.d_t}, d_s={cfg.d_s}), "
              f"fp64 numpy, heads pre-converted to fp64 outside the timed call")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (kd_inputs recipe, seeded)",
            "config": workload_desc(cfg, n_sample, args.dW, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------- timing helpers
class Timer:
    """Per-step CUDA events on the launching stream; barrier + synchronize on both sides; max over ranks."""

    def __init__(self, world, dev, stream):
        self.world, self.dev, self.stream = world, dev, stream

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def run(self, step, steps, warmup, sampler_gpu=None):
        """-> dict(median_ms, mean_ms, total_ms (max over ranks), per_step_ms (this rank), clocks)."""
        import torch
        for _ in range(max(3, warmup)):
            step()
        torch.cuda.synchronize()
        sampler = ClockSampler(sampler_gpu) if sampler_gpu is not None else None
        if sampler is not None:
            time.sleep(0.3)
        self.barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record(self.stream)
        for i in range(steps):
            step()
            ev[i + 1].record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        clocks = sampler.stop() if sampler is not None else None
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
        return {"median_ms": self.max_over_ranks(statistics.median(per)),
                "mean_ms": self.max_over_ranks(sum(per) / len(per)),
                "total_ms": self.max_over_ranks(ev[0].elapsed_time(ev[-1])), "per_step_ms": per, "clocks": clocks}

    def profiled(self, kd, step, steps):
        """The same step with the library's per-launch event brackets on (kd_profile_*): per-kernel time and launch
        counts for the roofline.  Outside the headline timing."""
        import torch
        torch.cuda.synchronize()
        kd.profile_read()
        kd.profile_enable(True)
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
        kd.profile_enable(False)
        return kd.profile_read()


# ------------------------------------------------------------------------------------------- vocab-sharded leg
def vocab_layout(args, cfg, world, rank):
    """(P_voc, group index, position j, simulated?) of this rank's vocab group."""
    sim = world == 1 and args.sim_vocab_shards > 1  # one GPU playing rank 0 of a P-way vocab group (no exchange)
    pv = args.sim_vocab_shards if sim else (args.vocab_ranks if args.vocab_ranks > 0 else world)
    if not sim and world % pv:
        raise SystemExit(f"--vocab-ranks {pv} must divide the world size {world}")
    return pv, rank // pv, rank % pv, sim


def vocab_sharded_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, world, rank, dev, want_dW, timer, local, own_tokens,
                      sampler_gpu=None):
    """Vocabulary sharding (BASELINE.json north_star) through ``sharding.vocab_sharded_fwd_bwd``.

    own_tokens=False (the N>1 headline): every rank holds the SAME tokens (Ht/Hs/mask identical on all ranks) and
    LM-head rows [v0, v1) of a P_voc-way group; dh_s is all-reduced per exchange chunk (strong scaling at fixed N; the
    job's tokens are counted once).  own_tokens=True (2-D grid, config 4: P_tok x P_voc): the group's tokens are its
    members' own slices all-gathered once outside the timing; each rank keeps dh_s of its own slice (reduce-scatter),
    weak over token groups.  With --sim-vocab-shards P on one GPU, rank 0's work of a P-way strong-scaling group."""
    import torch
    import torch.distributed as dist

    from paper_2603_01875_b200 import sharding

    pv, gi, j, sim = vocab_layout(args, cfg, world, rank)
    group = None
    if world > 1 and pv < world:
        for t in range(world // pv):  # every rank creates every group, in the same order
            g = dist.new_group(list(range(t * pv, (t + 1) * pv)))
            if t == gi:
                group = g
    bounds = sharding.vocab_shard_bounds(cfg.vocab, pv)
    v0, v1 = bounds[j]
    Wt_sh, Ws_sh = Wt[v0:v1].contiguous(), Ws[v0:v1].contiguous()
    if own_tokens and pv > 1 and not sim:
        def gather(x):
            parts = [torch.empty_like(x) for _ in range(pv)]
            dist.all_gather(parts, x.contiguous(), group=group)
            return torch.cat(parts)
        Ht_all, Hs_all = gather(Ht), gather(Hs)
        mask_all = gather(mask) if mask is not None else None
    else:
        Ht_all, Hs_all, mask_all = Ht, Hs, mask
    n_all = Ht_all.shape[0]
    n_eff_all = int(mask_all.sum().item()) if mask_all is not None else n_all
    n_groups = 1 if sim else max(1, world // pv)
    n_eff_job = n_eff_all * (n_groups if own_tokens else 1)
    dW = torch.empty(v1 - v0, cfg.d_s, dtype=torch.float32, device=dev) if want_dW else None
    kw = dict(vocab=cfg.vocab, v_begin=v0, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, loss_scale=1.0,
              want_dW=want_dW, accumulate_dW=False, group=group, dh_reduce="scatter" if own_tokens else "all")
    p2p = args.exchange == "p2p" and world > 1 and not sim and not own_tokens
    if p2p:  # arenas allocated and peer-mapped once (CUDA IPC), outside the timing
        chunk_p2p = sharding.default_exchange_chunk(n_all, v1 - v0, cfg.kind, cfg.d_t, cfg.d_s)
        kw["exchange"] = sharding.P2PExchange.create(group, cfg.d_s, max_rows=chunk_p2p, max_tokens=n_all, device=dev)
    res = {}

    def step():
        res["r"] = sharding.vocab_sharded_fwd_bwd(Ht_all, Wt_sh, Hs_all, Ws_sh, mask_all, dW_s=dW, **kw)

    t = timer.run(step, args.steps, args.warmup, sampler_gpu=sampler_gpu)
    prof = timer.profiled(kd, step, args.steps)
    ms = t["median_ms"]
    r = res["r"]
    chunk = sharding.default_exchange_chunk(n_all, v1 - v0, cfg.kind, cfg.d_t, cfg.d_s)
    rec_bytes = 20 * n_all * pv
    kj_bytes = 8 * n_all * pv if cfg.kind in ("jsd", "tvd") else 0
    dh_bytes = 4 * n_all * cfg.d_s
    grid = f"{n_groups} token group(s) x {pv} vocab shards" + (" (SIMULATED on one GPU)" if sim else "")
    out = {"value": n_eff_job / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "ms_per_step_mean": t["mean_ms"],
           "scaling": "weak" if own_tokens else "strong", "tokens_per_step": n_all * (n_groups if own_tokens else 1),
           "vocab_rows_per_gpu": v1 - v0, "grid": grid, "exchange_chunk_tokens": chunk,
           "layout": (f"vocab-sharded ({grid}): LM-head rows split in 128-row granules over each group of {pv} ranks; "
                      + ("each group all-gathers its members' token slices once, each rank keeps dh of its own"
                         if own_tokens else f"every rank holds the same {n_all} tokens, dh_s all-reduced")),
           "exchange_bytes_per_step_per_rank": {
               "records_allgather": rec_bytes, "kj_allgather": kj_bytes,
               ("dh_reduce_scatter" if own_tokens else "dh_allreduce_payload"): dh_bytes},
           "pipeline": ("per exchange chunk: pass 1 of chunk c+1 under the records all-gather of chunk c; the partial "
                        "dh rows stored by the dh reduction into their owners' slots (NVLink peer memory), the owners' "
                        "rank-order sums of chunk c stored into every rank after chunk c+1's kernels (kd_p2p)"
                        if p2p else
                        "per exchange chunk: pass 1 of chunk c+1 under the records all-gather of chunk c; the partial-dh "
                        "all-reduce of chunk c under chunk c+1's kernels (NCCL stream); only the last chunk's is exposed"),
           "dh_exchange": "p2p (library kernels over peer memory)" if p2p else "nccl",
           "loss_finite": bool(torch.isfinite(r.loss).all().item()),
           "kernels_ms_per_step": {k: v / args.steps for k, (n, v) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
           "gpu_launches_per_step": sum(n for n, _ in prof.values()) / args.steps, "_prof": prof,
           "_n_eff_rank": n_eff_all, "clocks": t["clocks"]}
    if sim:
        out["simulated"] = (f"one GPU runs rank 0's work of a {pv}-way vocab group (its {v1 - v0} head rows x all "
                            f"{n_all} tokens) with identity exchanges: the compute of one rank at P={pv}, no "
                            f"communication.  value = the job's tokens / this time, i.e. the P-GPU strong-scaling "
                            f"throughput excluding the exchanges")
    return out


def p2p_one_gpu_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, timer, want_dW, P=None, steps=None):
    """--sim-p2p P: the P-rank peer-exchange step emulated on one GPU (sharding.vocab_sharded_p2p_one_gpu): every
    rank's kernels in one stream, the peers' arenas local.  The time is the whole job's compute serialised on one GPU
    (so tokens/s ~ the single-GPU headline) plus the exchange kernels; their cost per rank is in the kernel split
    ("p2p": owner sums + counters; the peer stores ride inside reduce_dh).  Local HBM stands in for NVLink."""
    from paper_2603_01875_b200 import sharding
    P = P or args.sim_p2p
    steps = steps or args.steps
    n = Ht.shape[0]
    chunk = sharding.default_exchange_chunk(n, -(-cfg.vocab // P), cfg.kind, cfg.d_t, cfg.d_s)
    exs = sharding.P2PExchange.local_group(P, cfg.d_s, max_rows=chunk, max_tokens=n, device=Ht.device)
    res = {}

    def step():
        res["r"] = sharding.vocab_sharded_p2p_one_gpu(Ht, Wt, Hs, Ws, mask, exchanges=exs, T=cfg.temperature,
                                                     kind=cfg.kind, beta=cfg.jsd_beta, want_dW=want_dW,
                                                     exchange_chunk=chunk)

    t = timer.run(step, steps, args.warmup)
    prof = timer.profiled(kd, step, steps)
    n_eff = int(mask.sum().item()) if mask is not None else n
    import torch
    same = all(torch.equal(res["r"][0][1], o[1]) for o in res["r"][1:])
    del exs
    torch.cuda.empty_cache()
    return {"ranks_emulated": P, "value": n_eff / (t["median_ms"] / 1e3), "unit": UNIT, "ms_per_step": t["median_ms"],
            "exchange_chunk_tokens": chunk, "all_ranks_same_dh": bool(same),
            "steps": steps,
            "kernels_ms_per_step": {k: v / steps for k, (c, v) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "note": "one GPU runs all P ranks' kernels (no concurrency needed: every counter a kernel waits on was "
                    "raised by an earlier launch); the 'peer' stores go to local HBM, not NVLink"}


# ------------------------------------------------------------------------------------------- hand-off leg
def _handoff_teacher(conn, h_bits, vocab, device):
    """Teacher PROCESS of the hand-off leg: owns H_t (the batch's bit pattern) and, for comparison, a buffer the size
    of the full bf16 logits it would otherwise ship; exports both (kd_handoff_export) and waits."""
    import torch

    import paper_2603_01875_b200 as kd
    torch.cuda.set_device(device)
    ht = torch.from_numpy(h_bits.view(np.int16)).to(f"cuda:{device}").view(torch.bfloat16)
    logits = torch.zeros(h_bits.shape[0], vocab, dtype=torch.bfloat16, device=f"cuda:{device}")
    torch.cuda.synchronize()
    conn.send((kd.handoff_export(ht), tuple(ht.shape), kd.handoff_export(logits), tuple(logits.shape)))
    conn.recv()


def handoff_leg(args, cfg, kd, H_t_bits, Ht_local, Wt, Hs, Ws, mask, kw, out, dW, n_eff, stream, local):
    """KDFlow's hidden-state transfer between a teacher process and this (student)
    process through kd_handoff_* (CUDA IPC).  Measures (a) the pull of H_t into the student's buffer, (b) the pull of
    the full bf16 logits the hidden-state design avoids shipping (the ~37x volume of P:133), (c) the KD step reading
    the teacher's H_t in place (zero copy).  Same GPU here (gpurun gives one): the pulls are device-to-device copies
    through the exporter's mapping; on a multi-GPU node the same handle maps a peer GPU's memory over NVLink."""
    import multiprocessing as mp

    import torch
    ctx = mp.get_context("spawn")
    parent, child = ctx.Pipe()
    import torch as _t
    peer = args.handoff_peer if args.handoff_peer >= 0 else local
    if peer >= _t.cuda.device_count():
        return {"skipped": f"--handoff-peer {peer}: this box has {_t.cuda.device_count()} GPU(s)"}
    proc = ctx.Process(target=_handoff_teacher, args=(child, H_t_bits, cfg.vocab, peer))
    proc.start()
    try:
        h_ht, s_ht, h_lg, s_lg = parent.recv()
        # the mapped buffers live on the teacher's GPU (the peer's memory, reached over NVLink, when peer != local)
        m_ht = kd.HandoffTensor(h_ht, s_ht, torch.bfloat16, device=peer)
        m_lg = kd.HandoffTensor(h_lg, s_lg, torch.bfloat16, device=peer)
        assert torch.equal(m_ht.tensor.to(Ht_local.device), Ht_local)
        dst_ht = torch.empty_like(Ht_local)
        dst_lg = torch.empty(s_lg, dtype=torch.bfloat16, device=Ht_local.device)

        def timed(fn, reps):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        t_ht = timed(lambda: dst_ht.copy_(m_ht.tensor), 20)
        t_lg = timed(lambda: dst_lg.copy_(m_lg.tensor), 5)
        t_step = timed(lambda: kd.fused_fwd_bwd(m_ht.tensor, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw), args.steps)
        b_ht, b_lg = m_ht.nbytes, m_lg.nbytes
        del dst_lg
        m_ht.close()
        m_lg.close()
    finally:
        parent.send("done")
        proc.join(timeout=120)
    where = ("the same B200 — pulls are D2D copies through the exporter's mapping (read + write of the bytes)"
             if peer == local else f"GPU {peer} (teacher) and GPU {local} (student) — pulls are peer copies over "
             f"NVLink, the zero-copy step's TMA loads read the peer's H_t over NVLink")
    return {"transport": "kd_handoff_export/open (CUDA IPC); teacher and student are separate processes on " + where,
            "teacher_gpu": peer, "student_gpu": local,
            "h_t_bytes_per_step": b_ht, "full_logits_bytes_per_step": b_lg, "volume_ratio": b_lg / b_ht,
            "pull_h_t_ms": t_ht, "pull_logits_ms": t_lg, "time_ratio": t_lg / t_ht,
            "pull_h_t_GBps": b_ht / (t_ht / 1e3) / 1e9, "pull_logits_GBps": b_lg / (t_lg / 1e3) / 1e9,
            "zero_copy_step": {"value": n_eff / (t_step / 1e3), "unit": UNIT, "ms_per_step": t_step,
                               "what": "kd_fused_fwd_bwd reading the teacher process's H_t in place"}}


# ------------------------------------------------------------------------------------------- roofline
def roofline_of(prof, steps, pk, cfg, n_eff, v_rows, teacher_lse=False, topk=0, grad_precision="split"):
    """Dominant tensor kernel of the step from the profiled pass: algorithmic flop per launch (SURVEY §8(d):
    2·tokens·V_r·(d_t+d_s) for a fused pass, 2·tokens·V_r·d_s for a backward GEMM) over its mean launch time."""
    flops_pass = 2.0 * n_eff * v_rows * (cfg.d_t + cfg.d_s)  # per step: both LM-head GEMMs, one vocab sweep
    flops_g = 2.0 * n_eff * v_rows * cfg.d_s                   # G · W_s  (or Gᵀ · H_s)
    algo = {"pass1": 2.0 * n_eff * v_rows * cfg.d_s if (teacher_lse or topk) else flops_pass,
            "pass2": 2.0 * n_eff * v_rows * cfg.d_s if topk else flops_pass, "gemm_dh": flops_g, "gemm_dW": flops_g}
    gm = 2.0 if grad_precision == "split" else 1.0
    exec_mult = {"pass1": 1.0, "pass2": 1.0, "gemm_dh": gm, "gemm_dW": gm}
    kernels = {}
    total_ms = sum(t for _, t in prof.values()) or 1.0
    for name, (n, t) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        e = {"launches": n, "ms_per_step": t / steps, "share": t / total_ms}
        if name in algo:
            e["algorithmic_tflops"] = algo[name] * steps / (t / 1e3) / 1e12
            e["tensor_pipe_tflops_executed"] = e["algorithmic_tflops"] * exec_mult[name]
        if name == "stage_grad":
            # HBM-bound: per (token, v) 8 B of staged logits read + G written (split: 4 B, bf16: 2 B, JSD/TVD: 8 B)
            wb = 8 if cfg.kind in ("jsd", "tvd") else (4 if grad_precision == "split" else 2)
            e["algorithmic_bytes_per_launch"] = n_eff * v_rows * (8 + wb) * steps / n
            e["achieved_GBps"] = e["algorithmic_bytes_per_launch"] / (t / n / 1e3) / 1e9
            e["hbm_frac"] = e["achieved_GBps"] / pk["hbm_gbs"]
        kernels[name] = e
    dom = max((k for k in kernels if k in algo), key=lambda k: kernels[k]["ms_per_step"])
    peak_sust = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        cap = json.load(open(tpath)).get(dom, {})
        # the capture is one launch of a given workload (c2 shapes, all V rows, FKL, the default variant); another
        # workload's launch moves other bytes, so it gets no traffic figure
        same = (cfg.name == cap.get("config", "c2") and v_rows == cfg.vocab and not teacher_lse and not topk
                and grad_precision == "split")
        traffic = cap.get("dram_bytes_per_launch") if same else None
    n_l, t_l = prof[dom]
    achieved = algo[dom] * steps / n_l / (t_l / n_l / 1e3) / 1e12
    what = ("2*tokens*V_r*d_s flop" if (dom == "pass1" and teacher_lse) or (topk and dom.startswith("pass")) else
            "2*tokens*V_r*(d_t+d_s) flop" if dom.startswith("pass") else "2*tokens*V_r*d_s flop")
    roofline = {"bound": "tensor", "kernel": f"kd_pass_kernel ({dom})" if dom.startswith("pass") else dom,
                "achieved": achieved, "peak": peak_sust, "unit": "TFLOP/s", "frac": achieved / peak_sust,
                "traffic": traffic,
                "peak_note": f"bf16 dense, {pk['source']}, sustained (kernel timed inside a long step); "
                             f"burst {pk['bf16_tflops']}",
                "algorithmic_per_launch": f"{what} = {algo[dom] * steps / n_l:.4g}",
                "timing": "live CUDA events around each launch on its stream (kd_profile_*), in a profiled pass of "
                          "the same step run after the headline timing"}
    return roofline, kernels, peak_sust


# ------------------------------------------------------------------------------------------- e2e leg
def e2e_leg(args, timer, dev, stream, hosts, compute, n_tokens_job, n_out_rows, d_s):
    """Same metric through the public API with host buffers: every step uploads its inputs from pinned host memory
    (H2D) and reads its loss / dh_s back (D2H) inside the timed region.  Copies run on a side stream,
    double-buffered, so step i+1's upload and step i-1's download overlap step i's kernels (the pattern a training
    loop would use).  ``hosts``: pinned host tensors uploaded every step; ``compute(dev_inputs) -> (loss, dh)``."""
    import torch
    hloss = [torch.empty(n_out_rows, dtype=torch.float32).pin_memory() for _ in range(2)]
    hdh = [torch.empty(n_out_rows, d_s, dtype=torch.float32).pin_memory() for _ in range(2)]
    dbuf = [[torch.empty(h.shape, dtype=h.dtype, device=dev) for h in hosts] for _ in range(2)]
    outs = [None, None]
    cs = torch.cuda.Stream(device=dev)
    in_ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]

    def upload(b):
        with torch.cuda.stream(cs):
            for d, h in zip(dbuf[b], hosts):
                d.copy_(h, non_blocking=True)
            in_ready[b].record(cs)

    def run_pipeline(n):
        upload(0)
        for i in range(n):
            b = i & 1
            if i + 1 < n:
                if i >= 1:
                    cs.wait_event(done[b ^ 1])  # buffer b^1 was read by step i-1
                upload(b ^ 1)
            stream.wait_event(in_ready[b])
            outs[b] = compute(dbuf[b])
            done[b].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(done[b])
                hloss[b].copy_(outs[b][0], non_blocking=True)
                hdh[b].copy_(outs[b][1], non_blocking=True)

    run_pipeline(2)
    torch.cuda.synchronize()
    timer.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(cs)
    stream.wait_event(t0)
    run_pipeline(args.steps)
    t1.record(cs)
    torch.cuda.synchronize()
    ms = timer.max_over_ranks(t0.elapsed_time(t1))
    last = (args.steps - 1) & 1
    assert torch.equal(hloss[last], outs[last][0].cpu())
    h2d = sum(h.numel() * h.element_size() for h in hosts)
    d2h = n_out_rows * 4 + n_out_rows * d_s * 4
    return {"value": n_tokens_job * args.steps / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / args.steps}


# ------------------------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2603_01875_b200 as kd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())  # >1 rank per GPU only in the gloo test of the vocab leg
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("KD_DIST_BACKEND", "nccl")  # gloo: 2 ranks on one GPU (tests of the exchange)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    kd.lib()
    cfg = KI.CONFIGS[args.config]
    want_dW = args.dW or cfg.want_dW
    n_tok = args.tokens or cfg.n_tokens
    vocab_head = world > 1 and args.shard == "vocab"
    grid2d = 0 < args.vocab_ranks < world

    # ---- inputs: heads replicated (seed 1000); token sharding: each rank its own tokens (seed 1001 + rank); the
    # vocab-sharded headline: every rank the same tokens (seed 1001, rank 0's own)
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)

    def tokens(seed_off):
        H_t, H_s = KI.make_hidden(n_tok, W_t, W_s, seed=1001 + seed_off, head_seed=1000)
        m = KI.make_mask(KI.KDConfig(**{**cfg.__dict__, "n_seq": max(1, n_tok // cfg.seq_len)}),
                         seed=1002 + seed_off) if cfg.mask != "none" else None
        return H_t, H_s, (np.resize(m, n_tok) if m is not None else None)

    def up(b):
        return torch.from_numpy(b.view(np.int16)).to(dev).view(torch.bfloat16)

    H_t, H_s, mask_np = tokens(rank)
    Wt, Ws, Ht, Hs = up(W_t), up(W_s), up(H_t), up(H_s)
    mask = torch.from_numpy(mask_np).to(dev) if mask_np is not None else None
    n_eff = int(mask_np.sum()) if mask_np is not None else n_tok
    if vocab_head and not grid2d:
        if rank == 0:
            Ht_sh, Hs_sh, mask_sh, n_eff_sh = Ht, Hs, mask, n_eff
        else:
            H_t0, H_s0, m0 = tokens(0)
            Ht_sh, Hs_sh = up(H_t0), up(H_s0)
            mask_sh = torch.from_numpy(m0).to(dev) if m0 is not None else None
            n_eff_sh = int(m0.sum()) if m0 is not None else n_tok
    del W_t, W_s
    kw = dict(T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, loss_scale=1.0, want_dW=want_dW,
              accumulate_dW=False, grad_precision=args.grad_precision)
    if args.stage:
        if args.topk or args.teacher_lse:
            raise SystemExit("--stage combines with neither --topk nor --teacher-lse (kdfused.h stage_logits)")
        kw["stage_logits"] = True
    out = kd.KDResult(torch.empty(n_tok, dtype=torch.float32, device=dev),
                      torch.empty(n_tok, cfg.d_s, dtype=torch.float32, device=dev), None,
                      torch.zeros(1, dtype=torch.int64, device=dev))
    dW = torch.empty(cfg.vocab, cfg.d_s, dtype=torch.float32, device=dev) if want_dW else None
    stream = torch.cuda.current_stream()
    timer = Timer(world, dev, stream)
    pk = peaks()

    lse_t = tk = None
    if args.topk:
        if cfg.kind != "fkl":
            raise SystemExit("--topk is forward KL only (kd_topk_fwd_bwd)")
        tk = kd.teacher_topk(Ht, Wt, mask, k=args.topk, d_s=cfg.d_s, T=cfg.temperature)
    if args.teacher_lse:
        # the teacher side's record, produced once per batch by the teacher (not student work: outside the timing)
        lse_t = kd.teacher_lse(Ht, Wt, mask, d_s=cfg.d_s, T=cfg.temperature, kind=cfg.kind)

    def fused_step():
        if tk is not None:
            return kd.topk_fwd_bwd(Hs, Ws, tk[0], tk[1], mask, d_t=cfg.d_t, T=cfg.temperature, loss_scale=1.0,
                                   want_dW=want_dW, dW_s=dW, grad_precision=args.grad_precision, out=out)
        if lse_t is not None:
            return kd.fused_fwd_bwd_lse(Ht, Wt, Hs, Ws, lse_t, mask, dW_s=dW, out=out, **kw)
        return kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw)

    alongside = {}
    # ---- the token-sharded / single-GPU step (the headline at N = 1 or with --shard token)
    t_tok = timer.run(fused_step, args.steps, args.warmup, sampler_gpu=None if vocab_head else local)
    prof_tok = timer.profiled(kd, fused_step, args.steps)
    tok_value = world * n_eff / (t_tok["median_ms"] / 1e3)
    nonfinite = int(out.n_nonfinite.item())
    if vocab_head:
        vleg = vocab_sharded_leg(args, cfg, kd, Wt, Ws, Ht if grid2d else Ht_sh, Hs if grid2d else Hs_sh,
                                 mask if grid2d else mask_sh, world, rank, dev, want_dW, timer, local,
                                 own_tokens=grid2d, sampler_gpu=local)
        prof = vleg.pop("_prof")
        n_eff_rank = vleg.pop("_n_eff_rank")  # tokens this rank sweeps its vocab rows for
        clocks = vleg.pop("clocks")
        value, ms_med = vleg["value"], vleg["ms_per_step"]
        v_rows = vleg["vocab_rows_per_gpu"]
        alongside["token_sharded"] = {"value": tok_value, "unit": UNIT, "ms_per_step": t_tok["median_ms"],
                                      "scaling": "weak", "tokens_per_step": n_tok * world,
                                      "layout": f"token-sharded x{world}, full heads per rank, no data-path collective"}
        scaling = vleg["scaling"]
    else:
        prof, value, ms_med, clocks = prof_tok, tok_value, t_tok["median_ms"], t_tok["clocks"]
        v_rows, n_eff_rank, scaling = cfg.vocab, n_eff, "weak"
    launches_per_step = sum(n for n, _ in prof.values()) / args.steps
    roofline, kernels, peak_sust = roofline_of(prof, args.steps, pk, cfg, n_eff_rank, v_rows, args.teacher_lse,
                                               args.topk, args.grad_precision)
    step_useful = 2.0 * cfg.vocab * ((0 if args.topk else cfg.d_t) + 2 * cfg.d_s + (cfg.d_s if want_dW else 0))
    tokens_job_per_s = value
    useful_frac = step_useful * tokens_job_per_s / 1e12 / (peak_sust * world)

    # ---- e2e: the same metric through the public API with host buffers, H2D of the inputs and D2H of loss / dh_s
    # every step inside the timed region
    e2e = None
    if not args.no_e2e:
        if vocab_head and not grid2d:
            from paper_2603_01875_b200 import sharding
            pv, _, j, _ = vocab_layout(args, cfg, world, rank)
            v0, v1 = sharding.vocab_shard_bounds(cfg.vocab, pv)[j]
            Wt_sh, Ws_sh = Wt[v0:v1].contiguous(), Ws[v0:v1].contiguous()
            dWv = torch.empty(v1 - v0, cfg.d_s, dtype=torch.float32, device=dev) if want_dW else None
            hosts = [Ht_sh.cpu().pin_memory(), Hs_sh.cpu().pin_memory()] + \
                ([mask_sh.cpu().pin_memory()] if mask_sh is not None else [])

            def compute(d):
                r = sharding.vocab_sharded_fwd_bwd(d[0], Wt_sh, d[1], Ws_sh, d[2] if len(d) > 2 else None,
                                                   vocab=cfg.vocab, v_begin=v0, T=cfg.temperature, kind=cfg.kind,
                                                   beta=cfg.jsd_beta, want_dW=want_dW, dW_s=dWv)
                return r.loss, r.dh_s
            e2e = e2e_leg(args, timer, dev, stream, hosts, compute, n_eff_sh, n_tok, cfg.d_s)
            e2e["note"] = ("vocab-sharded step through sharding.vocab_sharded_fwd_bwd (the library's kd_vocab_* entry "
                           "points + NCCL): every rank uploads the batch's H_t/H_s (+mask) and reads back the full "
                           "loss / all-reduced dh_s; heads resident (each rank its rows)")
        elif not grid2d:
            outs = [kd.KDResult(torch.empty(n_tok, dtype=torch.float32, device=dev),
                                torch.empty(n_tok, cfg.d_s, dtype=torch.float32, device=dev), None,
                                torch.zeros(1, dtype=torch.int64, device=dev)) for _ in range(2)]
            flip = [0]
            if tk is not None:  # the top-k student never sees H_t: the teacher ships (idx, logit) pairs instead
                hosts = [Hs.cpu().pin_memory(), tk[0].cpu().pin_memory(), tk[1].cpu().pin_memory()]
            elif lse_t is not None:
                hosts = [Ht.cpu().pin_memory(), Hs.cpu().pin_memory(), lse_t.cpu().pin_memory()]
            else:
                hosts = [Ht.cpu().pin_memory(), Hs.cpu().pin_memory()]
            if mask is not None:
                hosts.append(mask.cpu().pin_memory())

            def compute(d):
                o = outs[flip[0]]
                flip[0] ^= 1
                m = d[-1] if mask is not None else None
                if tk is not None:
                    kd.topk_fwd_bwd(d[0], Ws, d[1], d[2], m, d_t=cfg.d_t, T=cfg.temperature, loss_scale=1.0,
                                    want_dW=want_dW, dW_s=dW, grad_precision=args.grad_precision, out=o)
                elif lse_t is not None:
                    kd.fused_fwd_bwd_lse(d[0], Wt, d[1], Ws, d[2], m, dW_s=dW, out=o, **kw)
                else:
                    kd.fused_fwd_bwd(d[0], Wt, d[1], Ws, m, dW_s=dW, out=o, **kw)
                return o.loss, o.dh_s
            e2e = e2e_leg(args, timer, dev, stream, hosts, compute, world * n_eff, n_tok, cfg.d_s)
            e2e["note"] = ("heads resident in HBM (weights); per step: " +
                           ("H_s + the teacher's top-k (idx, logit) pairs" if tk is not None else
                            "H_t/H_s + the teacher's LSE record" if lse_t is not None else "H_t/H_s") +
                           " (+mask) pinned-host->device and loss/dh_s device->pinned-host, on a copy stream "
                           "overlapped with the neighbouring steps")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle as it stands on a bounded sample at the full config shapes, all affinity cores
        v, dt, cores = oracle_tokens_per_s(cfg, args.cpu_sample_tokens, want_dW)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_sample_tokens} tokens at full {cfg.name} shapes, the headline workload"
                         f"{' (+dW_s)' if want_dW else ''}, fp64 numpy ({dt:.1f} s; BLAS threads = all {cores} "
                         f"affinity cores)"}
        if not want_dW:  # the same token subset including dW_s for that subset
            v2, dt2, _ = oracle_tokens_per_s(cfg, args.cpu_sample_tokens, True)
            cpu["with_dW"] = {"value": v2, "unit": UNIT, "cores": cores,
                              "sample": f"{args.cpu_sample_tokens} tokens at full {cfg.name} shapes + dW_s "
                                        f"({dt2:.1f} s)"}
        # configs[0] (the tiny check) timed whole, all cores
        tiny = KI.CONFIGS["tiny"]
        from oracle.kd_oracle import kd_fused_fwd_bwd as _oracle
        ti = KI.make_config_inputs(tiny)
        t0 = time.perf_counter()
        _oracle(KI.bf16_to_f64(ti.H_t), KI.bf16_to_f64(ti.W_t), KI.bf16_to_f64(ti.H_s), KI.bf16_to_f64(ti.W_s),
                T=tiny.temperature, kind=tiny.kind, want_dW=True)
        dt_t = time.perf_counter() - t0
        cpu["tiny_config_whole"] = {"value": tiny.n_tokens / dt_t, "unit": UNIT, "seconds": dt_t,
                                    "sample": f"configs[0] whole: {tiny.n_tokens} tokens, d={tiny.d_t}, V={tiny.vocab}, +dW"}
        try:  # the oracle on a single thread as well
            from threadpoolctl import threadpool_limits
            n1 = max(1, args.cpu_sample_tokens // 8)
            with threadpool_limits(limits=1):
                v1, dt1, _ = oracle_tokens_per_s(cfg, n1, want_dW)
            cpu["single_thread"] = {"value": v1, "unit": UNIT, "cores": 1,
                                    "sample": f"{n1} tokens at full {cfg.name} shapes ({dt1:.1f} s)"}
        except ImportError:
            pass

    if args.graph and not vocab_head:
        # the same step captured once into a CUDA graph and replayed (no per-launch host work; the library's calls
        # are capturable: no host syncs, no allocation, every launch on the caller's stream)
        cs_ = torch.cuda.Stream(device=dev)
        cs_.wait_stream(stream)
        with torch.cuda.stream(cs_):
            fused_step()
        stream.wait_stream(cs_)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            fused_step()
        tg = timer.run(graph.replay, args.steps, args.warmup)
        alongside["cuda_graph"] = {"value": world * n_eff / (tg["median_ms"] / 1e3), "unit": UNIT,
                                   "ms_per_step": tg["median_ms"],
                                   "what": "one step captured into a CUDA graph, replayed K times (same inputs)"}

    # ---- the staged variant (kd_problem.stage_logits) on the same inputs, timed the same way
    if not (args.stage or args.topk or args.teacher_lse or args.no_variants or vocab_head):
        kw_st = dict(kw, stage_logits=True)

        def staged():
            kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw_st)
        ts = timer.run(staged, args.steps, args.warmup)
        sprof = timer.profiled(kd, staged, args.steps)
        ms_st = ts["median_ms"]
        stot = sum(t for _, t in sprof.values()) or 1.0
        alongside["staged_variant"] = {
            "value": world * n_eff / (ms_st / 1e3), "unit": UNIT, "ms_per_step": ms_st,
            "what": "kd_problem.stage_logits=1 (SURVEY NEXT-2(ii)): pass 1 also writes the token chunk's fp32 logits "
                    "(2 x Nc x V x 4 B, one chunk at a time), an HBM-bound kernel forms G from them; no pass-2 sweep. "
                    "Same outputs within the same tolerances (tests/test_gpu_stage.py); same launch config otherwise",
            "useful_flop_frac": step_useful * world * n_eff / (ms_st / 1e3) / 1e12 / (peak_sust * world),
            "kernels": {k: {"launches": n, "ms_per_step": t / args.steps, "share": t / stot}
                        for k, (n, t) in sorted(sprof.items(), key=lambda kv: -kv[1][1])}}
        if "stage_grad" in sprof:
            n_l, t_l = sprof["stage_grad"]
            wb = 8 if cfg.kind in ("jsd", "tvd") else (4 if args.grad_precision == "split" else 2)
            b = n_eff * cfg.vocab * (8 + wb) * args.steps / n_l  # per launch (one token chunk)
            alongside["staged_variant"]["stage_grad_roofline"] = {
                "bound": "hbm", "achieved": b / (t_l / n_l / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": b / (t_l / n_l / 1e3) / 1e9 / pk["hbm_gbs"],
                "algorithmic_per_launch": f"tokens*V*(8 + {wb}) B = {b:.4g}"}

    if args.sim_p2p > 1 and world == 1:
        alongside["p2p_one_gpu"] = p2p_one_gpu_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, timer, want_dW)
    elif world == 1 and not args.no_variants and not (args.topk or args.teacher_lse or args.stage):
        # the peer-memory exchange's kernels at the full workload in every default run: two ranks emulated on this
        # GPU, 5 timed steps (a failure here is recorded, never allowed to drop the headline line)
        try:
            alongside["p2p_one_gpu"] = p2p_one_gpu_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, timer, want_dW, P=2,
                                                       steps=min(5, args.steps))
        except Exception as e:  # noqa: BLE001
            alongside["p2p_one_gpu"] = {"error": f"{type(e).__name__}: {e}"[:300]}

    if args.handoff and world == 1:
        alongside["handoff"] = handoff_leg(args, cfg, kd, H_t, Ht, Wt, Hs, Ws, mask, kw, out, dW, n_eff, stream, local)

    if not vocab_head and (world == 1 or args.shard == "token") and not (args.topk or args.teacher_lse or args.stage):
        # the vocab-sharded driver at this N: P = 1 identity exchanges at N = 1 (the N > 1 headline's code path), or
        # a P-way group simulated on one GPU (--sim-vocab-shards P: rank 0's share of the strong-scaling step)
        if world == 1:
            v = vocab_sharded_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, world, rank, dev, want_dW, timer, local,
                                  own_tokens=False)
            for k in ("_prof", "_n_eff_rank", "clocks"):
                v.pop(k)
            pv = max(1, args.sim_vocab_shards)
            v["strong_scaling_efficiency_excl_comm"] = v["value"] / (pv * value) if pv > 1 else None
            v["vs_fused_single_call"] = v["value"] / value if pv == 1 else None
            alongside["vocab_sharded"] = v

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_med, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic (kd_inputs recipe, seeded)",
                "config": workload_desc(cfg, n_tok, want_dW, world, args.grad_precision, args.teacher_lse, args.topk,
                                        args.stage),
                "clocks": clocks, "e2e": e2e,
                "gpu_launches": int(round(launches_per_step * args.steps)), "roofline": roofline, "cpu_baseline": cpu,
                "useful_flop_frac": useful_frac, "kernels": kernels, "nonfinite_tokens": nonfinite,
                "energy": ({"tokens_per_joule": value / clocks["power_w_median"],
                            "power_w_median": clocks["power_w_median"],
                            "note": "the step runs on the B200's software power cap: throughput = power budget / "
                                    "energy per token, so tokens per joule is the box-independent figure"}
                           if world == 1 and isinstance(clocks, dict) and clocks.get("power_w_median") else None),
                "timing": {"ms_per_step": "median of the K timed steps (per-step CUDA events), max over ranks",
                           "ms_per_step_mean": (vleg["ms_per_step_mean"] if vocab_head else t_tok["mean_ms"])},
                "tokens_loss_bearing_per_gpu": n_eff, **alongside}
        if vocab_head:
            line["config"]["parallelism"] = vleg["layout"]
            line["config"]["tokens_per_step"] = vleg["tokens_per_step"]
            line["vocab_sharded_headline"] = vleg
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
