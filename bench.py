#!/usr/bin/env python
"""bench.py — KD tokens/s of the fused KD hot path (BASELINE.json metric) on N B200s.

One step = one ``kd_fused_fwd_bwd`` call over one batch: recompute the teacher logits from H_t (V = 151936),
the student logits, the divergence, the per-token loss and dL/dh_s (BASELINE.json configs[1] by default:
Qwen3-8B d_t=4096 -> Qwen3-1.7B d_s=2048, 8 x 4096 tokens, FKL, T = 1).

    python bench.py [--gpus N --steps K --warmup W] [--config c2|c3_rkl|c3_jsd|c4|c5] [--dW]
    python bench.py --impl reference ...      # the fp64 CPU oracle on this box's host cores

Multi-GPU (torchrun): the headline value is token sharding with no data-path collective — every rank owns its
own 32768 tokens and a full copy of both heads (weak scaling); the only collectives are the timing barrier / max.
The north star's vocabulary sharding (LM-head rows split over the ranks, every rank sees all N·P tokens, NCCL
all-gather of the per-token records + reduce-scatter of dh) is measured in the same run and reported alongside under
"vocab_sharded" (``--shard vocab`` swaps the two).  Prints ONE JSON line on rank 0.
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kd", choices=["kd", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(KI.CONFIGS))
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per GPU (default: the config's)")
    ap.add_argument("--dW", action="store_true", help="also compute dL/dW_s")
    ap.add_argument("--grad-precision", default="split", choices=["split", "bf16"],
                    help="G fed to the backward GEMMs: split hi+lo bf16 (parity-grade, default) or one bf16 plane "
                         "(KD_GRAD_BF16, fast, not within the north-star gradient tolerance)")
    ap.add_argument("--shard", default="token", choices=["token", "vocab"],
                    help="layout of the headline value at N>1: token sharding (default, no data-path collective) or "
                         "vocab sharding (north star: LM-head rows split over ranks, record all-gather + dh "
                         "all-reduce over NCCL).  At N>1 the other layout is measured too and reported alongside.")
    ap.add_argument("--teacher-lse", action="store_true",
                    help="SURVEY §8(f) NEXT-2(i): the teacher ships its per-token LSE record with H_t (computed once by "
                         "kd_teacher_lse outside the timed region, as the teacher side would); the timed step is "
                         "kd_fused_fwd_bwd_lse, whose pass 1 sweeps the student head only (FKL/JSD/TVD)")
    ap.add_argument("--vocab-ranks", type=int, default=0,
                    help="vocab-sharded leg on a 2-D grid: ranks per vocab group (P_voc; default all ranks). "
                         "world / P_voc token groups (BASELINE config 4: 8x1, 4x2, 2x4, 1x8)")
    ap.add_argument("--sim-vocab-shards", type=int, default=0,
                    help="1 GPU: time rank 0's share of a P-way vocab-sharded step (compute only, no exchange)")
    ap.add_argument("--topk", type=int, default=0,
                    help="SURVEY §8(f) NEXT-3 negative control: the prior-art top-k teacher transfer (k <= 32).  The "
                         "teacher's (idx, logit) top-k is produced once by kd_teacher_topk outside the timed region; "
                         "the timed step is kd_topk_fwd_bwd (student head only, FKL against the truncated teacher)")
    ap.add_argument("--stage", action="store_true",
                    help="staged variant (kd_problem.stage_logits, SURVEY §8(f) NEXT-2(ii)): pass 1 writes the token "
                         "chunk's fp32 logits, an HBM-bound kernel forms G from them (no second tensor sweep)")
    ap.add_argument("--no-variants", action="store_true", help="skip the staged-variant leg of the default run")
    ap.add_argument("--graph", action="store_true", help="also time the step captured into a CUDA graph")
    ap.add_argument("--handoff", action="store_true",
                    help="add the hidden-state hand-off leg (SURVEY NEXT-4): teacher process -> student via CUDA IPC")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=128)
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
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


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


# ------------------------------------------------------------------------------------------- vocab-sharded leg
def vocab_sharded_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, world, rank, dev, want_dW):
    """Vocabulary sharding (BASELINE.json north_star), optionally on a 2-D grid (config 4:
    P_tok x P_voc).  The ranks form world / P_voc vocab groups of P_voc consecutive ranks; inside a group rank j keeps
    LM-head rows [v0, v1) of both heads (128-row granules) and sees every token of the group (the members' token
    slices are all-gathered once, outside the timed region), so per-GPU work stays that of one GPU (weak scaling).
    One step = ``sharding.vocab_sharded_fwd_bwd`` on the group: kd_vocab_stats -> NCCL all-gather of the 20 B/token
    records -> kd_vocab_backward (rank-order merge, pass 2, partial dh, local dW rows) -> NCCL reduce-scatter of dh
    (JSD/TVD add the (K, J) all-gather per token chunk)."""
    import torch
    import torch.distributed as dist

    from paper_2603_01875_b200 import sharding

    sim = world == 1 and args.sim_vocab_shards > 1  # one GPU playing rank 0 of a P-way vocab group (no exchange)
    pv = args.sim_vocab_shards if sim else (args.vocab_ranks if args.vocab_ranks > 0 else world)
    if not sim and world % pv:
        raise SystemExit(f"--vocab-ranks {pv} must divide the world size {world}")
    group, g0 = None, (rank // pv) * pv
    if world > 1 and pv < world:
        for t in range(world // pv):  # every rank creates every group, in the same order
            g = dist.new_group(list(range(t * pv, (t + 1) * pv)))
            if t == rank // pv:
                group = g
    j = rank - g0  # position inside the vocab group
    bounds = sharding.vocab_shard_bounds(cfg.vocab, pv)
    v0, v1 = bounds[j]
    Wt_sh, Ws_sh = Wt[v0:v1].contiguous(), Ws[v0:v1].contiguous()
    if sim:  # the group's N·P tokens: this rank's own tokens stand in for the P members' slices
        Ht_all, Hs_all = Ht.repeat(pv, 1), Hs.repeat(pv, 1)
        mask_all = mask.repeat(pv) if mask is not None else None
    elif pv > 1:
        def gather(x):
            parts = [torch.empty_like(x) for _ in range(pv)]
            dist.all_gather(parts, x.contiguous(), group=group)
            return torch.cat(parts)
        Ht_all, Hs_all = gather(Ht), gather(Hs)
        mask_all = gather(mask) if mask is not None else None
    else:
        Ht_all, Hs_all, mask_all = Ht, Hs, mask
    n_all = Ht_all.shape[0]
    n_eff_own = int(mask.sum().item()) if mask is not None else Ht.shape[0]
    n_eff_job = n_eff_own * (pv if sim else 1)
    if world > 1:
        t = torch.tensor([n_eff_own], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        n_eff_job = int(t.item())
    dW = torch.empty(v1 - v0, cfg.d_s, dtype=torch.float32, device=dev) if want_dW else None
    # each rank keeps dh_s / loss of its own tokens only (the student's backward continues on them): the dh
    # exchange is a reduce-scatter, half the bytes of an all-reduce
    kw = dict(vocab=cfg.vocab, v_begin=v0, T=cfg.temperature, kind=cfg.kind, beta=cfg.jsd_beta, loss_scale=1.0,
              want_dW=want_dW, accumulate_dW=False, group=group, dh_reduce="scatter")

    def step():
        return sharding.vocab_sharded_fwd_bwd(Ht_all, Wt_sh, Hs_all, Ws_sh, mask_all, dW_s=dW, **kw)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        r = step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    kd.profile_read()
    kd.profile_enable(True)
    e0.record(stream)
    for _ in range(args.steps):
        r = step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    kd.profile_enable(False)
    vprof = kd.profile_read()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rec_bytes = 20 * n_all * pv
    kj_bytes = 8 * n_all * pv if cfg.kind in ("jsd", "tvd") else 0
    grid = f"{max(1, world // pv)} token groups x {pv} vocab shards" + (" (SIMULATED on one GPU)" if sim else "")
    return {"value": n_eff_job * args.steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / args.steps,
            "scaling": "weak", "tokens_per_step": n_all * (world // pv), "vocab_rows_per_gpu": v1 - v0,
            "grid": grid,
            "layout": f"vocab-sharded ({grid}): LM-head rows split in 128-row granules over each group of {pv} "
                      f"ranks, every rank of a group sees its {n_all} tokens",
            "exchange_bytes_per_step_per_rank": {"records_allgather": rec_bytes, "kj_allgather": kj_bytes,
                                                 "dh_reduce_scatter": 4 * n_all * cfg.d_s * (pv - 1) // pv},
            "loss_finite": bool(torch.isfinite(r.loss).all().item()),
            "kernels_ms_per_step": {k: t / args.steps for k, (n, t) in sorted(vprof.items(), key=lambda kv: -kv[1][1])},
            **({"simulated": f"one GPU runs rank 0's work of a {pv}-way vocab group (its {v1 - v0} head rows x the "
                             f"group's {n_all} tokens) with identity exchanges: the compute of one rank at P={pv}, no "
                             f"communication; outputs are that shard's partial statistics, not the full result. "
                             f"value = the group's tokens per step / this time, i.e. the P-GPU job throughput "
                             f"excluding the exchanges"} if sim else {})}


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
    proc = ctx.Process(target=_handoff_teacher, args=(child, H_t_bits, cfg.vocab, local))
    proc.start()
    try:
        h_ht, s_ht, h_lg, s_lg = parent.recv()
        m_ht = kd.HandoffTensor(h_ht, s_ht, torch.bfloat16)
        m_lg = kd.HandoffTensor(h_lg, s_lg, torch.bfloat16)
        assert torch.equal(m_ht.tensor, Ht_local)
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
    return {"transport": "kd_handoff_export/open (CUDA IPC); teacher and student are separate processes on the same "
                         "B200 — pulls are D2D copies through the exporter's mapping (read + write of the bytes)",
            "h_t_bytes_per_step": b_ht, "full_logits_bytes_per_step": b_lg, "volume_ratio": b_lg / b_ht,
            "pull_h_t_ms": t_ht, "pull_logits_ms": t_lg, "time_ratio": t_lg / t_ht,
            "pull_h_t_GBps": b_ht / (t_ht / 1e3) / 1e9, "pull_logits_GBps": b_lg / (t_lg / 1e3) / 1e9,
            "zero_copy_step": {"value": n_eff / (t_step / 1e3), "unit": UNIT, "ms_per_step": t_step,
                               "what": "kd_fused_fwd_bwd reading the teacher process's H_t in place"}}


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

    # ---- inputs: heads replicated (seed 1000), each rank its own tokens (seed 1001 + rank)
    W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
    H_t, H_s = KI.make_hidden(n_tok, W_t, W_s, seed=1001 + rank, head_seed=1000)
    mask_np = KI.make_mask(KI.KDConfig(**{**cfg.__dict__, "n_seq": max(1, n_tok // cfg.seq_len)}),
                           seed=1002 + rank) if cfg.mask != "none" else None
    if mask_np is not None:
        mask_np = np.resize(mask_np, n_tok)

    def up(b):
        return torch.from_numpy(b.view(np.int16)).to(dev).view(torch.bfloat16)

    Wt, Ws, Ht, Hs = up(W_t), up(W_s), up(H_t), up(H_s)
    mask = torch.from_numpy(mask_np).to(dev) if mask_np is not None else None
    n_eff = int(mask_np.sum()) if mask_np is not None else n_tok
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

    lse_t = tk = None
    if args.topk:
        if cfg.kind != "fkl":
            raise SystemExit("--topk is forward KL only (kd_topk_fwd_bwd)")
        tk = kd.teacher_topk(Ht, Wt, mask, k=args.topk, d_s=cfg.d_s, T=cfg.temperature)
    if args.teacher_lse:
        # the teacher side's record, produced once per batch by the teacher (not student work: outside the timing)
        lse_t = kd.teacher_lse(Ht, Wt, mask, d_s=cfg.d_s, T=cfg.temperature, kind=cfg.kind)

    def step():
        if tk is not None:
            return kd.topk_fwd_bwd(Hs, Ws, tk[0], tk[1], mask, d_t=cfg.d_t, T=cfg.temperature, loss_scale=1.0,
                                   want_dW=want_dW, dW_s=dW, grad_precision=args.grad_precision, out=out)
        if lse_t is not None:
            return kd.fused_fwd_bwd_lse(Ht, Wt, Hs, Ws, lse_t, mask, dW_s=dW, out=out, **kw)
        return kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches_per_step = kd.last_launch_count()

    # ---- timed region (device events on the launching stream; live per-kernel events inside the library)
    sampler = ClockSampler(local)
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    kd.profile_read()
    kd.profile_enable(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    kd.profile_enable(False)
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    prof = kd.profile_read()
    ms_max = max_over_ranks(ms)
    value = world * n_eff * args.steps / (ms_max / 1000.0)
    nonfinite = int(out.n_nonfinite.item())

    # ---- roofline of the dominant kernel (live CUDA events)
    pk = peaks()
    flops_pass = 2.0 * n_eff * cfg.vocab * (cfg.d_t + cfg.d_s)  # both LM-head GEMMs, one vocab sweep
    flops_g = 2.0 * n_eff * cfg.vocab * cfg.d_s                   # G · W_s  (or Gᵀ · H_s)
    flops_p1 = 2.0 * n_eff * cfg.vocab * cfg.d_s if (args.teacher_lse or args.topk) else flops_pass  # student only
    flops_p2 = 2.0 * n_eff * cfg.vocab * cfg.d_s if args.topk else flops_pass
    algo = {"pass1": flops_p1, "pass2": flops_p2, "gemm_dh": flops_g, "gemm_dW": flops_g}
    gm = 2.0 if args.grad_precision == "split" else 1.0                 # split-bf16 G: 2 MMAs per product
    exec_mult = {"pass1": 1.0, "pass2": 1.0, "gemm_dh": gm, "gemm_dW": gm}
    kernels = {}
    total_ms = sum(t for _, t in prof.values()) or 1.0
    for name, (n, t) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        e = {"launches": n, "ms_per_step": t / args.steps, "share": t / total_ms}
        if name in algo:
            e["algorithmic_tflops"] = algo[name] * args.steps / (t / 1e3) / 1e12
            e["tensor_pipe_tflops_executed"] = e["algorithmic_tflops"] * exec_mult[name]
        if name == "stage_grad":
            # HBM-bound: per (token, v) 8 B of staged logits read + G written (split: 4 B, bf16: 2 B, JSD/TVD: 8 B)
            wb = 8 if cfg.kind in ("jsd", "tvd") else (4 if args.grad_precision == "split" else 2)
            e["algorithmic_bytes_per_launch"] = n_eff * cfg.vocab * (8 + wb) * args.steps / n
            e["achieved_GBps"] = e["algorithmic_bytes_per_launch"] / (t / n / 1e3) / 1e9
            e["hbm_frac"] = e["achieved_GBps"] / pk["hbm_gbs"]
        kernels[name] = e
    dom = max((k for k in kernels if k in algo), key=lambda k: kernels[k]["ms_per_step"])
    peak_sust = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom, {}).get("dram_bytes_per_launch")
    n_l, t_l = prof[dom]
    achieved = algo[dom] * args.steps / n_l / (t_l / n_l / 1e3) / 1e12
    roofline = {"bound": "tensor", "kernel": f"kd_pass_kernel ({dom})" if dom.startswith("pass") else dom,
                "achieved": achieved, "peak": peak_sust, "unit": "TFLOP/s", "frac": achieved / peak_sust,
                "traffic": traffic,
                "peak_note": f"bf16 dense, {pk['source']}, sustained (kernel timed inside a long step); "
                             f"burst {pk['bf16_tflops']}",
                "algorithmic_per_launch": (f"2*tokens*V*d_s flop = " if (dom == "pass1" and args.teacher_lse)
                                           or args.topk else
                                           f"2*tokens*V*(d_t+d_s) flop = " if dom.startswith("pass") else
                                           f"2*tokens*V*d_s flop = ") + f"{algo[dom] * args.steps / n_l:.4g}"}
    step_useful = 2.0 * n_eff * cfg.vocab * ((0 if args.topk else cfg.d_t) + 2 * cfg.d_s + (cfg.d_s if want_dW else 0))
    useful_frac = step_useful * args.steps / (ms_max / 1e3) / 1e12 / peak_sust

    # ---- e2e: same metric through the C-ABI with host buffers (pinned), every step's H2D of its inputs and D2H of
    # its results inside the timed region.  Copies run on a side stream, double-buffered, so step i+1's upload and
    # step i-1's download overlap step i's kernels (the public-API pattern a training loop would use).
    e2e = None
    if not args.no_e2e:
        hHt = Ht.cpu().pin_memory()
        hHs = Hs.cpu().pin_memory()
        hmask = mask.cpu().pin_memory() if mask is not None else None
        hlse = lse_t.cpu().pin_memory() if lse_t is not None else None
        htk = (tk[0].cpu().pin_memory(), tk[1].cpu().pin_memory()) if tk is not None else None
        hloss = [torch.empty(n_tok, dtype=torch.float32).pin_memory() for _ in range(2)]
        hdh = [torch.empty(n_tok, cfg.d_s, dtype=torch.float32).pin_memory() for _ in range(2)]
        dH = [(torch.empty_like(Ht), torch.empty_like(Hs), torch.empty_like(mask) if mask is not None else None,
               torch.empty_like(lse_t) if lse_t is not None else None,
               (torch.empty_like(tk[0]), torch.empty_like(tk[1])) if tk is not None else None) for _ in range(2)]
        outs = [kd.KDResult(torch.empty(n_tok, dtype=torch.float32, device=dev),
                            torch.empty(n_tok, cfg.d_s, dtype=torch.float32, device=dev), None,
                            torch.zeros(1, dtype=torch.int64, device=dev)) for _ in range(2)]
        cs = torch.cuda.Stream(device=dev)
        in_ready = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]

        def upload(b):
            with torch.cuda.stream(cs):
                if htk is None:  # the top-k student never sees H_t: the teacher ships (idx, logit) pairs instead
                    dH[b][0].copy_(hHt, non_blocking=True)
                else:
                    dH[b][4][0].copy_(htk[0], non_blocking=True)
                    dH[b][4][1].copy_(htk[1], non_blocking=True)
                dH[b][1].copy_(hHs, non_blocking=True)
                if hmask is not None:
                    dH[b][2].copy_(hmask, non_blocking=True)
                if hlse is not None:
                    dH[b][3].copy_(hlse, non_blocking=True)
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
                if htk is not None:
                    kd.topk_fwd_bwd(dH[b][1], Ws, dH[b][4][0], dH[b][4][1], dH[b][2], d_t=cfg.d_t, T=cfg.temperature,
                                    loss_scale=1.0, want_dW=want_dW, dW_s=dW, grad_precision=args.grad_precision,
                                    out=outs[b])
                elif hlse is not None:
                    kd.fused_fwd_bwd_lse(dH[b][0], Wt, dH[b][1], Ws, dH[b][3], dH[b][2], dW_s=dW, out=outs[b], **kw)
                else:
                    kd.fused_fwd_bwd(dH[b][0], Wt, dH[b][1], Ws, dH[b][2], dW_s=dW, out=outs[b], **kw)
                done[b].record(stream)
                with torch.cuda.stream(cs):
                    cs.wait_event(done[b])
                    hloss[b].copy_(outs[b].loss, non_blocking=True)
                    hdh[b].copy_(outs[b].dh_s, non_blocking=True)

        run_pipeline(2)
        torch.cuda.synchronize()
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(cs)
        stream.wait_event(t0)
        run_pipeline(args.steps)
        t1.record(cs)
        torch.cuda.synchronize()
        ms_e2e = max_over_ranks(t0.elapsed_time(t1))
        assert torch.equal(hloss[(args.steps - 1) & 1], outs[(args.steps - 1) & 1].loss.cpu())
        h2d = n_tok * ((0 if htk else cfg.d_t) + cfg.d_s) * 2 + (n_tok if mask is not None else 0) \
            + (8 * n_tok if hlse is not None else 0) + (8 * args.topk * n_tok if htk else 0)
        d2h = n_tok * 4 + n_tok * cfg.d_s * 4
        e2e = {"value": world * n_eff * args.steps / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "note": "heads resident in HBM (weights); per step: " +
                       ("H_s + the teacher's top-k (idx, logit) pairs" if htk else
                        "H_t/H_s + the teacher's LSE record" if hlse is not None else "H_t/H_s") +
                       " (+mask) pinned-host->device and loss/dh_s device->pinned-host, on a copy stream overlapped "
                       "with the neighbouring steps"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, cores = oracle_tokens_per_s(cfg, args.cpu_sample_tokens, want_dW)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_sample_tokens} tokens at full {cfg.name} shapes, fp64 numpy "
                         f"({dt:.1f} s; BLAS threads = all {cores} affinity cores)"}
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

    alongside = {}
    if args.graph:
        # the same step captured once into a CUDA graph and replayed (no per-launch host work; the library's calls
        # are capturable: no host syncs, no allocation, every launch on the caller's stream)
        cs_ = torch.cuda.Stream(device=dev)
        cs_.wait_stream(stream)
        with torch.cuda.stream(cs_):
            step()
        stream.wait_stream(cs_)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(max(3, args.warmup)):
            graph.replay()
        torch.cuda.synchronize()
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        ms_g = max_over_ranks(g0.elapsed_time(g1))
        alongside["cuda_graph"] = {"value": world * n_eff * args.steps / (ms_g / 1e3), "unit": UNIT,
                                   "ms_per_step": ms_g / args.steps,
                                   "what": "one step captured into a CUDA graph, replayed K times (same inputs)"}

    # ---- the staged variant (kd_problem.stage_logits) on the same inputs, timed the same way
    if not (args.stage or args.topk or args.teacher_lse or args.no_variants):
        kw_st = dict(kw, stage_logits=True)
        for _ in range(max(3, args.warmup)):
            kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw_st)
        torch.cuda.synchronize()
        barrier()
        kd.profile_read()
        kd.profile_enable(True)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, mask, dW_s=dW, out=out, **kw_st)
        s1.record(stream)
        torch.cuda.synchronize()
        barrier()
        kd.profile_enable(False)
        sprof = kd.profile_read()
        ms_st = max_over_ranks(s0.elapsed_time(s1))
        stot = sum(t for _, t in sprof.values()) or 1.0
        alongside["staged_variant"] = {
            "value": world * n_eff * args.steps / (ms_st / 1e3), "unit": UNIT, "ms_per_step": ms_st / args.steps,
            "what": "kd_problem.stage_logits=1 (SURVEY NEXT-2(ii)): pass 1 also writes the token chunk's fp32 logits "
                    "(2 x Nc x V x 4 B, one chunk at a time), an HBM-bound kernel forms G from them; no pass-2 sweep. "
                    "Same outputs within the same tolerances (tests/test_gpu_stage.py); same launch config otherwise",
            "useful_flop_frac": step_useful * args.steps / (ms_st / 1e3) / 1e12 / peak_sust,
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

    if args.handoff and world == 1:
        alongside["handoff"] = handoff_leg(args, cfg, kd, H_t, Ht, Wt, Hs, Ws, mask, kw, out, dW, n_eff, stream, local)

    # ---- the other layout, measured in the same run (north star: vocab sharding, token sharding alongside)
    if world > 1 or args.shard == "vocab" or args.sim_vocab_shards > 1:
        vleg = vocab_sharded_leg(args, cfg, kd, Wt, Ws, Ht, Hs, mask, world, rank, dev, want_dW)
        tleg = {"value": value, "unit": UNIT, "ms_per_step": ms_max / args.steps, "scaling": "weak",
                "tokens_per_step": n_tok * world, "layout": f"token-sharded x{world}, full heads per rank"}
        if args.shard == "vocab":
            value, ms_max = vleg["value"], vleg["ms_per_step"] * args.steps
            alongside["token_sharded"] = tleg
        else:
            alongside["vocab_sharded"] = vleg

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (kd_inputs recipe, seeded)",
                "config": workload_desc(cfg, n_tok, want_dW, world, args.grad_precision, args.teacher_lse, args.topk,
                                        args.stage),
                "clocks": clocks, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "roofline": roofline, "cpu_baseline": cpu,
                "useful_flop_frac": useful_frac, "kernels": kernels, "nonfinite_tokens": nonfinite,
                "tokens_loss_bearing_per_gpu": n_eff, **alongside}
        if args.shard == "vocab":
            line["config"]["parallelism"] = vleg["layout"]
            line["config"]["tokens_per_step"] = vleg["tokens_per_step"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
