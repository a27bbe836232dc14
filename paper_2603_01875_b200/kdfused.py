"""Thin ctypes binding of ``include/kdfused.h`` (argument marshalling only).

Every step of the KD hot path runs in the CUDA kernels of ``libkdfused.so``; this module only turns
torch tensors into device pointers + sizes, allocates outputs / workspace with PyTorch (plumbing), and
raises on a non-OK status.  There is no CPU fallback: if the library or a GPU is missing, calls fail
loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KD_LIB_PATH") or os.path.join(_HERE, "libkdfused.so")  # override: A/B experiments

KINDS = {"fkl": 0, "rkl": 1, "jsd": 2, "tvd": 3}
STATUS = {0: "KD_OK", 1: "KD_ERR_INVALID_ARG", 2: "KD_ERR_SHAPE", 3: "KD_ERR_ALIGNMENT", 4: "KD_ERR_UNSUPPORTED",
          5: "KD_ERR_WORKSPACE_TOO_SMALL", 6: "KD_ERR_CUDA"}
EXPORTED = ("kd_check_problem", "kd_workspace_size", "kd_fused_fwd_bwd", "kd_teacher_lse", "kd_fused_fwd_bwd_lse",
            "kd_teacher_topk", "kd_topk_fwd_bwd",
            "kd_vocab_stats", "kd_vocab_backward",
            "kd_vocab_partials", "kd_vocab_finish", "kd_p2p_arena_bytes", "kd_p2p_outputs", "kd_vocab_stats_p2p", "kd_vocab_backward_p2p",
            "kd_vocab_partials_p2p", "kd_vocab_finish_p2p",
            "kd_p2p_combine", "kd_p2p_wait", "kd_handoff_export", "kd_handoff_open", "kd_handoff_close",
            "kd_gemm_bf16_f32",
            "kd_last_launch_count", "kd_profile_enable", "kd_profile_read", "kd_profile_kernel_name",
            "kd_last_error", "kd_abi_version")


class KDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class KDProblem(ctypes.Structure):
    _fields_ = [("n_tokens", ctypes.c_int64), ("d_t", ctypes.c_int32), ("d_s", ctypes.c_int32),
                ("vocab", ctypes.c_int64), ("v_begin", ctypes.c_int64), ("v_end", ctypes.c_int64),
                ("temperature", ctypes.c_float), ("kind", ctypes.c_int32), ("jsd_beta", ctypes.c_float),
                ("loss_scale", ctypes.c_float), ("want_dW", ctypes.c_int32), ("accumulate_dW", ctypes.c_int32),
                ("chunk_tokens", ctypes.c_int32), ("grad_precision", ctypes.c_int32),
                ("stage_logits", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class KDP2P(ctypes.Structure):
    """kd_p2p: one rank's view of the peer-memory exchange (every rank's arena as mapped in this process)."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("d_s", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("max_rows", ctypes.c_int64), ("max_tokens", ctypes.c_int64),
                ("arena", ctypes.c_void_p * 8)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libkdfused.so (built in-tree by ``paper_2603_01875_b200.build``); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2603_01875_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, i64p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p
    P = ctypes.POINTER(KDProblem)
    L.kd_check_problem.argtypes = [P]
    L.kd_check_problem.restype = ctypes.c_int
    L.kd_workspace_size.argtypes = [P]
    L.kd_workspace_size.restype = sz
    L.kd_fused_fwd_bwd.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, i64p, vp, sz, vp]
    L.kd_fused_fwd_bwd.restype = ctypes.c_int
    L.kd_teacher_lse.argtypes = [P, vp, vp, vp, vp, vp, sz, vp]
    L.kd_teacher_lse.restype = ctypes.c_int
    L.kd_fused_fwd_bwd_lse.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64p, vp, sz, vp]
    L.kd_fused_fwd_bwd_lse.restype = ctypes.c_int
    L.kd_teacher_topk.argtypes = [P, vp, vp, vp, i32, vp, vp, vp, sz, vp]
    L.kd_teacher_topk.restype = ctypes.c_int
    L.kd_topk_fwd_bwd.argtypes = [P, vp, vp, vp, i32, vp, vp, vp, vp, vp, i64p, vp, sz, vp]
    L.kd_topk_fwd_bwd.restype = ctypes.c_int
    L.kd_vocab_stats.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.kd_vocab_stats.restype = ctypes.c_int
    L.kd_vocab_backward.argtypes = [P, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, i64p, vp, sz, vp]
    L.kd_vocab_backward.restype = ctypes.c_int
    L.kd_vocab_partials.argtypes = [P, vp, vp, vp, vp, vp, vp, i32, vp, vp, sz, vp]
    L.kd_vocab_partials.restype = ctypes.c_int
    L.kd_vocab_finish.argtypes = [P, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, i64p, vp, sz, vp]
    L.kd_vocab_finish.restype = ctypes.c_int
    X = ctypes.POINTER(KDP2P)
    L.kd_p2p_arena_bytes.argtypes = [i32, ctypes.c_int64, ctypes.c_int64, i32]
    L.kd_p2p_arena_bytes.restype = sz
    L.kd_p2p_outputs.argtypes = [X, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
    L.kd_p2p_outputs.restype = ctypes.c_int
    L.kd_vocab_stats_p2p.argtypes = [P, vp, vp, vp, vp, vp, vp, sz, X, i32, vp]
    L.kd_vocab_stats_p2p.restype = ctypes.c_int
    L.kd_vocab_backward_p2p.argtypes = [P, vp, vp, vp, vp, vp, vp, i32, vp, vp, i64p, vp, sz, X, i32, ctypes.c_uint32,
                                        vp]
    L.kd_vocab_backward_p2p.restype = ctypes.c_int
    L.kd_vocab_partials_p2p.argtypes = [P, vp, vp, vp, vp, vp, vp, sz, X, i32, ctypes.c_uint32, vp]
    L.kd_vocab_partials_p2p.restype = ctypes.c_int
    L.kd_vocab_finish_p2p.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, i64p, vp, sz, X, i32, ctypes.c_uint32, vp]
    L.kd_vocab_finish_p2p.restype = ctypes.c_int
    L.kd_p2p_combine.argtypes = [X, i32, ctypes.c_int64, ctypes.c_int64, vp, i32, ctypes.c_uint32, vp]
    L.kd_p2p_combine.restype = ctypes.c_int
    L.kd_p2p_wait.argtypes = [X, ctypes.c_uint32, vp]
    L.kd_p2p_wait.restype = ctypes.c_int
    L.kd_handoff_export.argtypes = [vp, ctypes.c_uint64, vp]
    L.kd_handoff_export.restype = ctypes.c_int
    L.kd_handoff_open.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_uint64)]
    L.kd_handoff_open.restype = ctypes.c_int
    L.kd_handoff_close.argtypes = [vp]
    L.kd_handoff_close.restype = ctypes.c_int
    L.kd_gemm_bf16_f32.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
    L.kd_gemm_bf16_f32.restype = ctypes.c_int
    L.kd_last_launch_count.restype = ctypes.c_int32
    L.kd_profile_enable.argtypes = [i32]
    L.kd_profile_enable.restype = i32
    L.kd_profile_read.argtypes = [vp, vp, i32]
    L.kd_profile_read.restype = i32
    L.kd_profile_kernel_name.argtypes = [i32]
    L.kd_profile_kernel_name.restype = ctypes.c_char_p
    L.kd_last_error.restype = ctypes.c_char_p
    L.kd_abi_version.restype = ctypes.c_int32
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise KDError(status, lib().kd_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


GRAD_PRECISION = {"split": 0, "bf16": 1}


def make_problem(n_tokens, d_t, d_s, vocab, *, T=1.0, kind="fkl", beta=0.5, loss_scale=1.0, want_dW=False,
                 accumulate_dW=False, v_begin=0, v_end=None, chunk_tokens=0, grad_precision="split",
                 stage_logits=False) -> KDProblem:
    p = KDProblem()
    p.n_tokens, p.d_t, p.d_s, p.vocab = int(n_tokens), int(d_t), int(d_s), int(vocab)
    p.v_begin = int(v_begin)
    p.v_end = int(vocab if v_end is None else v_end)
    p.temperature = float(T)
    p.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
    p.jsd_beta = float(beta)
    p.loss_scale = float(loss_scale)
    p.want_dW = int(bool(want_dW))
    p.accumulate_dW = int(bool(accumulate_dW))
    p.chunk_tokens = int(chunk_tokens)
    p.grad_precision = GRAD_PRECISION[grad_precision] if isinstance(grad_precision, str) else int(grad_precision)
    p.stage_logits = int(bool(stage_logits))
    return p


def workspace_size(p: KDProblem) -> int:
    _check(lib().kd_check_problem(ctypes.byref(p)))
    return int(lib().kd_workspace_size(ctypes.byref(p)))


_ws_cache: dict = {}
_ws_graph_held: list = []  # buffers a captured CUDA graph may still point at: never freed


def _workspace(nbytes: int, device, stream=None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """The call's workspace: the caller's ``workspace`` tensor if given (required size checked by the library),
    else a cached buffer keyed by (device, stream).

    The cached buffer is allocated ON the launch stream, so when it is outgrown and dropped the caching allocator
    only reuses its memory in that stream's order (after the kernels already queued there).  A buffer handed out
    while the stream is being captured into a CUDA graph is kept alive for the life of the process, so a later,
    larger call can never free memory a graph replays into."""
    if workspace is not None:
        if not workspace.is_cuda or workspace.device != torch.device(device):
            raise ValueError("workspace must be a CUDA tensor on the inputs' device")
        return workspace
    dev = torch.device(device)
    s = torch.cuda.current_stream(dev) if stream is None else stream
    key = (dev, s.cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        _ws_cache.pop(key, None)
        with torch.cuda.stream(s):
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    if torch.cuda.is_current_stream_capturing() and not any(b is buf for b in _ws_graph_held):
        _ws_graph_held.append(buf)
    return buf


def last_launch_count() -> int:
    return int(lib().kd_last_launch_count())


def profile_enable(on: bool) -> bool:
    """Bracket every library launch with CUDA events (live per-kernel timing)."""
    return bool(lib().kd_profile_enable(int(bool(on))))


def profile_read() -> dict:
    """{kernel name: (launches, total_ms)} since the last read (synchronises the recorded events)."""
    L = lib()
    n = 32
    launches = (ctypes.c_int32 * n)()
    total = (ctypes.c_double * n)()
    k = L.kd_profile_read(launches, total, n)
    if k < 0:
        raise RuntimeError("kd_profile_read: an event failed")
    return {L.kd_profile_kernel_name(i).decode(): (int(launches[i]), float(total[i]))
            for i in range(min(k, n)) if launches[i] > 0}


def _as_bf16(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.bfloat16:
        raise ValueError(f"{name} must be bfloat16")
    return t.contiguous()


@dataclass
class KDResult:
    loss: torch.Tensor          # [N] f32
    dh_s: torch.Tensor          # [N, d_s] f32
    dW_s: torch.Tensor | None   # [V_r, d_s] f32
    n_nonfinite: torch.Tensor   # [1] i64 (device)


def fused_fwd_bwd(h_t, W_t, h_s, W_s, mask=None, *, T=1.0, kind="fkl", beta=0.5, loss_scale=1.0, want_dW=False,
                  accumulate_dW=False, dW_s=None, chunk_tokens=0, grad_precision="split", stage_logits=False,
                  out=None, stream=None, workspace=None) -> KDResult:
    """kd_fused_fwd_bwd: per-token loss, dL/dh_s and (optionally) dL/dW_s for device tensors.

    ``stage_logits=True`` selects the staged variant (pass 1 writes the chunk's fp32 logits, G from them)."""
    h_t, W_t, h_s, W_s = (_as_bf16(x, n) for x, n in ((h_t, "h_t"), (W_t, "W_t"), (h_s, "h_s"), (W_s, "W_s")))
    N, d_t = h_t.shape
    V, d_s = W_s.shape
    # outputs live with the student's tensors: h_t may be a teacher buffer mapped from a peer GPU (kd_handoff_open),
    # read in place over NVLink by the kernels running on the student's device
    dev = h_s.device
    p = make_problem(N, d_t, d_s, V, T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, chunk_tokens=chunk_tokens, grad_precision=grad_precision,
                     stage_logits=stage_logits)
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    if out is None:
        loss = torch.empty(N, dtype=torch.float32, device=dev)
        dh = torch.empty(N, d_s, dtype=torch.float32, device=dev)
        nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        loss, dh, nnf = out.loss, out.dh_s, out.n_nonfinite
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if accumulate_dW else torch.empty)(V, d_s, dtype=torch.float32, device=dev)
    ws = _workspace(workspace_size(p), dev, stream, workspace)
    _check(lib().kd_fused_fwd_bwd(ctypes.byref(p), _ptr(h_t), _ptr(W_t), _ptr(h_s), _ptr(W_s), _ptr(mask),
                                  _ptr(loss), _ptr(dh), _ptr(dW_s) if want_dW else None, _ptr(nnf), _ptr(ws),
                                  ws.numel(), _stream_handle(stream)))
    return KDResult(loss, dh, dW_s if want_dW else None, nnf)


def teacher_lse(h_t, W_t, mask=None, *, d_s, T=1.0, kind="fkl", chunk_tokens=0, out=None,
                stream=None, workspace=None) -> torch.Tensor:
    """kd_teacher_lse: the teacher's per-token base-2 LSE record [2, N] (M_t, log2 S_t) at temperature T.

    ``d_s`` / ``kind`` / ``chunk_tokens`` must match the student call that consumes the record (they size the
    workspace and fix the token chunking, which the record reproduces bit for bit)."""
    h_t, W_t = _as_bf16(h_t, "h_t"), _as_bf16(W_t, "W_t")
    N, d_t = h_t.shape
    V = W_t.shape[0]
    p = make_problem(N, d_t, d_s, V, T=T, kind=kind, chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=h_t.device, dtype=torch.uint8).contiguous()
    lse = out if out is not None else torch.zeros(2, N, dtype=torch.float32, device=h_t.device)
    ws = _workspace(workspace_size(p), h_t.device, stream, workspace)
    _check(lib().kd_teacher_lse(ctypes.byref(p), _ptr(h_t), _ptr(W_t), _ptr(mask), _ptr(lse), _ptr(ws), ws.numel(),
                                _stream_handle(stream)))
    return lse


def fused_fwd_bwd_lse(h_t, W_t, h_s, W_s, lse_t, mask=None, *, T=1.0, kind="fkl", beta=0.5, loss_scale=1.0,
                      want_dW=False, accumulate_dW=False, dW_s=None, chunk_tokens=0, grad_precision="split",
                      out=None, stream=None, workspace=None) -> KDResult:
    """kd_fused_fwd_bwd_lse: kd_fused_fwd_bwd with the teacher's LSE record supplied (pass 1: student head only)."""
    h_t, W_t, h_s, W_s = (_as_bf16(x, n) for x, n in ((h_t, "h_t"), (W_t, "W_t"), (h_s, "h_s"), (W_s, "W_s")))
    N, d_t = h_t.shape
    V, d_s = W_s.shape
    dev = h_t.device
    if not lse_t.is_cuda or lse_t.dtype != torch.float32 or tuple(lse_t.shape) != (2, N):
        raise ValueError("lse_t must be a CUDA float32 tensor of shape [2, N]")
    lse_t = lse_t.contiguous()
    p = make_problem(N, d_t, d_s, V, T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, chunk_tokens=chunk_tokens, grad_precision=grad_precision)
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    if out is None:
        loss = torch.empty(N, dtype=torch.float32, device=dev)
        dh = torch.empty(N, d_s, dtype=torch.float32, device=dev)
        nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        loss, dh, nnf = out.loss, out.dh_s, out.n_nonfinite
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if accumulate_dW else torch.empty)(V, d_s, dtype=torch.float32, device=dev)
    ws = _workspace(workspace_size(p), dev, stream, workspace)
    _check(lib().kd_fused_fwd_bwd_lse(ctypes.byref(p), _ptr(h_t), _ptr(W_t), _ptr(h_s), _ptr(W_s), _ptr(mask),
                                      _ptr(lse_t), _ptr(loss), _ptr(dh), _ptr(dW_s) if want_dW else None, _ptr(nnf),
                                      _ptr(ws), ws.numel(), _stream_handle(stream)))
    return KDResult(loss, dh, dW_s if want_dW else None, nnf)


def teacher_topk(h_t, W_t, mask=None, *, k, d_s, T=1.0, chunk_tokens=0, stream=None, workspace=None):
    """kd_teacher_topk: the top-k teacher baseline's transfer (idx [N, k] int32, val [N, k] float32 raw logits)."""
    h_t, W_t = _as_bf16(h_t, "h_t"), _as_bf16(W_t, "W_t")
    N, d_t = h_t.shape
    V = W_t.shape[0]
    p = make_problem(N, d_t, d_s, V, T=T, chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=h_t.device, dtype=torch.uint8).contiguous()
    idx = torch.full((N, k), -1, dtype=torch.int32, device=h_t.device)
    val = torch.zeros(N, k, dtype=torch.float32, device=h_t.device)
    ws = _workspace(workspace_size(p), h_t.device, stream, workspace)
    _check(lib().kd_teacher_topk(ctypes.byref(p), _ptr(h_t), _ptr(W_t), _ptr(mask), int(k), _ptr(idx), _ptr(val),
                                 _ptr(ws), ws.numel(), _stream_handle(stream)))
    return idx, val


def topk_fwd_bwd(h_s, W_s, topk_idx, topk_val, mask=None, *, d_t=64, T=1.0, loss_scale=1.0, want_dW=False,
                 accumulate_dW=False, dW_s=None, chunk_tokens=0, grad_precision="split", out=None,
                 stream=None, workspace=None) -> KDResult:
    """kd_topk_fwd_bwd: FKL against the renormalised top-k teacher (student head only)."""
    h_s, W_s = _as_bf16(h_s, "h_s"), _as_bf16(W_s, "W_s")
    N, d_s = h_s.shape
    V = W_s.shape[0]
    dev = h_s.device
    k = int(topk_idx.shape[1])
    if topk_idx.dtype != torch.int32 or topk_val.dtype != torch.float32 or tuple(topk_val.shape) != (N, k) \
            or tuple(topk_idx.shape) != (N, k) or not topk_idx.is_cuda or not topk_val.is_cuda:
        raise ValueError("topk_idx / topk_val must be CUDA int32 / float32 tensors of shape [N, k]")
    topk_idx, topk_val = topk_idx.contiguous(), topk_val.contiguous()
    p = make_problem(N, d_t, d_s, V, T=T, kind="fkl", loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, chunk_tokens=chunk_tokens, grad_precision=grad_precision)
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    if out is None:
        loss = torch.empty(N, dtype=torch.float32, device=dev)
        dh = torch.empty(N, d_s, dtype=torch.float32, device=dev)
        nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        loss, dh, nnf = out.loss, out.dh_s, out.n_nonfinite
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if accumulate_dW else torch.empty)(V, d_s, dtype=torch.float32, device=dev)
    ws = _workspace(workspace_size(p), dev, stream, workspace)
    _check(lib().kd_topk_fwd_bwd(ctypes.byref(p), _ptr(h_s), _ptr(W_s), _ptr(mask), k, _ptr(topk_idx),
                                 _ptr(topk_val), _ptr(loss), _ptr(dh), _ptr(dW_s) if want_dW else None, _ptr(nnf),
                                 _ptr(ws), ws.numel(), _stream_handle(stream)))
    return KDResult(loss, dh, dW_s if want_dW else None, nnf)


def vocab_stats(h_t, W_t_shard, h_s, W_s_shard, mask=None, *, vocab, v_begin, T=1.0, kind="fkl",
                chunk_tokens=0, stream=None, workspace=None) -> torch.Tensor:
    """kd_vocab_stats: this vocab shard's per-token record [5, N] (to be all-gathered)."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(x, "input") for x in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, v_begin=v_begin, v_end=v_begin + V_r,
                     chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=h_t.device, dtype=torch.uint8).contiguous()
    rec = torch.empty(5, N, dtype=torch.float32, device=h_t.device)
    ws = _workspace(workspace_size(p), h_t.device, stream, workspace)
    _check(lib().kd_vocab_stats(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                _ptr(mask), _ptr(rec), _ptr(ws), ws.numel(), _stream_handle(stream)))
    return rec


def vocab_backward(h_t, W_t_shard, h_s, W_s_shard, recs, mask=None, *, vocab, v_begin, T=1.0, kind="fkl",
                   loss_scale=1.0, want_dW=False, accumulate_dW=False, dW_s=None, chunk_tokens=0,
                   stream=None, workspace=None) -> KDResult:
    """kd_vocab_backward: merge the [P, 5, N] records; loss, PARTIAL dh_s (sum over ranks), local dW_s."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(x, "input") for x in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    dev = h_t.device
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, v_begin=v_begin, v_end=v_begin + V_r, chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    recs = recs.to(device=dev, dtype=torch.float32).contiguous()
    loss = torch.empty(N, dtype=torch.float32, device=dev)
    dh = torch.empty(N, d_s, dtype=torch.float32, device=dev)
    nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if accumulate_dW else torch.empty)(V_r, d_s, dtype=torch.float32, device=dev)
    ws = _workspace(workspace_size(p), dev, stream, workspace)
    _check(lib().kd_vocab_backward(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                   _ptr(mask), _ptr(recs), int(recs.shape[0]), _ptr(loss), _ptr(dh),
                                   _ptr(dW_s) if want_dW else None, _ptr(nnf), _ptr(ws), ws.numel(),
                                   _stream_handle(stream)))
    return KDResult(loss, dh, dW_s if want_dW else None, nnf)


# ------------------------------------------------------------------ peer-memory exchange (kd_p2p)
P2P_SETS = 3  # receive-slot sets rotated over exchange chunks (kdfused.h)


def p2p_arena_bytes(world: int, max_rows: int, max_tokens: int, d_s: int) -> int:
    n = int(lib().kd_p2p_arena_bytes(int(world), int(max_rows), int(max_tokens), int(d_s)))
    if n == 0:
        raise KDError(1, "kd_p2p_arena_bytes: invalid arguments")
    return n


def make_p2p(world: int, rank: int, d_s: int, max_rows: int, max_tokens: int, arenas) -> KDP2P:
    """A kd_p2p view: ``arenas`` = every rank's arena base address (ints) as mapped in this process."""
    x = KDP2P()
    x.world, x.rank, x.d_s, x.reserved = int(world), int(rank), int(d_s), 0
    x.max_rows, x.max_tokens = int(max_rows), int(max_tokens)
    for j, a in enumerate(arenas):
        x.arena[j] = int(a)
    return x


def p2p_outputs(x: KDP2P, device, n_tokens: int, d_s: int):
    """(dh_out [n_tokens, d_s], loss_out [n_tokens]) views of this rank's arena: valid until the next step on it, and
    only while the arena's owner (sharding.P2PExchange.own) is alive — the views do not keep it alive."""
    dh, ls = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().kd_p2p_outputs(ctypes.byref(x), ctypes.byref(dh), ctypes.byref(ls)))
    dev = torch.device(device)
    dh_t = torch.as_tensor(_DevView(dh.value, (int(x.max_tokens), d_s), "<f4"), device=dev)[:n_tokens]
    ls_t = torch.as_tensor(_DevView(ls.value, (int(x.max_tokens),), "<f4"), device=dev)[:n_tokens]
    return dh_t, ls_t


def vocab_stats_p2p(h_t, W_t_shard, h_s, W_s_shard, mask=None, *, x: KDP2P, set: int, vocab, v_begin, T=1.0,
                    kind="fkl", chunk_tokens=0, stream=None, workspace=None):
    """kd_vocab_stats_p2p: this shard's record into record set ``set`` of every rank's arena (the all-gather)."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(t, "input") for t in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, v_begin=v_begin, v_end=v_begin + V_r,
                     chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=h_t.device, dtype=torch.uint8).contiguous()
    ws = _workspace(workspace_size(p), h_t.device, stream, workspace)
    _check(lib().kd_vocab_stats_p2p(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                    _ptr(mask), _ptr(ws), ws.numel(), ctypes.byref(x), int(set),
                                    _stream_handle(stream)))


def vocab_backward_p2p(h_t, W_t_shard, h_s, W_s_shard, recs, mask=None, *, x: KDP2P, set: int, vocab, v_begin,
                       T=1.0, kind="fkl", loss_scale=1.0, want_dW=False, accumulate_dW=False, dW_s=None,
                       chunk_tokens=0, records_target: int = 0, stream=None, workspace=None) -> KDResult:
    """kd_vocab_backward_p2p: as vocab_backward, but the partial dh_s (and FKL's partial loss) rows go straight to
    their owners' receive slots of set ``set``; the result carries the local loss (RKL) and dW_s only.
    recs=None: the records kd_vocab_stats_p2p gathered into the arena (waiting for ``records_target``)."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(t, "input") for t in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    dev = h_t.device
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, v_begin=v_begin, v_end=v_begin + V_r, chunk_tokens=chunk_tokens)
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    n_ranks = x.world
    if recs is not None:
        recs = recs.to(device=dev, dtype=torch.float32).contiguous()
        n_ranks = int(recs.shape[0])
    loss = torch.empty(N, dtype=torch.float32, device=dev) if kind == "rkl" else None
    nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if accumulate_dW else torch.empty)(V_r, d_s, dtype=torch.float32, device=dev)
    ws = _workspace(workspace_size(p), dev, stream, workspace)
    _check(lib().kd_vocab_backward_p2p(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                       _ptr(mask), _ptr(recs), n_ranks, _ptr(loss),
                                       _ptr(dW_s) if want_dW else None, _ptr(nnf), _ptr(ws), ws.numel(),
                                       ctypes.byref(x), int(set), int(records_target) & 0xFFFFFFFF,
                                       _stream_handle(stream)))
    return KDResult(loss, None, dW_s if want_dW else None, nnf)


def vocab_partials_p2p(h_t, W_t_shard, h_s, W_s_shard, mask=None, *, x: KDP2P, set: int, vocab, v_begin, T=1.0,
                       kind="jsd", beta=0.5, loss_scale=1.0, want_dW=False, accumulate_dW=False,
                       records_target: int, stream=None) -> VocabFixState:
    """kd_vocab_partials_p2p: merge the arena's records of set ``set``, pass 2, (K, J) partials into every rank's
    arena.  Returns the state kd_vocab_finish_p2p needs (the problem and the workspace holding the G planes)."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(t, "input") for t in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    dev = h_t.device
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, v_begin=v_begin, v_end=v_begin + V_r, chunk_tokens=max(1, N))
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    ws = torch.empty(max(workspace_size(p), 256), dtype=torch.uint8, device=dev)  # carries the G planes to finish
    _check(lib().kd_vocab_partials_p2p(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                       _ptr(mask), _ptr(ws), ws.numel(), ctypes.byref(x), int(set),
                                       int(records_target) & 0xFFFFFFFF, _stream_handle(stream)))
    return VocabFixState(p, ws)


def vocab_finish_p2p(state, h_t, W_t_shard, h_s, W_s_shard, mask=None, *, x: KDP2P, set: int, kj_target: int,
                     dW_s=None, stream=None) -> KDResult:
    """kd_vocab_finish_p2p: (K, J) sums from the arena, loss (local), G fix-up, dW_s rows, partial dh rows to the
    owners' slots."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(t, "input") for t in (h_t, W_t_shard, h_s, W_s_shard))
    p = state.problem
    N = int(p.n_tokens)
    V_r, d_s = W_s_shard.shape
    dev = h_t.device
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    loss = torch.empty(N, dtype=torch.float32, device=dev)
    nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    want_dW = bool(p.want_dW)
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if p.accumulate_dW else torch.empty)(V_r, d_s, dtype=torch.float32, device=dev)
    _check(lib().kd_vocab_finish_p2p(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                     _ptr(mask), _ptr(loss), _ptr(dW_s) if want_dW else None, _ptr(nnf),
                                     _ptr(state.workspace), state.workspace.numel(), ctypes.byref(x), int(set),
                                     int(kj_target) & 0xFFFFFFFF, _stream_handle(stream)))
    return KDResult(loss, None, dW_s if want_dW else None, nnf)


def p2p_combine(x: KDP2P, set: int, n_rows: int, row0: int, mask=None, *, with_loss: bool, target: int,
                stream=None):
    """kd_p2p_combine: owner side of one exchange chunk (waits for the arrivals counter to reach ``target``)."""
    if mask is not None:
        mask = mask.to(dtype=torch.uint8).contiguous()
    _check(lib().kd_p2p_combine(ctypes.byref(x), int(set), int(n_rows), int(row0), _ptr(mask), int(bool(with_loss)),
                                int(target) & 0xFFFFFFFF, _stream_handle(stream)))


def p2p_wait(x: KDP2P, target: int, stream=None):
    """kd_p2p_wait: hold the stream until this rank's done counter reaches ``target``."""
    _check(lib().kd_p2p_wait(ctypes.byref(x), int(target) & 0xFFFFFFFF, _stream_handle(stream)))


@dataclass
class VocabFixState:
    """What kd_vocab_partials leaves for kd_vocab_finish: the problem and the workspace holding the chunk's
    G planes (a private buffer, so no other call can reuse it in between)."""
    problem: KDProblem
    workspace: torch.Tensor


def vocab_partials(h_t, W_t_shard, h_s, W_s_shard, recs, mask=None, *, vocab, v_begin, T=1.0, kind="jsd",
                   beta=0.5, loss_scale=1.0, want_dW=False, accumulate_dW=False, chunk_tokens=0,
                   stream=None):
    """kd_vocab_partials (JSD/TVD shards, one token chunk): -> (kj [2, N] this shard's (K, J) partials, state)."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(x, "input") for x in (h_t, W_t_shard, h_s, W_s_shard))
    N, d_t = h_t.shape
    V_r, d_s = W_s_shard.shape
    dev = h_t.device
    p = make_problem(N, d_t, d_s, vocab, T=T, kind=kind, beta=beta, loss_scale=loss_scale, want_dW=want_dW,
                     accumulate_dW=accumulate_dW, v_begin=v_begin, v_end=v_begin + V_r,
                     chunk_tokens=chunk_tokens or max(N, 1))
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    recs = recs.to(device=dev, dtype=torch.float32).contiguous()
    kj = torch.empty(2, N, dtype=torch.float32, device=dev)
    ws = torch.empty(max(workspace_size(p), 256), dtype=torch.uint8, device=dev)
    _check(lib().kd_vocab_partials(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                   _ptr(mask), _ptr(recs), int(recs.shape[0]), _ptr(kj), _ptr(ws), ws.numel(),
                                   _stream_handle(stream)))
    return kj, VocabFixState(p, ws)


def vocab_finish(state: VocabFixState, h_t, W_t_shard, h_s, W_s_shard, kj_all, mask=None, *, dW_s=None,
                 stream=None) -> KDResult:
    """kd_vocab_finish: sum the [P, 2, N] (K, J) partials in rank order; loss, PARTIAL dh_s, local dW_s."""
    h_t, W_t_shard, h_s, W_s_shard = (_as_bf16(x, "input") for x in (h_t, W_t_shard, h_s, W_s_shard))
    p = state.problem
    N, d_s = int(p.n_tokens), int(p.d_s)
    V_r = int(p.v_end - p.v_begin)
    dev = h_t.device
    if mask is not None:
        mask = mask.to(device=dev, dtype=torch.uint8).contiguous()
    kj_all = kj_all.to(device=dev, dtype=torch.float32).contiguous()
    loss = torch.empty(N, dtype=torch.float32, device=dev)
    dh = torch.empty(N, d_s, dtype=torch.float32, device=dev)
    nnf = torch.zeros(1, dtype=torch.int64, device=dev)
    want_dW = bool(p.want_dW)
    if want_dW and dW_s is None:
        dW_s = (torch.zeros if p.accumulate_dW else torch.empty)(V_r, d_s, dtype=torch.float32, device=dev)
    _check(lib().kd_vocab_finish(ctypes.byref(p), _ptr(h_t), _ptr(W_t_shard), _ptr(h_s), _ptr(W_s_shard),
                                 _ptr(mask), _ptr(kj_all), int(kj_all.shape[0]), _ptr(loss), _ptr(dh),
                                 _ptr(dW_s) if want_dW else None, _ptr(nnf), _ptr(state.workspace),
                                 state.workspace.numel(), _stream_handle(stream)))
    return KDResult(loss, dh, dW_s if want_dW else None, nnf)


def gemm_bf16_f32(A, B, *, M, N, K, a_mn_major=False, b_mn_major=False, stream=None) -> torch.Tensor:
    """kd_gemm_bf16_f32: D[M, N] = A·Bᵀ (operands bf16, fp32 accumulate in TMEM)."""
    A = _as_bf16(A, "A")
    B = _as_bf16(B, "B")
    D = torch.empty(M, N, dtype=torch.float32, device=A.device)
    _check(lib().kd_gemm_bf16_f32(_ptr(A), _ptr(B), _ptr(D), M, N, K, int(a_mn_major), int(b_mn_major),
                                  _stream_handle(stream)))
    return D


# ------------------------------------------------------------------ hidden-state hand-off
HANDOFF_HANDLE_BYTES = 96


def handoff_export(t: torch.Tensor) -> bytes:
    """kd_handoff_export: an opaque handle (bytes) through which ANOTHER process maps ``t``'s storage (CUDA IPC).
    The caller keeps ``t`` alive and unmodified until every importer has closed it."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("handoff_export needs a contiguous CUDA tensor")
    buf = ctypes.create_string_buffer(HANDOFF_HANDLE_BYTES)
    _check(lib().kd_handoff_export(_ptr(t), t.numel() * t.element_size(), buf))
    return buf.raw


class _DevView:
    """A device byte range exposed through __cuda_array_interface__ (zero-copy torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.bfloat16: "<V2", torch.float32: "<f4", torch.uint8: "|u1", torch.int32: "<i4"}


class HandoffTensor:
    """kd_handoff_open: the exporter's buffer mapped into this process; ``.tensor`` is a zero-copy view
    (reads go to the exporter's memory — over NVLink when it lives on another GPU).  ``close()`` unmaps it."""

    def __init__(self, handle: bytes, shape, dtype, device=None):
        ptr, nbytes = ctypes.c_void_p(), ctypes.c_uint64()
        _check(lib().kd_handoff_open(ctypes.create_string_buffer(handle, HANDOFF_HANDLE_BYTES), ctypes.byref(ptr),
                                     ctypes.byref(nbytes)))
        self.ptr, self.nbytes = ptr.value, int(nbytes.value)
        numel = 1
        for x in shape:
            numel *= int(x)
        esz = torch.empty((), dtype=dtype).element_size()
        if numel * esz != self.nbytes:
            self.close()
            raise ValueError(f"handle covers {self.nbytes} bytes, shape {tuple(shape)} x {esz} B does not match")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dtype == torch.bfloat16:  # __cuda_array_interface__ has no bf16: map as int16 and reinterpret
            t = torch.as_tensor(_DevView(self.ptr, shape, "<i2"), device=dev).view(torch.bfloat16)
        else:
            t = torch.as_tensor(_DevView(self.ptr, shape, _TYPESTR[dtype]), device=dev)
        self.tensor = t

    def close(self):
        if self.ptr:
            self.tensor = None
            _check(lib().kd_handoff_close(ctypes.c_void_p(self.ptr)))
            self.ptr = None
