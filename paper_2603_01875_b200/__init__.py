"""paper_2603_01875_b200 — B200-native (sm_100a) fused KD hot path of KDFlow (arxiv 2603.01875).

The student-side recompute of the teacher's full-vocabulary logits from transferred hidden states,
the FKL / RKL / JSD / TVD divergence against the student's logits, and its gradient into dL/dh_s and
dL/dW_s — hand-written tcgen05/TMA kernels behind the C ABI in ``include/kdfused.h``.
"""
from .kdfused import (HandoffTensor, KDError, KDP2P, KDProblem, KDResult, VocabFixState, fused_fwd_bwd, handoff_export, fused_fwd_bwd_lse, gemm_bf16_f32,
                      last_launch_count, lib, make_problem, profile_enable, profile_read, vocab_backward,
                      teacher_lse, teacher_topk, topk_fwd_bwd, vocab_finish, vocab_partials, vocab_stats, workspace_size)

__all__ = ["HandoffTensor", "KDP2P", "handoff_export", "KDError", "KDProblem", "KDResult", "VocabFixState", "fused_fwd_bwd", "fused_fwd_bwd_lse", "gemm_bf16_f32",
           "last_launch_count", "lib", "make_problem", "profile_enable", "profile_read", "vocab_backward",
           "teacher_lse", "teacher_topk", "topk_fwd_bwd", "vocab_finish", "vocab_partials", "vocab_stats", "workspace_size"]
