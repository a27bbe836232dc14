"""CPU oracle for the KDFlow student-side hot path (arxiv 2603.01875).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2603_01875_b200``) never imports it
and shares no code with it: the two meet only at the seeded input generator
``kd_inputs`` (which holds none of the method's arithmetic).

Contents
--------
``kd_oracle``    the plain definition, fp64 numpy: dense LM-head logits,
                 temperature log-softmax, FKL / RKL / JSD / TVD, analytic
                 gradient w.r.t. the student logits, and the fused
                 ``kd_fused_fwd_bwd`` composition (loss, dL/dh_s, dL/dW_s).
``kd_blockwise`` the second, vocabulary-chunked formulation (online
                 log-sum-exp records + the pairwise merge operator,
                 simulated vocab shards).  It is NOT used as the reference;
                 tests pin it to ``kd_oracle`` (<= 1e-12) so that the merge
                 algebra the multi-GPU exchange relies on is checked on CPU.
``kd_topk``      the prior-art top-k teacher transfer (SURVEY §8(f) NEXT-3,
                 SPEC S:267-275 kd_loss_topk): teacher top-k selection, the
                 renormalised truncated teacher p̂, FKL against the full
                 student softmax and its student-side composition — the
                 negative control for P:37 / P:130.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n
(SPEC is an interface donor only).  Readings of silent/garbled points are
listed in DESIGN.md section "Readings".
"""
