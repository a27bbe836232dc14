/* kdfused.h — C ABI of the B200-native (sm_100a) fused knowledge-distillation hot path.
 *
 * What it computes (§3.2): the student receives only the teacher's final hidden
 * states H_t and "locally recomputes the full logit distributions using the teacher's language model
 * head", which "preserv[es] the mathematical equivalence to standard logit-based KD" (P:136,
 * P:266).  One call computes, for every token n with mask_n = 1,
 *
 *     Z_t = H_t · W_tᵀ ,  Z_s = H_s · W_sᵀ                       (both LM heads, fused; never stored)
 *     p = softmax(Z_t / T) , q = softmax(Z_s / T)
 *     ℓ_n = FKL Σ p ln(p/q) | RKL Σ q ln(q/p) | JSD_β β KL(p‖m)+(1−β) KL(q‖m), m = βp+(1−β)q
 *           | TVD ½ Σ |p − q|                                     (P:153 names all four)
 *     G   = loss_scale · mask_n · ∂ℓ_n/∂Z_s                          (teacher constant)
 *     dL/dh_s = G · W_s ,   dL/dW_s (+)= Gᵀ · H_s                    ("backward passes")
 *
 * The vocabulary is swept in 256-column tiles (SM-pair UMMA, 256 tokens x 256 vocab rows) with an online
 * log-sum-exp, so no [tokens × V] logit tensor exists in HBM (BASELINE.json north_star).  Definitions and the
 * readings of points the paper leaves open (no T² factor, β convention, reduction, masking) are in DESIGN.md
 * "Readings" R1-R22.
 *
 * Conventions for every entry point
 *  - All tensor pointers are DEVICE pointers (cudaMalloc / PyTorch CUDA memory), row-major, owned by
 *    the caller; the library never allocates device memory and never frees caller memory.
 *  - Every call is asynchronous on `stream` (no host synchronisation; the caller keeps inputs alive
 *    until the stream passes the call).  Invalid arguments are rejected BEFORE any launch with a
 *    non-zero kd_status; kd_last_error() then returns a thread-local message.
 *  - bf16 matrices need 16-byte aligned base pointers; hidden widths d_t, d_s must be multiples of 64.
 *  - Rows with mask = 0 are never read (NaN garbage there cannot affect any output).
 *  - Results are deterministic (fixed reduction orders, no atomics in any floating-point sum).
 */
#ifndef KDFUSED_H_
#define KDFUSED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KDFUSED_ABI_VERSION 3  /* 3: the peer-memory exchange (kd_p2p) */

typedef enum {
  KD_FKL = 0, /* forward KL  Σ p ln(p/q) */
  KD_RKL = 1, /* reverse KL  Σ q ln(q/p) */
  KD_JSD = 2, /* β-JSD, m = βp + (1−β)q, β ∈ (0,1)            (reading R4) */
  KD_TVD = 3  /* total variation ½ Σ |p − q| */
} kd_div_kind;

typedef enum {
  KD_OK = 0,
  KD_ERR_INVALID_ARG = 1,         /* T <= 0 or non-finite, β ∉ (0,1), unknown kind, NULL required ptr */
  KD_ERR_SHAPE = 2,               /* inconsistent / unsupported sizes (d % 64 != 0, empty vocab range) */
  KD_ERR_ALIGNMENT = 3,           /* a pointer is not 16-byte aligned */
  KD_ERR_UNSUPPORTED = 4,         /* valid request this build does not implement */
  KD_ERR_WORKSPACE_TOO_SMALL = 5, /* workspace_bytes < kd_workspace_size(p) or misaligned workspace */
  KD_ERR_CUDA = 6                 /* a CUDA runtime/driver call failed (message in kd_last_error) */
} kd_status;

/* Precision of the logit gradient G fed to the backward GEMMs.
 *   KD_GRAD_SPLIT_BF16 (default, parity-grade): G = hi + lo, two bf16 planes (<= 2^-16 relative) and two MMAs
 *     per product; the largest entries' exact residuals are added back (R11).
 *   KD_GRAD_BF16 (fast): one bf16 plane (<= 2^-8 relative per element; the residual fix still restores the
 *     largest entries exactly), half the backward tensor work.  NOT within the north-star gradient
 *     tolerance in general (tests/test_gpu_full.py measures it against the oracle with its own bound). */
typedef enum { KD_GRAD_SPLIT_BF16 = 0, KD_GRAD_BF16 = 1 } kd_grad_precision;

/* Problem description (plain data, no pointers). */
typedef struct {
  int64_t n_tokens;      /* N: packed token rows (ragged sequences concatenated by the caller), >= 0 */
  int32_t d_t;           /* teacher hidden width, multiple of 64 */
  int32_t d_s;           /* student hidden width, multiple of 64 */
  int64_t vocab;         /* global V (151936 for Qwen3) */
  int64_t v_begin;       /* this caller's vocabulary rows [v_begin, v_end); [0, V) on one GPU */
  int64_t v_end;
  float temperature;     /* T > 0, applied to teacher and student logits (reading R2: no T² factor) */
  int32_t kind;          /* kd_div_kind */
  float jsd_beta;        /* JSD only; in (0,1); BASELINE.json pins 0.5 */
  float loss_scale;      /* L = loss_scale · Σ_n mask_n ℓ_n; 1/max(1,Σmask) gives SPEC's mean */
  int32_t want_dW;       /* 0: skip dL/dW_s */
  int32_t accumulate_dW; /* 1: dW_s += (gradient accumulation, P:210 GA=8); 0: dW_s = */
  int32_t chunk_tokens;  /* token chunk Nc bounding the G scratch (0 = default: ~36 MiB of H_t|H_s rows, clamped to
                            [1024, 4096], so the chunk stays L2-resident; rounded up to the 256-row pair tile) */
  int32_t grad_precision;/* kd_grad_precision: how G reaches the backward GEMMs */
  int32_t stage_logits;  /* 0 (default): pass 2 recomputes both LM heads to form G — no logit ever reaches HBM.
                            1: the STAGED variant, kd_fused_fwd_bwd only: pass 1 also writes
                            its raw fp32 logit tiles of the current token chunk (2·Nc·V·4 B of workspace, one chunk at a
                            time, never the [N × V] logits of the call) and an HBM-bound kernel forms G from them —
                            no second tensor-core sweep.  Same outputs within the same tolerances (same arithmetic).
                            Other entry points return KD_ERR_UNSUPPORTED when it is set. */
  int32_t reserved[3];   /* must be zero */
} kd_problem;

/* Host-only validation of `p` (no CUDA call): the status kd_fused_fwd_bwd / kd_vocab_* would return for
 * the problem itself (pointer checks aside). */
kd_status kd_check_problem(const kd_problem* p);

/* Bytes of device workspace kd_fused_fwd_bwd needs for `p` (a pure function of p and the current
 * device's SM count).  Returns 0 if p is invalid (see kd_last_error). */
size_t kd_workspace_size(const kd_problem* p);

/* The whole hot path in one call (single GPU, or one token shard of a token-sharded job).
 *   h_t  [N, d_t]   bf16  teacher final (post-norm) hidden states
 *   W_t  [V_r, d_t] bf16  teacher LM-head rows v_begin..v_end (nn.Linear layout, reading R7)
 *   h_s  [N, d_s]   bf16  student final hidden states
 *   W_s  [V_r, d_s] bf16  student LM-head rows
 *   mask [N]        u8    1 = loss-bearing token, 0 = masked; NULL = all ones
 *   loss [N]        f32   out: per-token divergence ℓ_n in nats (0 where mask = 0)
 *   dh_s [N, d_s]   f32   out: loss_scale · mask_n · ∂ℓ_n/∂h_s[n]
 *   dW_s [V_r, d_s] f32   out (want_dW): ∂L/∂W_s (accumulated if accumulate_dW), else may be NULL
 *   n_nonfinite [1] i64   out (device): number of tokens whose ℓ_n is non-finite; may be NULL
 *   workspace            device scratch of >= kd_workspace_size(p) bytes, 256-byte aligned
 * Requires v_begin == 0 and v_end == vocab (use the kd_vocab_* entry points for vocab shards). */
kd_status kd_fused_fwd_bwd(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                           const void* W_s, const uint8_t* mask, float* loss, float* dh_s, float* dW_s,
                           int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, void* stream);

/* ---- teacher-shipped LSE (the recompute-reduced variant).  The paper's teacher
 * ships only H_t and the student recomputes everything, so pass 1 sweeps BOTH heads just to
 * learn the two log-sum-exps.  If the teacher side also ships its per-token LSE record (8 B/token next to
 * the 2·d_t B/token of H_t), the student's pass 1 sweeps the student head only: at BASELINE config 2 the
 * executed tensor work drops from 2V(2d_t+3d_s) to 2V(d_t+4d_s) flop/token (split-bf16 G).  Same results:
 * the record is the one the fused call computes for itself, so
 * kd_teacher_lse + kd_fused_fwd_bwd_lse reproduce kd_fused_fwd_bwd bit for bit for the same problem.
 *
 * kd_teacher_lse (teacher side; full vocabulary, v_begin = 0, v_end = vocab; d_s / kind are only used to size
 *   the workspace, so pass the student's problem unchanged):
 *   h_t  [N, d_t] bf16, W_t [V, d_t] bf16, mask [N] u8 or NULL (rows with mask = 0 are not written)
 *   lse_t [2][N] f32 out: lse_t[0][n] = M_t = max_v z_v·log2(e)/T, lse_t[1][n] = log2 Σ_v 2^{z_v·log2(e)/T − M_t}
 *         (the base-2 LSE of Z_t/T as two numbers; ln-LSE = ln2·(M_t + lse_t[1][n])).  Kept apart because
 *         one fp32 number (ulp 2e-6 at |LSE| ~ 30) would cancel in q − p for peaked rows.
 *   workspace >= kd_workspace_size(p).
 * kd_fused_fwd_bwd_lse: kd_fused_fwd_bwd with the teacher record `lse_t` [2][N] (as above; rows with
 *   mask = 0 are not read) supplied; pass 1 reads W_t not at all.  FKL, JSD and TVD; RKL returns
 *   KD_ERR_UNSUPPORTED (its gradient needs the RKL value, a cross term of both heads, before pass 2).
 *   Errors otherwise as kd_fused_fwd_bwd; lse_t NULL with N > 0 is KD_ERR_INVALID_ARG. */
kd_status kd_teacher_lse(const kd_problem* p, const void* h_t, const void* W_t, const uint8_t* mask, float* lse_t,
                         void* workspace, size_t workspace_bytes, void* stream);
kd_status kd_fused_fwd_bwd_lse(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                               const void* W_s, const uint8_t* mask, const float* lse_t, float* loss, float* dh_s,
                               float* dW_s, int64_t* n_nonfinite, void* workspace, size_t workspace_bytes,
                               void* stream);

/* ---- top-k teacher baseline: the prior-art transfer KDFlow replaces — "only transferring
 * the top-k logits breaks the mathematical equivalence of the loss function" (Table 1).  A
 * negative control: it measures what is lost (and what the student step costs without the teacher head).
 * Definition (SPEC, oracle/kd_topk.py): K_n = the k largest teacher logits of row n (ties: lower index
 * first, reading R17); p̂ = softmax of those k logits / T, 0 off the support; q = softmax(z_s / T) over the full
 * vocabulary; ℓ_n = FKL_topk = Σ_{v∈K_n} p̂_v ln(p̂_v / q_v); G = loss_scale·mask_n·(q − p̂)/T.
 *
 * kd_teacher_topk (teacher side; full vocabulary; d_s / kind only size the workspace):
 *   h_t [N, d_t] bf16, W_t [V, d_t] bf16, mask [N] u8 or NULL (rows with mask = 0 are not written)
 *   k in [1, min(V, 32)] (k > 32: KD_ERR_UNSUPPORTED; k < 1 or k > V: KD_ERR_INVALID_ARG)
 *   topk_idx [N, k] i32 out: vocabulary indices, by (logit desc, index asc)
 *   topk_val [N, k] f32 out: the raw teacher logits z_t = h_t·W_t[v] (fp32 tensor-core accumulation; not / T)
 * kd_topk_fwd_bwd (student side; forward KL only — RKL against a truncated teacher is +inf, KD_ERR_UNSUPPORTED):
 *   the student's own head only: h_s [N, d_s], W_s [V, d_s] (p->d_t is ignored but must be a valid width);
 *   topk_idx / topk_val as written by kd_teacher_topk (or any teacher: k distinct indices in [0, V) per row);
 *   loss, dh_s, dW_s, n_nonfinite, workspace as kd_fused_fwd_bwd.  A row holding an index outside [0, V) or a
 *   non-finite logit gets loss NaN (counted in n_nonfinite) and no teacher term in G. */
kd_status kd_teacher_topk(const kd_problem* p, const void* h_t, const void* W_t, const uint8_t* mask, int32_t k,
                          int32_t* topk_idx, float* topk_val, void* workspace, size_t workspace_bytes, void* stream);
kd_status kd_topk_fwd_bwd(const kd_problem* p, const void* h_s, const void* W_s, const uint8_t* mask, int32_t k,
                          const int32_t* topk_idx, const float* topk_val, float* loss, float* dh_s, float* dW_s,
                          int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, void* stream);

/* ---- vocabulary-sharded execution (north_star: "vocabulary sharding of W_t/W_s, with a tiny
 * all-reduce of per-token stats").  Rank r owns rows [v_begin, v_end) of both heads.
 * FKL/RKL: kd_vocab_stats -> exchange -> kd_vocab_backward.  JSD/TVD: see kd_vocab_partials below.
 *   1) kd_vocab_stats      -> rec [5][N] f32: this shard's per-token record (base-2 running maxima,
 *                              sums, and for RKL the cross term; R10), 0-filled for masked rows.
 *   2) caller all-gathers the P records into recs [P][5][N] (any transport; 20 B/token/rank).
 *   3) kd_vocab_backward   merges the P records in rank order (deterministic), writes this shard's
 *                              PARTIAL dh_s (caller all-reduces SUM over ranks), the local dW_s rows and the
 *                              loss: RKL the full ℓ_n (merged from the records' cross terms); FKL this shard's
 *                              PARTIAL Σ_{v in shard} p_v ln(p_v/q_v) with the global LSEs (caller all-reduces
 *                              SUM, with dh_s) — so FKL records need no cross term and pass 1 sweeps the two
 *                              heads decoupled.  */
kd_status kd_vocab_stats(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                         const void* W_s, const uint8_t* mask, float* rec, void* workspace,
                         size_t workspace_bytes, void* stream);
kd_status kd_vocab_backward(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                            const void* W_s, const uint8_t* mask, const float* recs, int32_t n_ranks,
                            float* loss, float* dh_s_partial, float* dW_s, int64_t* n_nonfinite,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ---- peer-memory exchange of the vocab-sharded step (the north star's "NCCL
 * all-reduce over NVLink" of the partial dh_s done by the library's own kernels over NVSwitch peer memory).
 * The partial dh_s / FKL loss rows of a shard leave the dh split-K reduction (k_reduce_dh) and the loss
 * reduction straight into the OWNING rank's receive slot — a reduce-scatter fused into the kernel that
 * produces the rows — and the owner sums the P partials in rank order (deterministic) and stores the sum
 * into every rank's output: a two-shot all-reduce, 2(P-1)/P x the chunk's bytes per rank on the wire.
 *
 * Arena (one per rank, kd_p2p_arena_bytes, device memory, 256-byte aligned, ZEROED by its owner before
 * first use; every rank maps every other rank's arena, e.g. kd_handoff_export/open = CUDA IPC over NVLink):
 *   [0, 256)   counters, one u32 per SOURCE rank t (written by rank t only): arrivals[t] at byte 4t
 *              (rank t pushed its partials of a chunk here), done[t] at byte 32 + 4t (owner t stored its
 *              sums of a chunk here), records[t] at byte 64 + 4t (rank t's record of a chunk is here),
 *              kj[t] at byte 96 + 4t (JSD/TVD: rank t's (K, J) partials of a chunk are here).
 *              A wait for chunk c needs EVERY source at c+1 (a shared sum could be satisfied by a rank
 *              running a chunk ahead).  Counters only grow (modulo 2^32, compared wrap-safe); after k
 *              exchange chunks every counter is k, so the caller's target for chunk c is base + c + 1.
 *   then       3 sets each of receive slots [world][R][d_s] f32, loss slots [world][R] f32, records
 *              [world][5][ceil4(max_rows)] f32 and (K, J) partials [world][2][ceil4(max_rows)] f32,
 *              R = ceil(max_rows / world); dh_out [max_tokens][d_s] f32; loss_out [max_tokens] f32.
 * Protocol per exchange chunk c (n_c <= max_rows tokens, rows [row0, row0 + n_c) of the step), every rank:
 *   kd_vocab_stats_p2p(set = c % 3)           its record into every rank's record set (the all-gather);
 *                                              then records[rank] of every rank += 1
 *   kd_vocab_backward_p2p(set = c % 3, recs = NULL, records_target = base + c + 1)
 *                                              waits for the P records, merges them in rank order, pushes
 *                                              its partials; then arrivals[rank] of every owner += 1
 *   kd_p2p_combine(set = c % 3, target = base + c + 1)   owner of rows [me*R_c, (me+1)*R_c) of the
 *                                              chunk (R_c = ceil(n_c / world)): waits for the P arrivals,
 *                                              sums, stores into every rank's dh_out/loss_out rows
 *                                              row0 + ..., masked rows 0; then done[rank] of every rank += 1
 *   kd_p2p_wait(done target)                  before a slot set is reused (chunk c+3 waits for
 *                                              done >= base + c + 1 from every owner) and before
 *                                              dh_out/loss_out are read (done >= base + n_chunks)
 * dh_out / loss_out hold the step's result until the owners' combines of the NEXT step rewrite them; those cannot
 * start before this rank's kd_vocab_backward_p2p of the next step, so a consumer enqueued on this rank's stream
 * before its next step is safe (on another stream: order it before the next step's calls).
 * A rank may defer kd_p2p_combine(c) behind its next chunk's kernels (sharding.py does), hiding the wait, and
 * run kd_vocab_stats_p2p(c+1) before kd_vocab_backward_p2p(c) — record set (c+1) % 3 was last read by chunk c-2,
 * whose combine (which waited for every rank's backward of c-2) this rank has already run.
 * Waits are bounded: a counter that does not arrive within ~60 s traps the kernel (the launch fails with
 * a CUDA error) instead of hanging the device.  world <= 8; all ranks pass identical problem shapes. */
#define KD_P2P_MAX_RANKS 8
typedef struct {
  int32_t world;       /* ranks of the vocab group, 1..8 */
  int32_t rank;        /* this rank's index */
  int32_t d_s;         /* student width (multiple of 4) */
  int32_t reserved;
  int64_t max_rows;    /* capacity: tokens per exchange chunk */
  int64_t max_tokens;  /* capacity of dh_out / loss_out: tokens per step */
  void* arena[KD_P2P_MAX_RANKS]; /* every rank's arena as mapped in THIS process (arena[rank]: own) */
} kd_p2p;
/* Bytes of one rank's arena; 0 for invalid arguments. */
size_t kd_p2p_arena_bytes(int32_t world, int64_t max_rows, int64_t max_tokens, int32_t d_s);
/* Device pointers of this rank's dh_out [max_tokens][d_s] and loss_out [max_tokens] inside its arena. */
kd_status kd_p2p_outputs(const kd_p2p* x, float** dh_out, float** loss_out);
/* kd_vocab_stats into the arena: this rank's record [5][n_tokens] lands in slot [rank] of record set `set` of
 * EVERY rank (written here, copied to the peers), then every rank's records counter += 1.
 * Errors: as kd_vocab_stats; KD_ERR_SHAPE if n_tokens > max_rows or d_s != x->d_s. */
kd_status kd_vocab_stats_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                             const void* W_s, const uint8_t* mask, void* workspace, size_t workspace_bytes,
                             const kd_p2p* x, int32_t set, void* stream);
/* kd_vocab_backward with the exchange: no dh_s_partial argument (the rows go to the owners' slots);
 * recs = NULL: the records of arena set `set`, after waiting for this rank's records counter to reach
 * records_target (else recs [n_ranks][5][n_tokens] as kd_vocab_backward, records_target ignored);
 * `loss`: RKL -> the full per-token loss (as kd_vocab_backward, local), FKL -> unused (NULL allowed; the
 * partial loss goes to the owners and the sum lands in loss_out).  n_ranks must equal x->world.
 * Errors: as kd_vocab_backward; KD_ERR_INVALID_ARG for a bad set / rank / world; KD_ERR_SHAPE if
 * n_tokens > max_rows or d_s != x->d_s; KD_ERR_ALIGNMENT for an arena not 256-byte aligned. */
kd_status kd_vocab_backward_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                const void* W_s, const uint8_t* mask, const float* recs, int32_t n_ranks,
                                float* loss, float* dW_s, int64_t* n_nonfinite, void* workspace,
                                size_t workspace_bytes, const kd_p2p* x, int32_t set, uint32_t records_target,
                                void* stream);
/* JSD/TVD shards with the exchange (one token chunk per call pair, as kd_vocab_partials / kd_vocab_finish):
 *   kd_vocab_partials_p2p waits for the P records of set `set` (records_target), merges them, runs pass 2 (G
 *     planes kept in `workspace`) and all-gathers this shard's (K, J) partials into every rank's arena; then
 *     kj[rank] of every rank += 1.
 *   kd_vocab_finish_p2p (same problem, inputs, workspace) waits for the P (K, J) partials (kj_target), sums them
 *     in rank order, writes the full per-token `loss` (local), the G fix-up, the local dW_s rows, and stores the
 *     partial dh_s rows into their owners' slots; then arrivals[rank] of every owner += 1.  kd_p2p_combine
 *     with with_loss = 0 follows as for FKL/RKL. */
kd_status kd_vocab_partials_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                const void* W_s, const uint8_t* mask, void* workspace, size_t workspace_bytes,
                                const kd_p2p* x, int32_t set, uint32_t records_target, void* stream);
kd_status kd_vocab_finish_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                              const void* W_s, const uint8_t* mask, float* loss, float* dW_s,
                              int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, const kd_p2p* x,
                              int32_t set, uint32_t kj_target, void* stream);
/* Owner side of exchange chunk `set`: n_rows = the chunk's tokens, row0 = its first row in dh_out,
 * mask = the chunk's mask [n_rows] or NULL, with_loss = 1 for FKL (sum the partial losses).
 * Errors: KD_ERR_SHAPE if n_rows > max_rows or row0 + n_rows > max_tokens. */
kd_status kd_p2p_combine(const kd_p2p* x, int32_t set, int64_t n_rows, int64_t row0, const uint8_t* mask,
                         int32_t with_loss, uint32_t arrivals_target, void* stream);
/* Holds `stream` until every owner's done counter in this rank's arena reaches done_target (wrap-safe). */
kd_status kd_p2p_wait(const kd_p2p* x, uint32_t done_target, void* stream);

/* ---- JSD / TVD vocab shards: one more exchange.  The JSD gradient needs the per-token
 * K = KL(q||m) = sum over the FULL vocabulary (the TVD one sum_v q*sign(q - p)), known only after every
 * shard's pass 2 (R4, R5).  Per token chunk (n_tokens <= the chunk, KD_ERR_SHAPE otherwise; the
 * caller slices the batch, see sharding.py):
 *   1) kd_vocab_stats as above over the chunk's rows; all-gather recs [P][5][n].
 *   2) kd_vocab_partials: merge (rank order) + pass 2 -> this shard's G planes (kept in `workspace`) and
 *      kj [2][n] f32 = (K, J) partial sums over this shard's vocab rows, in bits (J: the loss sum of the
 *      same shard: JSD sum p*log2(p/m), TVD sum |q - p|), 0 for masked rows.
 *   3) caller all-gathers kj into kj_all [P][2][n] (8 B/token/rank).
 *   4) kd_vocab_finish with the SAME problem, inputs and workspace (no other call on it in between): sums
 *      kj_all in rank order (deterministic), writes the loss, the G fix-up, this shard's PARTIAL dh_s
 *      (caller all-reduces SUM) and the local dW_s rows.
 * Errors: KD_ERR_UNSUPPORTED for FKL/RKL (use kd_vocab_backward); others as kd_fused_fwd_bwd. */
kd_status kd_vocab_partials(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                            const void* W_s, const uint8_t* mask, const float* recs, int32_t n_ranks,
                            float* kj, void* workspace, size_t workspace_bytes, void* stream);
kd_status kd_vocab_finish(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                          const void* W_s, const uint8_t* mask, const float* kj_all, int32_t n_ranks,
                          float* loss, float* dh_s_partial, float* dW_s, int64_t* n_nonfinite,
                          void* workspace, size_t workspace_bytes, void* stream);

/* ---- hidden-state hand-off, teacher process -> student process.  KDFlow's transfer
 * mechanism: the teacher ships only its final hidden states H_t ("transmit only the hidden states", P:131-135;
 * 2·d_t B/token instead of 2·V B/token of logits, the ~37× of P:133 at d_t = 4096, V = 151936), and the student
 * recomputes the logits with the teacher's LM head (kd_fused_fwd_bwd).  On one B200 node the two sides are
 * processes on the same or on NVLink-connected GPUs; these calls move a device buffer between them as a CUDA IPC
 * handle, so the student reads H_t in place (zero copy; over NVLink when the exporter is another GPU) or pulls
 * it into its own buffer with one device-to-device copy.
 *   kd_handoff_export: `handle` (KD_HANDOFF_HANDLE_BYTES bytes, caller-owned, any alignment) receives the IPC handle
 *     of the allocation holding [dev_ptr, dev_ptr + bytes) and dev_ptr's offset inside it (allocations made by
 *     cudaMalloc / the PyTorch caching allocator; VMM / managed memory -> KD_ERR_CUDA).  The exporting process keeps
 *     the buffer alive (and unmodified) until every importer has closed it.
 *   kd_handoff_open: maps the exported buffer into this process (another process than the exporter's) and
 *     returns the device pointer of the exported byte range and its length in *bytes; the mapping is
 *     read-write, the synchronisation of producer and consumer is the caller's (e.g. an event or a pipe).
 *   kd_handoff_close: unmaps a pointer returned by kd_handoff_open.
 * Errors: NULL arguments -> KD_ERR_INVALID_ARG (before any CUDA call); a handle not written by
 * kd_handoff_export -> KD_ERR_INVALID_ARG; CUDA failures -> KD_ERR_CUDA. */
#define KD_HANDOFF_HANDLE_BYTES 96
kd_status kd_handoff_export(const void* dev_ptr, uint64_t bytes, void* handle);
kd_status kd_handoff_open(const void* handle, void** dev_ptr, uint64_t* bytes);
kd_status kd_handoff_close(void* dev_ptr);

/* Building block exposed for verification: D[M, N] = A · Bᵀ with bf16 operands and fp32 tcgen05
 * accumulation.  A is [M, K] (a_mn_major = 0) or stored transposed as [K, M] (a_mn_major = 1); B is
 * [N, K] (b_mn_major = 0) or [K, N] (b_mn_major = 1).  D is [M, N] fp32 row-major.  M, N, K >= 1,
 * N % 32 == 0, K % 8 == 0 (K-major) / M, N % 8 == 0 (MN-major). */
kd_status kd_gemm_bf16_f32(const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                           int32_t a_mn_major, int32_t b_mn_major, void* stream);

/* Number of kernel launches the last successful call on this thread enqueued (bench bookkeeping). */
int32_t kd_last_launch_count(void);

/* Live per-kernel timing (used by bench.py for the roofline figure).  While enabled, every kernel the
 * library launches is bracketed by two CUDA events on the call's stream (negligible GPU cost).
 * kd_profile_read synchronises those events, fills launches[i] / total_ms[i] for kernel id i
 * (0 <= i < min(max_kernels, count)), clears the record and returns the number of kernel ids (or -1 if
 * an event failed).  kd_profile_kernel_name(i) names id i ("pass1", "pass2", "gemm_dh", ...). */
int32_t kd_profile_enable(int32_t on);
int32_t kd_profile_read(int32_t* launches, double* total_ms, int32_t max_kernels);
const char* kd_profile_kernel_name(int32_t id);

/* Thread-local message describing the last non-OK status (never NULL). */
const char* kd_last_error(void);

/* KDFUSED_ABI_VERSION of the loaded library. */
int32_t kd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KDFUSED_H_ */
