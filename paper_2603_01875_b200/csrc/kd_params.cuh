// kd_params.cuh — parameter blocks shared by the kernels and the host plan (kd_api.cu).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace kd {

enum Kind : int { KIND_FKL = 0, KIND_RKL = 1, KIND_JSD = 2, KIND_TVD = 3,
                  KIND_TOPK = 4 /* kernel-internal: teacher-only pass 1 selecting the per-row top-kTopK logits */ };
constexpr int kTopK = 32;  // largest k of the top-k teacher baseline (kd_teacher_topk): per-thread register lists

constexpr int kBM = 128;        // token rows per CTA tile (one TMEM lane per token; an SM pair covers 256)
constexpr int kBK = 64;         // K per pipeline stage (one 128-byte swizzle row of bf16)
// Fused-pass epilogue: epi_parts() warps per TMEM lane quarter, each owning a contiguous part of the tile's columns.
// FKL/RKL (and every pass 1) use 3 parts (12 warps, <= 128 registers); JSD/TVD pass 2 needs more registers and uses 2.
#ifndef KD_P1_PARTS
#define KD_P1_PARTS 3  // epilogue warps per TMEM lane quarter in pass 1 (A/B knob)
#endif
__host__ __device__ constexpr int epi_parts(int pass, int kind) {
  return (pass == 2 && kind >= 2) ? 2 : (pass == 1 ? KD_P1_PARTS : 3);
}
__host__ __device__ constexpr int pass_threads(int parts) { return 128 + 32 * 4 * parts; }  // warps 0-3: TMA/MMA/alloc/idle
// Per token row, each (vocab split, column part) writes its own partial record / K-J partial / residual slots:
// "record slots" = n_split * parts, merged downstream in a fixed order.
#ifndef KD_FSTAT_PLANES
#define KD_FSTAT_PLANES 7
#endif
constexpr int kFstatPlanes = KD_FSTAT_PLANES;  // per-row final statistics planes (PassParams::fstats)
constexpr int kCorrSlots = 2;              // residual slots per (token row, vocab split)
constexpr float kCorrThresh = 7.8125e-3f;  // 2^-7: entries below it stay in the dh GEMM

// Fused dual-GEMM pass over one token chunk (rows [row0, row0 + n_rows) of the packed token list).
// Work unit = (m_tile, vocab split); split s covers vocab tiles [s*v_tiles/n_split, (s+1)*v_tiles/n_split).
struct PassParams {
  const int* n_eff;   // device: number of valid packed rows (whole call)
  int row0;           // first packed row of the chunk
  int n_rows;         // chunk capacity (multiple of kBM)
  int kb_t, kb_s;     // K blocks of the teacher / student GEMM (d/64)
  int v_tiles;        // ceil(V_r / BN), BN = the vocab tile (UMMA N) of the launch
  int V_r;            // local vocabulary rows
  int n_split;
  float alpha;        // log2(e) / T
  // pass 1 output: partial records, plane f at part + f*part_plane, index (split*parts + part)*n_rows + r
  float* part;
  long long part_plane;
  // pass 2 inputs/outputs
  const float* fstats;  // [kFstatPlanes][n_rows]: M_t, log2 S_t, M_s, log2 S_s (base-2 LSE parts of z/T),
                        // ell2 (bits), RKL only: dlr_hi, dlr_lo (the gradient's per-row offset, see k_merge_stats)
  float gscale;         // c = loss_scale / T (FKL/RKL already folded with ln2 where needed)
  float beta;           // JSD beta
  __nv_bfloat16* g_hi;  // Gᵀ: [g_ld][n_rows] (vocab-major, token rows contiguous)
  __nv_bfloat16* g_lo;  // NULL: KD_GRAD_BF16 (one plane)
  float* g_a;           // JSD/TVD: [g_ld][n_rows] fp32 planes
  float* g_b;
  int g_ld;             // vocab rows of the scratch: multiple of 64, >= V_r
  float* kpart;         // JSD/TVD: [2][n_split*parts][n_rows] per-(unit, part) partial (K, J)
  // FKL/RKL extracted entries: per (row, split·parts slot) the vocab index and exact fp32 g of the two largest
  // |g| > kCorrThresh ([n_rows][n_split*parts][kCorrSlots]; 0 = empty).  They are zeroed in G after the dW GEMM and
  // added back in fp32 by k_reduce_dh, so the dh GEMM never accumulates them
  int* corr_v;
  float* corr_r;
  float* zscr;          // decoupled pass 2: per-CTA [BN][128] fp32 staging of the teacher half-tile
  int l2_hints;         // bit 0: TMA loads of H evict_last, of W evict_first; bit 1: discard staged z_t lines;
                        // bit 3: L2 prefetch of the next vocab tile's head rows
  unsigned long long* dbg;  // KD_EPI_TIMING builds only: epilogue cycle counters (see kd_pass.cu)
  // decoupled pass 1 only: the half-tile sides swept, [side_lo, side_hi) of {0 = teacher, 1 = student}.
  // (0, 2) = both (default); (1, 2) = student only (teacher LSE supplied by the caller);
  // (0, 1) = teacher only (kd_teacher_lse).
  int side_lo, side_hi;
  // KIND_TOPK pass 1: per (record slot, row) the kTopK largest teacher logits, sorted by (value desc, index asc):
  // tk_val / tk_idx [n_split*parts][n_rows][kTopK]
  float* tk_val;
  int* tk_idx;
  // Work-unit assignment.  Units u = split·m_tiles + m_tile (token tiles of a split consecutive) are dealt to worker
  // slots: slots [0, die_w0) take units [0, die_s0·m_tiles) round-robin, slots [die_w0, n_workers) the rest.
  // die_map == NULL: slot = pair index, die_w0 = n_workers, die_s0 = n_split (plain round-robin).  Otherwise
  // (die-aware mode) die_map[smid] is the SM's L2 partition (die) and each pair claims a slot of its
  // own die from sched[die] (sched[2]: overflow onto the other die's free slots), so the token tiles that share a
  // vocab split's head rows run on one die and read them from one L2 partition.  sched: 3 ints, zero at launch.
  const uint8_t* die_map;
  int* sched;
  int die_w0, die_s0;
  // staged variant, pass 1 only: NULL = off; else the raw fp32 logits of the chunk,
  // teacher plane Z_tᵀ [g_ld][n_rows] at zst, student plane Z_sᵀ at zst + g_ld·n_rows (columns < g_ld written)
  float* zst;
};

// Destination of per-token output rows (k_reduce_dh: dh_s rows, k_loss_rows: loss).  Local form: base[0] + orow·ld
// (rows_per_owner larger than any row).  Peer-exchange form (kd_vocab_backward_p2p): row orow of the
// exchange chunk belongs to owner j = orow / rows_per_owner and is stored into owner j's receive slot
// base[j] + (src_row + orow − j·rows_per_owner)·ld, base[j] = owner j's slot set as mapped in this process (NVLink
// peer memory for j != rank); sys_fence = 1 then ends every storing thread with fence.sc.sys, so the stores are
// performed system-wide before the kernel completes and the stream's signal kernel (k_p2p_signal) raises the
// owners' arrival counters.
constexpr int kP2PMaxRanks = 8;
constexpr int kP2PSets = 3;  // receive-slot sets rotated over exchange chunks (kd_vocab_backward_p2p `set`)
struct RowDst {
  float* base[kP2PMaxRanks];
  long long rows_per_owner;
  long long src_row;
  long long ld;
  int sys_fence;
};
__host__ __device__ inline float* row_dst(const RowDst& d, long long orow) {
  const long long j = orow / d.rows_per_owner;
  return d.base[j] + (d.src_row + orow - j * d.rows_per_owner) * d.ld;
}
inline RowDst local_rows(float* base, long long ld) {
  RowDst d{};
  d.base[0] = base;
  d.rows_per_owner = 1ll << 62;
  d.src_row = 0;
  d.ld = ld;
  d.sys_fence = 0;
  return d;
}

// Owner side of the peer exchange (k_p2p_combine): the P partial rows of this owner's slice of an exchange chunk are
// summed in rank order (deterministic) and the sum is stored into every rank's output (dh_out / loss_out rows of the
// chunk, peer memory for the other ranks).
struct P2PCombine {
  const float* slots;               // this owner's slot set [P][R][d_s] (partials pushed by every rank)
  const float* lslots;              // [P][R] partial losses (FKL), or NULL
  float* out[kP2PMaxRanks];         // rank t's dh_out + row0·d_s, as mapped in this process
  float* lout[kP2PMaxRanks];        // rank t's loss_out + row0 (FKL), or NULL
  const uint8_t* mask;              // the chunk's mask [n_rows] or NULL: masked rows get 0 (never read)
  const unsigned* arrivals;         // this owner's arrival counters [P], one per source rank
  unsigned target;                  // wait until arrivals[t] - target >= 0 for every t (wrap-safe)
  int P, me, d_s;
  long long R, n_rows;              // rows per owner (ceil(n_rows / P)) and the chunk's rows
};
// kd_vocab_stats_p2p: this rank's record planes [5][plane] (rows < `rows` valid) copied into n_dst peers' slots.
// The all-gather of a per-rank block: this rank's [planes][plane] f32 block (rows < `rows` valid) copied into the same
// slot of n_dst peers' arenas (records: 5 planes, JSD/TVD (K, J): 2).
struct P2PCopy {
  const float* src;
  float* dst[kP2PMaxRanks];
  int n_dst, planes;
  long long rows, plane;
};
struct P2PFlags {
  unsigned* f[kP2PMaxRanks];        // this rank's counter slot in each destination arena (as mapped here)
  int n;
};

// Logit-gradient kernel of the staged variant (kd_stage.cu): pass 2's outputs from the staged logits.
struct StageParams {
  const int* n_eff;
  int row0, n_rows, V_r, g_ld;
  float alpha, gscale, beta;
  const float* zst;     // [2][g_ld][n_rows] (teacher plane, then student plane)
  const float* fstats;  // [kFstatPlanes][n_rows] as PassParams::fstats
  __nv_bfloat16* g_hi;
  __nv_bfloat16* g_lo;
  float* g_a;
  float* g_b;
  float* kpart;         // FKL: loss partials [n_slots][n_rows]; JSD/TVD: (K, J) [2][n_slots][n_rows]
  int* corr_v;          // FKL/RKL residual-fix slots [n_rows][n_slots][kCorrSlots]
  float* corr_r;
};

// Generic bf16 GEMM with fp32 TMEM accumulation: D[M, N] = sum_{a < NUM_A} A_a[M, K] * B[N, K]^T.
enum GemmEpi : int { EPI_STORE = 0, EPI_ACCUM = 1 };
enum DynDim : int { DYN_NONE = 0, DYN_M = 1, DYN_K = 2 };

constexpr int kGemmBN = 256;
constexpr int kGemmEpiWarps = 8;  // backward-GEMM epilogue warps: 2 per TMEM lane quarter, each half the columns
constexpr int kGemmThreads = 128 + 32 * kGemmEpiWarps;  // warps 0-3: TMA / MMA / TMEM alloc / idle

struct GemmParams {
  int M, N, K;         // static extents (the dynamic one is an upper bound)
  int dyn_dim;         // DynDim: which extent is min(cap, *dyn - dyn_base)
  const int* dyn;      // device counter (n_eff)
  int dyn_base;
  int k_split;         // split-K factor (EPI_STORE writes partial slabs)
  int kb_per_acc;      // K blocks per TMEM accumulator before it is flushed (fp32 "promotion"); see kd_gemm.cu
  float* out;          // fp32
  long long out_ld;    // row stride (elements)
  long long out_split_stride;  // elements between split-K slabs
};

}  // namespace kd
