// kd_aux.cu — the small, HBM/latency-bound steps around the fused sweeps (sm_100a).
//
//   A0  mask compaction: idx[] of loss-bearing rows + device count n_eff; gather H rows into packed
//       buffers so masked rows are never read by the GEMMs (R9).
//   A2  merge of the per-(token, vocab split) records with the pairwise operator (R10), in a
//       fixed split order (deterministic), -> base-2 LSEs and the FKL / RKL per-token loss.
//   A3b JSD / TVD: K = Σ_v q·ℓ_v (or Σ q·s) from per-unit partials, the loss, then the elementwise fix-up
//       G = c·(G_a − K·G_b) into split-bf16 planes.
//   A4r split-K reduction of the dh GEMM partial slabs + scatter of packed rows to their original rows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

constexpr float kLn2 = 0.6931471805599453f;

// ------------------------------------------------------------------ A0: compaction (single block)
__global__ void __launch_bounds__(1024) k_compact(const uint8_t* __restrict__ mask, int N, int* __restrict__ idx,
                                                  int* __restrict__ n_eff) {
  __shared__ int warp_sums[32];
  __shared__ int carry_s;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < N; base += 1024) {
    const int i = base + tid;
    const int f = (i < N && mask[i] != 0) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 31) warp_sums[w] = pre + f;
    __syncthreads();
    if (w == 0) {
      int s = warp_sums[lane];
      int x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      warp_sums[lane] = x - s;  // exclusive
    }
    __syncthreads();
    const int carry = carry_s;
    if (f) idx[carry + warp_sums[w] + pre] = i;
    __syncthreads();
    if (tid == 1023) carry_s = carry + warp_sums[31] + pre + f;
    __syncthreads();
  }
  if (tid == 0) *n_eff = carry_s;
}

__global__ void k_set_count(int* __restrict__ n_eff, int n) { *n_eff = n; }

// packed[r] = src[idx[r]] for r < n_eff, zero rows for n_eff <= r < N (keeps the dW K-sum finite)
__global__ void __launch_bounds__(256) k_gather_rows(const __nv_bfloat16* __restrict__ src, long long src_ld,
                                                     __nv_bfloat16* __restrict__ dst, int d,
                                                     const int* __restrict__ idx, const int* __restrict__ n_eff) {
  const int r = blockIdx.x;
  const int ne = *n_eff;
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)r * d);
  const int nv = d / 8;
  if (r < ne) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)idx[r] * src_ld);
    for (int j = threadIdx.x; j < nv; j += blockDim.x) o[j] = s[j];
  } else {
    for (int j = threadIdx.x; j < nv; j += blockDim.x) o[j] = make_uint4(0, 0, 0, 0);
  }
}

// loss[n] = 0, dh[n, :] = 0 for masked rows (they are never computed)
__global__ void __launch_bounds__(256) k_zero_masked(const uint8_t* __restrict__ mask, float* __restrict__ loss,
                                                     float* __restrict__ dh, int d_s) {
  const int n = blockIdx.x;
  if (mask[n] != 0) return;
  if (threadIdx.x == 0 && loss) loss[n] = 0.f;
  if (!dh) return;  // peer exchange: the owner writes the masked rows' zeros (k_p2p_combine)
  float4* o = reinterpret_cast<float4*>(dh + (size_t)n * d_s);
  for (int j = threadIdx.x; j < d_s / 4; j += blockDim.x) o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ A2: merge of split records
// Merge of R records of one row with the pairwise operator, in its closed form: with M = max_r m_r,
//   S = Σ_r 2^{m_r − M} S_r ,   U = Σ_r 2^{m_p,r − M_p} (U_r − ((M_p − m_p,r) − (M_q − m_q,r)) S_p,r)
// (identical to folding ⊕ in record order; the oracle's kd_blockwise pins that algebra).  Factors come from
// fp32 exp2f of an exact fp32 difference — the dominant record's factor is exactly 1 — and the sums are
// accumulated in fp64 with explicit roundings (no contraction), so the p- and q-side stay bitwise symmetric
// and S ≈ 1 + Σ(small) keeps the 1e-7-level accuracy p_top ≈ 1 needs.
struct Rec {
  double Mp, Mq, Sp, Sq, U;
};
// One warp per row: lane l takes records l, l+32, ...; max and sums are combined with a fixed xor-shuffle tree
// (deterministic, and the same tree for the p- and q-side).
__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_max_f(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ Rec merge_records(const float* __restrict__ part, long long plane, long long split_stride,
                                             int n, long long ri, int lane) {
  float Mp = -INFINITY, Mq = -INFINITY;
  for (int s = lane; s < n; s += 32) {
    const size_t i = (size_t)s * split_stride + ri;
    if (part[2 * plane + i] == 0.f) continue;  // empty record = identity
    Mp = fmaxf(Mp, part[i]);
    Mq = fmaxf(Mq, part[plane + i]);
  }
  Mp = warp_max_f(Mp);
  Mq = warp_max_f(Mq);
  double Sp = 0.0, Sq = 0.0, U = 0.0;
  for (int s = lane; s < n; s += 32) {
    const size_t i = (size_t)s * split_stride + ri;
    const float sp = part[2 * plane + i];
    if (sp == 0.f) continue;
    const float dp = __fsub_rn(Mp, part[i]), dq = __fsub_rn(Mq, part[plane + i]);
    const double fp = (double)exp2f(-dp), fq = (double)exp2f(-dq);
    Sp = __dadd_rn(Sp, __dmul_rn(fp, (double)sp));
    Sq = __dadd_rn(Sq, __dmul_rn(fq, (double)part[3 * plane + i]));
    U = __dadd_rn(U, __dmul_rn(fp, __dsub_rn((double)part[4 * plane + i],
                                             __dmul_rn(__dsub_rn((double)dp, (double)dq), (double)sp))));
  }
  return Rec{Mp, Mq, warp_sum_d(Sp), warp_sum_d(Sq), warp_sum_d(U)};
}

// mode 0: final statistics of the chunk's rows (fstats [kFstatPlanes][n_rows] + FKL/RKL loss); mode 1: the merged record itself
// (vocab-shard partial, written per ORIGINAL row).  Records of row r for split s live at
// part[f*plane + s*split_stride + row], row = r (chunk-local) or the original row (orig_rows = 1).
__global__ void __launch_bounds__(256) k_merge_stats(const float* __restrict__ part, long long plane,
                                                     long long split_stride, int n_split, int n_rows, int row0,
                                                     const int* __restrict__ n_eff, int kind, int mode,
                                                     float* __restrict__ fstats, float* __restrict__ loss,
                                                     float* __restrict__ rec, long long rec_plane,
                                                     const int* __restrict__ idx, int orig_rows,
                                                     long long* __restrict__ nonfinite, int write_loss,
                                                     const float* __restrict__ tstats_in) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  const long long ri = orig_rows ? orow : r;
  const Rec A = merge_records(part, plane, split_stride, n_split, ri, lane);
  if (lane != 0) return;
  if (mode == 1) {
    // a shard's record goes over the wire as fp32 (20 B/token); re-centre S to keep the max exact
    rec[orow] = (float)A.Mp;
    rec[rec_plane + orow] = (float)A.Mq;
    rec[2 * rec_plane + orow] = (float)(A.Sp * exp2(A.Mp - (double)(float)A.Mp));
    rec[3 * rec_plane + orow] = (float)(A.Sq * exp2(A.Mq - (double)(float)A.Mq));
    rec[4 * rec_plane + orow] = (float)A.U;
    return;
  }
  if (mode == 2) {
    // kd_teacher_lse: the teacher's base-2 LSE as (M_t, log2 S_t) per ORIGINAL row — the same two fp32 numbers
    // mode 0 leaves in fstats, so a caller-supplied record reproduces the fused path exactly
    rec[orow] = (float)A.Mp;
    rec[rec_plane + orow] = (float)log2(A.Sp);
    return;
  }
  const float lp = (float)log2(A.Sp), lq = (float)log2(A.Sq);
  const double ell2d = __dadd_rn(__dsub_rn(__ddiv_rn(A.U, A.Sp), log2(A.Sp)), log2(A.Sq));  // FKL / RKL, bits
  const float ell2 = (float)ell2d;
  const bool rkl = kind == KIND_RKL;
  // LSE_2 = M + log2 S kept as two numbers (see kd_pass.cu, pass 2)
  fstats[r] = (float)(rkl ? A.Mq : A.Mp);        // M_t  (inputs were fp32 maxima: exact)
  fstats[n_rows + r] = rkl ? lq : lp;            // log2 S_t
  fstats[2 * n_rows + r] = (float)(rkl ? A.Mp : A.Mq);  // M_s
  fstats[3 * n_rows + r] = rkl ? lp : lq;        // log2 S_s
  fstats[4 * n_rows + r] = ell2;
  if (rkl) {
    // RKL's per-row gradient offset dlr = (log2 S_s − log2 S_t) + RKL (bits), with the two log2 S as the fp32 values
    // pass 2 normalises with, as an unevaluated hi + lo pair: one fp32 number would put its rounding (~1e-7 relative
    // of an RKL of several bits) on every g_v = c·q_v·(u_s − u_t − dlr) alike — a common-mode error that Σ_v g_v b_v
    // multiplies by E_q[b] (the Zipf-bias column of dh_s).  Found by tests/test_gpu_general.py at T = 0.5.
    const double dlr = __dadd_rn(__dsub_rn((double)lp, (double)lq), ell2d);  // RKL: S_p is the student's sum
    const float hi = (float)dlr;
    fstats[5 * n_rows + r] = hi;
    fstats[6 * n_rows + r] = (float)__dsub_rn(dlr, (double)hi);
  }
  if (tstats_in) {  // teacher LSE supplied by the caller (kd_fused_fwd_bwd_lse): pass 1 swept the student only
    fstats[r] = tstats_in[orow];
    fstats[n_rows + r] = tstats_in[rec_plane + orow];
  }
  if (write_loss && (kind == KIND_FKL || kind == KIND_RKL)) {
    const float ell = ell2 * kLn2;
    loss[orow] = ell;
    if (!isfinite(ell)) atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), 1ull);
  }
}

__global__ void k_zero_records(const uint8_t* __restrict__ mask, int N, float* __restrict__ rec, long long plane) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N || mask[n] != 0) return;
  for (int f = 0; f < 5; ++f) rec[f * plane + n] = 0.f;
}

// ------------------------------------------------------------------ A3b: JSD / TVD
// Per-row K (and the loss from K, J).  Local mode (kj_ranks == NULL): sum this call's per-(unit, part) partials
// kpart [2][n_split][n_rows].  Vocab-shard mode: sum the P ranks' per-token totals kj_ranks [P][2][N] (original
// row index) in rank order — the C2 exchange of SURVEY §8(e), deterministic for a fixed P.
__global__ void __launch_bounds__(256) k_kfix_rows(const float* __restrict__ kpart, int n_split, int n_rows, int row0,
                                                   const int* __restrict__ n_eff, int kind, float beta,
                                                   float* __restrict__ kfin, float* __restrict__ loss,
                                                   const int* __restrict__ idx, long long* __restrict__ nonfinite,
                                                   const float* __restrict__ kj_ranks, int n_ranks, long long N) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= n_rows) return;
  if (r >= valid) { kfin[r] = 0.f; return; }
  const int orow = idx ? idx[row0 + r] : row0 + r;
  float K = 0.f, J = 0.f;
  if (kj_ranks) {
    for (int q = 0; q < n_ranks; ++q) {
      K += kj_ranks[(size_t)q * 2 * N + orow];
      J += kj_ranks[(size_t)q * 2 * N + N + orow];
    }
  } else {
    const size_t plane = (size_t)n_split * n_rows;
    for (int s = 0; s < n_split; ++s) {
      K += kpart[(size_t)s * n_rows + r];
      J += kpart[plane + (size_t)s * n_rows + r];
    }
  }
  kfin[r] = K;
  float ell;
  if (kind == KIND_JSD) ell = kLn2 * (beta * J + (1.f - beta) * K);  // K, J in bits
  else ell = 0.5f * J;
  loss[orow] = ell;
  if (!isfinite(ell)) atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), 1ull);
}

// This shard's per-token (K, J) totals for the C2 exchange: kj [2][N] at the original row, summed over the
// call's (unit, part) partials in slot order.  Rows not visited (masked) stay as the caller zeroed them.
__global__ void __launch_bounds__(256) k_kj_rows(const float* __restrict__ kpart, int n_split, int n_rows, int row0,
                                                 const int* __restrict__ n_eff, const int* __restrict__ idx,
                                                 float* __restrict__ kj, long long N) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  float K = 0.f, J = 0.f;
  const size_t plane = (size_t)n_split * n_rows;
  for (int s = 0; s < n_split; ++s) {
    K += kpart[(size_t)s * n_rows + r];
    J += kpart[plane + (size_t)s * n_rows + r];
  }
  const int orow = idx ? idx[row0 + r] : row0 + r;
  kj[orow] = K;
  kj[N + orow] = J;
}

// G = scale·(G_a − K_r·G_b) -> split bf16, over the transposed scratch [g_ld][n_rows]: element (v, r) at v*n_rows + r,
// rows [0, rows_pad) (the rows pass 2 wrote).  n_rows % 4 == 0.
__global__ void __launch_bounds__(256) k_kfix_apply(const float* __restrict__ ga, const float* __restrict__ gb,
                                                    const float* __restrict__ kfin, int g_ld, int n_rows, int row0,
                                                    const int* __restrict__ n_eff, float scale,
                                                    __nv_bfloat16* __restrict__ ghi, __nv_bfloat16* __restrict__ glo) {
  const int valid = min(n_rows, *n_eff - row0);
  const int rows_pad = valid > 0 ? min(n_rows, (valid + 255) / 256 * 256) : 0;
  const int per_v4 = rows_pad / 4;
  const long long total4 = (long long)g_ld * per_v4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const long long v = i / per_v4;
    const int r = (int)(i % per_v4) * 4;
    const size_t e = (size_t)v * n_rows + r;
    const float4 a = *reinterpret_cast<const float4*>(ga + e);
    const float4 b = *reinterpret_cast<const float4*>(gb + e);
    const float4 K = *reinterpret_cast<const float4*>(kfin + r);
    uint32_t h0, l0, h1, l1;
    split2(scale * (a.x - K.x * b.x), scale * (a.y - K.y * b.y), h0, l0);
    split2(scale * (a.z - K.z * b.z), scale * (a.w - K.w * b.w), h1, l1);
    *reinterpret_cast<uint2*>(ghi + e) = make_uint2(h0, h1);
    if (glo) *reinterpret_cast<uint2*>(glo + e) = make_uint2(l0, l1);  // NULL: KD_GRAD_BF16
  }
}

// ------------------------------------------------------------------ A4x: extracted entries out of the dh GEMM's G
// Pass 2 (FKL/RKL) records per (row, slot) the two largest entries |g| > 2^-7 with their exact fp32 value
// (corr_v / corr_r [n_rows][n_slots]).  After the dW GEMM has read the full G, they are zeroed in both planes so the
// dh GEMM accumulates only the small entries (its truncating fp32 accumulator then never carries their large partial
// sums), and k_reduce_dh adds g·W_s[v, :] for them in fp32.  One thread per (row, slot entry); rows < n_eff only.
__global__ void __launch_bounds__(256) k_extract_zero(const int* __restrict__ corr_v, const float* __restrict__ corr_r,
                                                      int n_slots, int n_rows, int row0, const int* __restrict__ n_eff,
                                                      __nv_bfloat16* __restrict__ ghi, __nv_bfloat16* __restrict__ glo) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = (int)(i / n_slots);
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  if (corr_r[i] == 0.f) return;
  const size_t e = (size_t)corr_v[i] * n_rows + r;
  ghi[e] = __ushort_as_bfloat16((unsigned short)0);
  if (glo) glo[e] = __ushort_as_bfloat16((unsigned short)0);
}

cudaError_t launch_extract_zero(const int* corr_v, const float* corr_r, int n_slots, int n_rows, int row0,
                                const int* n_eff, __nv_bfloat16* ghi, __nv_bfloat16* glo, cudaStream_t s) {
  const long long n = (long long)n_rows * n_slots;
  if (n > 0) k_extract_zero<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(corr_v, corr_r, n_slots, n_rows, row0, n_eff,
                                                                        ghi, glo);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ A4r: dh split-K reduce + extracted entries + scatter
// One warp per (token row, 512-column block): lane j owns the float4 columns cb + 128·i + 4j, i = 0..3 (512-B warp
// runs), and the split loop is unrolled by four so a lane keeps 16 loads in flight (round 1's warp-per-row form
// reached ~2.2 TB/s, latency-bound at 14 warps per SM).
//   dh[orig(r), :] = Σ_ks part[ks][r, :]  +  Σ_{slot} g_slot · W_s[v_slot, :]
// The second sum restores the entries extracted from the dh GEMM (k_extract_zero): their exact fp32 g, added in a
// fixed (slot) order — deterministic.  corr2 (top-k baseline): exact residuals g − (hi + lo) of the support entries
// that were not extracted.  The summation order per element (splits 0..k−1, then the slots in order) is the round-1
// kernel's, so the results are unchanged bit for bit.  d_s % 4 == 0.
constexpr int kRedCols = 512;  // columns per warp
__device__ __forceinline__ void red_add_rows(float (&acc)[16], const float* __restrict__ rr, const int* __restrict__ vv,
                                             int n, const __nv_bfloat16* __restrict__ Ws, int d_s, int cb, int lane) {
  for (int base = 0; base < n; base += 32) {
    const float myr = base + lane < n ? rr[base + lane] : 0.f;
    unsigned live = __ballot_sync(0xffffffffu, myr != 0.f);
    while (live) {
      const int src = __ffs(live) - 1;
      live &= live - 1;
      const float coef = __shfl_sync(0xffffffffu, myr, src);
      const __nv_bfloat16* w = Ws + (size_t)vv[base + src] * d_s;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int col = cb + 128 * i + 4 * lane;
        if (col < d_s) {
          const uint2 q = *reinterpret_cast<const uint2*>(w + col);
          acc[4 * i + 0] = fmaf(coef, bf16lo_to_f32(q.x), acc[4 * i + 0]);
          acc[4 * i + 1] = fmaf(coef, bf16hi_to_f32(q.x), acc[4 * i + 1]);
          acc[4 * i + 2] = fmaf(coef, bf16lo_to_f32(q.y), acc[4 * i + 2]);
          acc[4 * i + 3] = fmaf(coef, bf16hi_to_f32(q.y), acc[4 * i + 3]);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_reduce_dh(const float* __restrict__ part, long long split_stride, int k_split,
                                                   int d_s, int n_rows, int row0, const int* __restrict__ n_eff,
                                                   const int* __restrict__ idx, const RowDst dst,
                                                   const int* __restrict__ corr_v, const float* __restrict__ corr_r,
                                                   int n_slots, const __nv_bfloat16* __restrict__ Ws,
                                                   const int* __restrict__ corr2_v, const float* __restrict__ corr2_r,
                                                   int n_slots2) {
  const int lane = threadIdx.x & 31;
  const int n_cb = (d_s + kRedCols - 1) / kRedCols;
  const long long w = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int r = (int)(w / n_cb);
  const int cb = (int)(w % n_cb) * kRedCols;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  float acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.f;
  const float* src = part + (size_t)r * d_s;
  int ks = 0;
  for (; ks + 4 <= k_split; ks += 4) {
    float4 x[4][4];
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int col = cb + 128 * i + 4 * lane;
        x[s][i] = col < d_s ? *reinterpret_cast<const float4*>(src + (ks + s) * split_stride + col)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[4 * i + 0] += x[s][i].x;
        acc[4 * i + 1] += x[s][i].y;
        acc[4 * i + 2] += x[s][i].z;
        acc[4 * i + 3] += x[s][i].w;
      }
  }
  for (; ks < k_split; ++ks) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int col = cb + 128 * i + 4 * lane;
      if (col < d_s) {
        const float4 a = *reinterpret_cast<const float4*>(src + ks * split_stride + col);
        acc[4 * i + 0] += a.x;
        acc[4 * i + 1] += a.y;
        acc[4 * i + 2] += a.z;
        acc[4 * i + 3] += a.w;
      }
    }
  }
  if (corr_r) red_add_rows(acc, corr_r + (size_t)r * n_slots, corr_v + (size_t)r * n_slots, n_slots, Ws, d_s, cb, lane);
  if (corr2_r)  // top-k baseline: exact residuals of the k support entries (k_topk_fix)
    red_add_rows(acc, corr2_r + (size_t)r * n_slots2, corr2_v + (size_t)r * n_slots2, n_slots2, Ws, d_s, cb, lane);
  float* out = row_dst(dst, orow);  // local dh row, or the owner's receive slot (peer exchange)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int col = cb + 128 * i + 4 * lane;
    if (col < d_s) *reinterpret_cast<float4*>(out + col) = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
  }
  if (dst.sys_fence) __threadfence_system();
}

// ------------------------------------------------------------------ SM -> L2 partition (die) probe
// One CTA per SM (the dynamic shared memory forces it); thread 0 times a dependent chase of L2-resident loads
// (ld.global.cg) on each of n_lines single lines.  A line's latency is lower from the SMs of the die whose L2
// partition homes it, so each line splits the SMs into a near and a far set; the host combines the lines into a
// die map (kd_api.cu).  Used once per device to place the fused passes' work units.
__global__ void k_die_probe(const unsigned* __restrict__ buf, const long long* __restrict__ line_off, int n_lines,
                            int steps, unsigned* __restrict__ out) {
  extern __shared__ unsigned char probe_smem[];
  if (threadIdx.x != 0) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  unsigned* o = out + (size_t)blockIdx.x * (n_lines + 1);
  o[0] = smid;
  for (int l = 0; l < n_lines; ++l) {
    const unsigned* q = buf + line_off[l];
    unsigned i = 0;
    for (int s = 0; s < 32; ++s) i = __ldcg(q + i);  // warm the line into L2 (each line holds 0: a self-loop)
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) i = __ldcg(q + i);
    const long long t1 = clock64();
    o[1 + l] = (unsigned)((t1 - t0) / steps) + (i == 0xFFFFFFFFu ? 1u : 0u);
  }
  probe_smem[0] = 0;
}

cudaError_t launch_die_probe(const unsigned* buf, const long long* line_off, int n_lines, int steps, unsigned* out,
                             int sms, int smem_bytes, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_die_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  k_die_probe<<<sms, 32, smem_bytes, s>>>(buf, line_off, n_lines, steps, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_compact(const uint8_t* mask, int N, int* idx, int* n_eff, cudaStream_t s) {
  if (mask) k_compact<<<1, 1024, 0, s>>>(mask, N, idx, n_eff);
  else k_set_count<<<1, 1, 0, s>>>(n_eff, N);
  return cudaGetLastError();
}
// ------------------------------------------------------------------ top-k teacher baseline
// (value desc, index asc) order of the candidate lists
__device__ __forceinline__ bool tk_better(float x, int xi, float y, int yi) { return x > y || (x == y && xi < yi); }

// Per row: the k best of the n_slots sorted candidate lists the top-k pass wrote (tk_val/tk_idx
// [n_slots][n_rows][kTopK]).  One warp per row: lane l folds lists l, l+32, ... into its own register top-kTopK
// (a list stops at its first non-improving entry), then k rounds of a warp arg-best pop the global order.
// Output per ORIGINAL row: out_idx [N][k] (global vocab index), out_val [N][k] (raw teacher logit).
__global__ void __launch_bounds__(256) k_topk_merge(const float* __restrict__ tk_val, const int* __restrict__ tk_idx,
                                                    int n_slots, int n_rows, int row0, const int* __restrict__ n_eff,
                                                    const int* __restrict__ idx, int k, int v_base,
                                                    int* __restrict__ out_idx, float* __restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  float tv[kTopK];
  int ti[kTopK];
#pragma unroll
  for (int j = 0; j < kTopK; ++j) { tv[j] = -INFINITY; ti[j] = 0x7fffffff; }
  for (int sl = lane; sl < n_slots; sl += 32) {
    const size_t base = ((size_t)sl * n_rows + r) * kTopK;
#pragma unroll 1
    for (int j = 0; j < kTopK; ++j) {
      float x = tk_val[base + j];
      int xi = tk_idx[base + j];
      if (!tk_better(x, xi, tv[kTopK - 1], ti[kTopK - 1])) break;  // the list is sorted: nothing further improves
#pragma unroll
      for (int t = 0; t < kTopK; ++t) {
        const bool gt = tk_better(x, xi, tv[t], ti[t]);
        const float a = tv[t];
        const int b = ti[t];
        tv[t] = gt ? x : a;
        ti[t] = gt ? xi : b;
        x = gt ? a : x;
        xi = gt ? b : xi;
      }
    }
  }
  const int orow = idx ? idx[row0 + r] : row0 + r;
  for (int j = 0; j < k; ++j) {
    float bv = tv[0];
    int bi = ti[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (tk_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) {
      out_idx[(size_t)orow * k + j] = bi == 0x7fffffff ? -1 : bi + v_base;
      out_val[(size_t)orow * k + j] = bv;
    }
    if (ti[0] == bi && tv[0] == bv) {  // the owner pops its head (indices are unique across lists)
#pragma unroll
      for (int t = 0; t < kTopK - 1; ++t) { tv[t] = tv[t + 1]; ti[t] = ti[t + 1]; }
      tv[kTopK - 1] = -INFINITY;
      ti[kTopK - 1] = 0x7fffffff;
    }
  }
}

// Student side of the top-k baseline, after its student-only pass 2 wrote G = gscale·q for every column: per row,
// put the truncated teacher back in at its k support columns,
//   p̂_j = 2^{a_j − m} / Σ_i 2^{a_i − m},  a_j = α·val_j  (renormalised over the support)
//   g_j = gscale·(q_j − p̂_j)   (split bf16 hi + lo, overwriting the pass-2 entry; stale residual slots dropped)
//   ℓ   = ln2 · Σ_j p̂_j (log2 p̂_j − log2 q_j)     (FKL_topk; q from the same base-2 LSE record as pass 2)
// with z_s at the support recomputed as an fp32 dot product h_s[n]·W_s[v] (warp per row; k·d_s MACs).
// An index outside [0, V) makes the row's loss NaN (counted in n_nonfinite) and leaves G untouched there.
__global__ void __launch_bounds__(256) k_topk_fix(const __nv_bfloat16* __restrict__ hs, const __nv_bfloat16* __restrict__ Ws,
                                                  int d_s, int V, int n_rows, int row0, const int* __restrict__ n_eff,
                                                  const int* __restrict__ idx, int k, const int* __restrict__ tk_i,
                                                  const float* __restrict__ tk_v, float alpha,
                                                  const float* __restrict__ fstats, float gscale,
                                                  __nv_bfloat16* __restrict__ ghi, __nv_bfloat16* __restrict__ glo,
                                                  int* __restrict__ corr_v, float* __restrict__ corr_r, int n_corr,
                                                  int* __restrict__ tkr_v, float* __restrict__ tkr_r,
                                                  float* __restrict__ loss, long long* __restrict__ nonfinite) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  const bool mine = lane < k;
  const int v_me = mine ? tk_i[(size_t)orow * k + lane] : -1;
  const float a_me = mine ? tk_v[(size_t)orow * k + lane] * alpha : -INFINITY;
  const bool bad = __any_sync(0xffffffffu, mine && (v_me < 0 || v_me >= V || !isfinite(a_me)));
  // z_s at the support columns
  const __nv_bfloat16* h = hs + (size_t)(row0 + r) * d_s;
  float zs_me = 0.f;
  for (int j = 0; j < k; ++j) {
    const int v = __shfl_sync(0xffffffffu, v_me, j);
    float acc = 0.f;
    if (!bad) {
      const __nv_bfloat16* w = Ws + (size_t)v * d_s;
      for (int e = lane * 8; e < d_s; e += 256) {
        const uint4 hv = *reinterpret_cast<const uint4*>(h + e);
        const uint4 wv = *reinterpret_cast<const uint4*>(w + e);
        const uint32_t hh[4] = {hv.x, hv.y, hv.z, hv.w}, ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc = fmaf(bf16lo_to_f32(hh[q]), bf16lo_to_f32(ww[q]), acc);
          acc = fmaf(bf16hi_to_f32(hh[q]), bf16hi_to_f32(ww[q]), acc);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == j) zs_me = acc;
  }
  float m = a_me;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float e_me = mine ? exp2f(a_me - m) : 0.f;
  float S = e_me;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
  const float Ms2 = fstats[2 * n_rows + r], lSs = fstats[3 * n_rows + r];
  const float ph = e_me / S;
  const float u = fmaf(zs_me, alpha, -Ms2);        // log2 q + log2 S_s
  float ell = mine ? ph * ((a_me - m - log2f(S)) - (u - lSs)) : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ell += __shfl_xor_sync(0xffffffffu, ell, o);
  ell *= kLn2;
  if (bad) ell = __int_as_float(0x7fc00000);
  // G at the support: start from the value pass 2 formed for q there (hi + lo + its exact residual, if it recorded
  // one: then bit-for-bit the fp32 gscale·q of the GEMM logits, consistent with the LSE record; the dot-product
  // logit above differs from the GEMM's by its rounding, and e^{δz} would move q_top ≈ 1 by δz itself)
  // pass 2 extracted up to two entries per (row, slot) with their exact fp32 g (k_extract_zero / k_reduce_dh): a support
  // column found there takes its value from the slot, and the slot then carries the corrected value
  __shared__ int s_slot[8][32];
  int* my_slot = s_slot[threadIdx.x >> 5];
  my_slot[lane] = -1;
  __syncwarp();
  if (!bad && corr_v) {
    const size_t cb = (size_t)r * n_corr;
    for (int base = 0; base < n_corr; base += 32) {  // warp-uniform trip count (shuffles inside)
      const int i = base + lane;
      const int cv = i < n_corr ? corr_v[cb + i] : -1;
      const float cr = i < n_corr ? corr_r[cb + i] : 0.f;
      int hit = -1;
      for (int j = 0; j < k; ++j)
        if (cv == __shfl_sync(0xffffffffu, v_me, j)) hit = j;
      if (hit >= 0 && cr != 0.f) my_slot[hit] = (int)(cb + i);  // each support column is in one slot at most
    }
  }
  __syncwarp();
  if (mine) {
    float res = 0.f;
    if (!bad) {
      const size_t e = (size_t)v_me * n_rows + r;
      const int sl = my_slot[lane];
      const float g_old = sl >= 0 ? corr_r[sl] : __bfloat162float(ghi[e]) + (glo ? __bfloat162float(glo[e]) : 0.f);
      const float g = g_old - gscale * ph;
      const uint32_t hb = pack_bf16x2(g, 0.f);
      const float lo = g - bf16lo_to_f32(hb);
      const __nv_bfloat16 lb = __float2bfloat16_rn(lo);
      ghi[e] = __ushort_as_bfloat16((unsigned short)(hb & 0xFFFFu));
      if (glo) glo[e] = lb;
      if (sl >= 0) {
        corr_r[sl] = g;  // still extracted: the dh path takes it from the slot
      } else {
        // exact residual of the stored split (k_reduce_dh adds res·W_s[v]): |g| reaches 1 at the support
        res = g - (bf16lo_to_f32(hb) + (glo ? __bfloat162float(lb) : 0.f));
      }
    }
    tkr_v[(size_t)r * k + lane] = bad ? 0 : v_me;
    tkr_r[(size_t)r * k + lane] = res;
  }
  if (lane == 0) {
    loss[orow] = ell;
    if (!isfinite(ell)) atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), 1ull);
  }
}

cudaError_t launch_topk_merge(const float* tk_val, const int* tk_idx, int n_slots, int n_rows, int row0,
                              const int* n_eff, const int* idx, int k, int v_base, int* out_idx, float* out_val,
                              cudaStream_t s) {
  k_topk_merge<<<(n_rows + 7) / 8, 256, 0, s>>>(tk_val, tk_idx, n_slots, n_rows, row0, n_eff, idx, k, v_base,
                                                 out_idx, out_val);
  return cudaGetLastError();
}
cudaError_t launch_topk_fix(const __nv_bfloat16* hs, const __nv_bfloat16* Ws, int d_s, int V, int n_rows, int row0,
                            const int* n_eff, const int* idx, int k, const int* tk_i, const float* tk_v, float alpha,
                            const float* fstats, float gscale, __nv_bfloat16* ghi, __nv_bfloat16* glo, int* corr_v,
                            float* corr_r, int n_corr, int* tkr_v, float* tkr_r, float* loss, long long* nonfinite,
                            cudaStream_t s) {
  if (d_s % 8) return cudaErrorInvalidValue;
  k_topk_fix<<<(n_rows + 7) / 8, 256, 0, s>>>(hs, Ws, d_s, V, n_rows, row0, n_eff, idx, k, tk_i, tk_v, alpha, fstats,
                                               gscale, ghi, glo, corr_v, corr_r, n_corr, tkr_v, tkr_r, loss, nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_gather(const __nv_bfloat16* src, long long src_ld, __nv_bfloat16* dst, int d, int N,
                          const int* idx, const int* n_eff, cudaStream_t s) {
  if (N > 0) k_gather_rows<<<N, 256, 0, s>>>(src, src_ld, dst, d, idx, n_eff);
  return cudaGetLastError();
}
cudaError_t launch_zero_masked(const uint8_t* mask, int N, float* loss, float* dh, int d_s, cudaStream_t s) {
  if (N > 0) k_zero_masked<<<N, 256, 0, s>>>(mask, loss, dh, d_s);
  return cudaGetLastError();
}
cudaError_t launch_merge(const float* part, long long plane, long long split_stride, int n_split, int n_rows,
                         int row0, const int* n_eff, int kind, int mode, float* fstats, float* loss, float* rec,
                         long long rec_plane, const int* idx, int orig_rows, long long* nonfinite, int write_loss,
                         cudaStream_t s, const float* tstats_in) {
  k_merge_stats<<<(n_rows + 7) / 8, 256, 0, s>>>(part, plane, split_stride, n_split, n_rows, row0, n_eff, kind,
                                                      mode, fstats, loss, rec, rec_plane, idx, orig_rows, nonfinite,
                                                      write_loss, tstats_in);
  return cudaGetLastError();
}

// FKL loss of the decoupled path: ℓ = ln2 · Σ_slots partial (each partial = Σ_v p_v (log2 p_v − log2 q_v) over one
// (vocab split, column part)), summed in fp64 in fixed slot order.
__global__ void __launch_bounds__(256) k_loss_rows(const float* __restrict__ lpart, int n_slots, int n_rows, int row0,
                                                   const int* __restrict__ n_eff, const RowDst loss,
                                                   const int* __restrict__ idx, long long* __restrict__ nonfinite) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  double acc = 0.0;
  for (int s = 0; s < n_slots; ++s) acc += (double)lpart[(size_t)s * n_rows + r];
  const float ell = (float)(acc * 0.6931471805599453);
  const int orow = idx ? idx[row0 + r] : row0 + r;
  *row_dst(loss, orow) = ell;
  if (!isfinite(ell)) atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), 1ull);
  if (loss.sys_fence) __threadfence_system();
}
cudaError_t launch_loss_rows(const float* lpart, int n_slots, int n_rows, int row0, const int* n_eff, const RowDst& loss,
                             const int* idx, long long* nonfinite, cudaStream_t s) {
  k_loss_rows<<<(n_rows + 255) / 256, 256, 0, s>>>(lpart, n_slots, n_rows, row0, n_eff, loss, idx, nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_zero_records(const uint8_t* mask, int N, float* rec, long long plane, cudaStream_t s) {
  if (N > 0) k_zero_records<<<(N + 255) / 256, 256, 0, s>>>(mask, N, rec, plane);
  return cudaGetLastError();
}
cudaError_t launch_kfix(const float* kpart, int n_split, int n_rows, int row0, const int* n_eff, int kind, float beta,
                        float* kfin, float* loss, const int* idx, long long* nonfinite, const float* ga,
                        const float* gb, int g_ld, float scale, __nv_bfloat16* ghi, __nv_bfloat16* glo,
                        int num_sms, const float* kj_ranks, int n_ranks, long long N, cudaStream_t s) {
  k_kfix_rows<<<(n_rows + 255) / 256, 256, 0, s>>>(kpart, n_split, n_rows, row0, n_eff, kind, beta, kfin, loss, idx,
                                                    nonfinite, kj_ranks, n_ranks, N);
  k_kfix_apply<<<num_sms * 8, 256, 0, s>>>(ga, gb, kfin, g_ld, n_rows, row0, n_eff, scale, ghi, glo);
  return cudaGetLastError();
}
cudaError_t launch_kj_rows(const float* kpart, int n_split, int n_rows, int row0, const int* n_eff, const int* idx,
                           float* kj, long long N, cudaStream_t s) {
  k_kj_rows<<<(n_rows + 255) / 256, 256, 0, s>>>(kpart, n_split, n_rows, row0, n_eff, idx, kj, N);
  return cudaGetLastError();
}
cudaError_t launch_reduce_dh(const float* part, long long split_stride, int k_split, int d_s, int n_rows, int row0,
                             const int* n_eff, const int* idx, const RowDst& dh, const int* corr_v,
                             const float* corr_r, int n_slots, const __nv_bfloat16* Ws, cudaStream_t s,
                             const int* corr2_v, const float* corr2_r, int n_slots2) {
  if (d_s % 4 != 0) return cudaErrorInvalidValue;
  const long long warps = (long long)n_rows * ((d_s + kRedCols - 1) / kRedCols);
  if (warps == 0) return cudaSuccess;
  k_reduce_dh<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(part, split_stride, k_split, d_s, n_rows, row0, n_eff, idx, dh, corr_v,
                                                corr_r, n_slots, Ws, corr2_v, corr2_r, n_slots2);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ peer exchange of the vocab-sharded step (§8)
// The partial dh_s / FKL loss rows of a vocab shard leave k_reduce_dh / k_loss_rows straight into the owning rank's
// receive slot (RowDst, NVLink peer memory); k_p2p_signal then raises every owner's arrival counter; k_p2p_combine
// (the owner) waits for the P arrivals, sums the P partials in rank order and stores the sum into every rank's
// output; k_p2p_signal raises every rank's done counter; k_p2p_wait holds a stream until its done counter arrives.
// Counters only grow (wrap-safe comparison); the host tracks their targets.  Every wait is bounded (~60 s, then
// __trap) so a lost peer fails the launch instead of hanging the GPU.
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ void p2p_spin_until(const unsigned* flag, unsigned target) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  while ((int)(ld_acquire_sys_u32(flag) - target) < 0) {
    __nanosleep(ns);
    if (ns < 4096) ns *= 2;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) __trap();  // a peer never arrived
  }
}

__global__ void k_p2p_signal(const P2PFlags f) {
  // stream-ordered after the kernels whose peer stores it publishes (each of their threads ended with fence.sc.sys)
  __threadfence_system();
  if (threadIdx.x < f.n) red_release_sys_add_u32(f.f[threadIdx.x], 1u);
}

// ctr[0..n): one counter per source rank; returns when every source has reached `target`
__device__ void p2p_wait_all(const unsigned* ctr, int n, unsigned target) {
  for (int t = 0; t < n; ++t) p2p_spin_until(ctr + t, target);
}

__global__ void k_p2p_wait(const unsigned* ctr, int n, unsigned target) {
  if (threadIdx.x == 0) p2p_wait_all(ctr, n, target);
}

__global__ void __launch_bounds__(256) k_p2p_combine(const P2PCombine c) {
  if (threadIdx.x == 0) p2p_wait_all(c.arrivals, c.P, c.target);
  __syncthreads();
  const long long r0 = (long long)c.me * c.R;
  const long long nr = max(0ll, min(c.n_rows, r0 + c.R) - r0);
  const int v4 = c.d_s / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long slot_stride = c.R * c.d_s;  // between source ranks
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nr * v4; e += stride) {
    const long long i = e / v4;
    const int col = (int)(e % v4) * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!c.mask || c.mask[r0 + i]) {
      const float* src = c.slots + i * c.d_s + col;
      for (int r = 0; r < c.P; ++r) {  // rank order: deterministic for a fixed P
        const float4 x = __ldcg(reinterpret_cast<const float4*>(src + r * slot_stride));
        acc.x += x.x;
        acc.y += x.y;
        acc.z += x.z;
        acc.w += x.w;
      }
    }
    for (int t = 0; t < c.P; ++t) *reinterpret_cast<float4*>(c.out[t] + (r0 + i) * c.d_s + col) = acc;
  }
  if (c.lslots) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += stride) {
      float acc = 0.f;
      if (!c.mask || c.mask[r0 + i])
        for (int r = 0; r < c.P; ++r) acc += __ldcg(c.lslots + r * c.R + i);
      for (int t = 0; t < c.P; ++t) c.lout[t][r0 + i] = acc;
    }
  }
  __threadfence_system();
}

__global__ void __launch_bounds__(256) k_p2p_copy(const P2PCopy c) {
  const long long per = (c.rows + 3) / 4;  // float4 groups per plane (plane and the slot are 16-B aligned)
  const long long total = c.planes * per;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long f = e / per, k = (e % per) * 4;
    const float* src = c.src + f * c.plane + k;
    const long long left = c.rows - k;
    if (left >= 4 && (c.plane % 4) == 0) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src));
      for (int t = 0; t < c.n_dst; ++t) *reinterpret_cast<float4*>(c.dst[t] + f * c.plane + k) = v;
    } else {
      for (long long q = 0; q < min(4ll, left); ++q) {
        const float v = __ldcg(src + q);
        for (int t = 0; t < c.n_dst; ++t) c.dst[t][f * c.plane + k + q] = v;
      }
    }
  }
  __threadfence_system();
}

cudaError_t launch_p2p_copy(const P2PCopy& c, int num_sms, cudaStream_t s) {
  const long long work = c.planes * ((c.rows + 3) / 4);
  const int blocks = (int)std::max(1ll, std::min<long long>(num_sms, (work + 255) / 256));
  k_p2p_copy<<<blocks, 256, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_p2p_signal(const P2PFlags& f, cudaStream_t s) {
  k_p2p_signal<<<1, 32, 0, s>>>(f);
  return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const unsigned* ctr, int n, unsigned target, cudaStream_t s) {
  k_p2p_wait<<<1, 32, 0, s>>>(ctr, n, target);
  return cudaGetLastError();
}
cudaError_t launch_p2p_combine(const P2PCombine& c, int num_sms, cudaStream_t s) {
  // one CTA per SM at most: the waiting CTAs must leave room for NCCL's kernels of the records exchange
  const long long nr = c.R;
  const long long work = nr * (c.d_s / 4);
  const int blocks = (int)std::max(1ll, std::min<long long>(num_sms, (work + 255) / 256));
  k_p2p_combine<<<blocks, 256, 0, s>>>(c);
  return cudaGetLastError();
}

}  // namespace kd
