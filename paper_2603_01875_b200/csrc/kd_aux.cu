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
  if (threadIdx.x == 0) loss[n] = 0.f;
  float4* o = reinterpret_cast<float4*>(dh + (size_t)n * d_s);
  for (int j = threadIdx.x; j < d_s / 4; j += blockDim.x) o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ A2: merge of split records
// The merge runs in fp64 (a few dozen records per token, negligible cost): one split holds S ≈ 1 and the
// others add small amounts, which fp32 would round away at the 1e-7 level p_top ≈ 1 is sensitive to.
struct Rec {
  double Mp, Mq, Sp, Sq, U;
};
__device__ __forceinline__ void rec_merge(Rec& A, const Rec& B) {
  if (B.Sp == 0.0) return;  // empty record = identity
  if (A.Sp == 0.0) { A = B; return; }
  const double Mp = fmax(A.Mp, B.Mp), Mq = fmax(A.Mq, B.Mq);
  const double dpa = Mp - A.Mp, dqa = Mq - A.Mq, dpb = Mp - B.Mp, dqb = Mq - B.Mq;
  const double fpa = exp2(-dpa), fpb = exp2(-dpb);
  Rec R;
  R.Mp = Mp;
  R.Mq = Mq;
  // explicit roundings (no FMA contraction): the p- and q-side sums stay bitwise symmetric, so equal logits
  // give exactly equal statistics (self-distillation ⇒ loss and gradient exactly 0)
  R.Sp = __dadd_rn(__dmul_rn(fpa, A.Sp), __dmul_rn(fpb, B.Sp));
  R.Sq = __dadd_rn(__dmul_rn(exp2(-dqa), A.Sq), __dmul_rn(exp2(-dqb), B.Sq));
  R.U = __dadd_rn(__dmul_rn(fpa, __dsub_rn(A.U, __dmul_rn(__dsub_rn(dpa, dqa), A.Sp))),
                  __dmul_rn(fpb, __dsub_rn(B.U, __dmul_rn(__dsub_rn(dpb, dqb), B.Sp))));
  A = R;
}

// mode 0: final statistics of the chunk's rows (fstats + FKL/RKL loss); mode 1: the merged record itself
// (vocab-shard partial, written per ORIGINAL row).  Records of row r for split s live at
// part[f*plane + s*split_stride + row], row = r (chunk-local) or the original row (orig_rows = 1).
__global__ void __launch_bounds__(256) k_merge_stats(const float* __restrict__ part, long long plane,
                                                     long long split_stride, int n_split, int n_rows, int row0,
                                                     const int* __restrict__ n_eff, int kind, int mode,
                                                     float* __restrict__ fstats, float* __restrict__ loss,
                                                     float* __restrict__ rec, long long rec_plane,
                                                     const int* __restrict__ idx, int orig_rows,
                                                     long long* __restrict__ nonfinite) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  const long long ri = orig_rows ? orow : r;
  Rec A{-INFINITY, -INFINITY, 0.0, 0.0, 0.0};
  for (int s = 0; s < n_split; ++s) {
    const size_t i = (size_t)s * split_stride + ri;
    Rec B{part[i], part[plane + i], part[2 * plane + i], part[3 * plane + i], part[4 * plane + i]};
    rec_merge(A, B);
  }
  if (mode == 1) {
    // a shard's record goes over the wire as fp32 (20 B/token); re-centre S to keep the max exact
    rec[orow] = (float)A.Mp;
    rec[rec_plane + orow] = (float)A.Mq;
    rec[2 * rec_plane + orow] = (float)(A.Sp * exp2(A.Mp - (double)(float)A.Mp));
    rec[3 * rec_plane + orow] = (float)(A.Sq * exp2(A.Mq - (double)(float)A.Mq));
    rec[4 * rec_plane + orow] = (float)A.U;
    return;
  }
  const float lp = (float)log2(A.Sp), lq = (float)log2(A.Sq);
  const float ell2 = (float)__dadd_rn(__dsub_rn(__ddiv_rn(A.U, A.Sp), log2(A.Sp)), log2(A.Sq));  // FKL / RKL, bits
  const bool rkl = kind == KIND_RKL;
  // LSE_2 = M + log2 S kept as two numbers (see kd_pass.cu, pass 2)
  fstats[r] = (float)(rkl ? A.Mq : A.Mp);        // M_t  (inputs were fp32 maxima: exact)
  fstats[n_rows + r] = rkl ? lq : lp;            // log2 S_t
  fstats[2 * n_rows + r] = (float)(rkl ? A.Mp : A.Mq);  // M_s
  fstats[3 * n_rows + r] = rkl ? lp : lq;        // log2 S_s
  fstats[4 * n_rows + r] = ell2;
  if (kind == KIND_FKL || kind == KIND_RKL) {
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
__global__ void __launch_bounds__(256) k_kfix_rows(const float* __restrict__ kpart, int n_split, int n_rows, int row0,
                                                   const int* __restrict__ n_eff, int kind, float beta,
                                                   float* __restrict__ kfin, float* __restrict__ loss,
                                                   const int* __restrict__ idx, long long* __restrict__ nonfinite) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= n_rows) return;
  if (r >= valid) { kfin[r] = 0.f; return; }
  float K = 0.f, J = 0.f;
  const size_t plane = (size_t)n_split * n_rows;
  for (int s = 0; s < n_split; ++s) {
    K += kpart[(size_t)s * n_rows + r];
    J += kpart[plane + (size_t)s * n_rows + r];
  }
  kfin[r] = K;
  float ell;
  if (kind == KIND_JSD) ell = kLn2 * (beta * J + (1.f - beta) * K);  // K, J in bits
  else ell = 0.5f * J;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  loss[orow] = ell;
  if (!isfinite(ell)) atomicAdd(reinterpret_cast<unsigned long long*>(nonfinite), 1ull);
}

// G = scale·(G_a − K_r·G_b) -> split bf16, over rows [0, rows_pad) and columns [0, g_ld)
__global__ void __launch_bounds__(256) k_kfix_apply(const float* __restrict__ ga, const float* __restrict__ gb,
                                                    const float* __restrict__ kfin, int g_ld, int n_rows, int row0,
                                                    const int* __restrict__ n_eff, float scale,
                                                    __nv_bfloat16* __restrict__ ghi, __nv_bfloat16* __restrict__ glo) {
  const int per_row4 = g_ld / 4;
  const int valid = min(n_rows, *n_eff - row0);
  const int rows_pad = valid > 0 ? min(n_rows, (valid + kBM - 1) / kBM * kBM) : 0;  // rows pass 2 wrote
  const long long total4 = (long long)rows_pad * per_row4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row4);
    const float K = kfin[r];
    const float4 a = reinterpret_cast<const float4*>(ga)[i];
    const float4 b = reinterpret_cast<const float4*>(gb)[i];
    uint32_t h0, l0, h1, l1;
    split2(scale * (a.x - K * b.x), scale * (a.y - K * b.y), h0, l0);
    split2(scale * (a.z - K * b.z), scale * (a.w - K * b.w), h1, l1);
    reinterpret_cast<uint2*>(ghi)[i] = make_uint2(h0, h1);
    reinterpret_cast<uint2*>(glo)[i] = make_uint2(l0, l1);
  }
}

// ------------------------------------------------------------------ A4r: dh split-K reduce + scatter
__global__ void __launch_bounds__(256) k_reduce_dh(const float* __restrict__ part, long long split_stride, int k_split,
                                                   int d_s, int n_rows, int row0, const int* __restrict__ n_eff,
                                                   const int* __restrict__ idx, float* __restrict__ dh) {
  const int valid = min(n_rows, *n_eff - row0);
  const int per_row4 = d_s / 4;
  const long long total4 = (long long)max(valid, 0) * per_row4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row4);
    const int j = (int)(i % per_row4);
    float4 acc = reinterpret_cast<const float4*>(part)[i];
    for (int s = 1; s < k_split; ++s) {
      const float4 b = reinterpret_cast<const float4*>(part + s * split_stride)[i];
      acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
    }
    const int orow = idx ? idx[row0 + r] : row0 + r;
    reinterpret_cast<float4*>(dh + (size_t)orow * d_s)[j] = acc;
  }
}

// ------------------------------------------------------------------ A4c: split-bf16 residual fix of dh
// dh[row] += Σ_{split, slot} r · W_s[v, :], in a fixed (split, slot) order — deterministic.
// One warp per row: the lanes scan the row's n_split·kCorrSlots slots (contiguous), then the warp applies the
// non-empty ones (typically a handful) with coalesced row FMAs.
__global__ void __launch_bounds__(256) k_corr_dh(const int* __restrict__ corr_v, const float* __restrict__ corr_r,
                                                 int n_split, int n_rows, int row0, const int* __restrict__ n_eff,
                                                 const int* __restrict__ idx, const __nv_bfloat16* __restrict__ Ws,
                                                 int d_s, float* __restrict__ dh) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int valid = min(n_rows, *n_eff - row0);
  if (r >= valid) return;
  const int orow = idx ? idx[row0 + r] : row0 + r;
  float* out = dh + (size_t)orow * d_s;
  const int nslots = n_split * kCorrSlots;
  const float* rr = corr_r + (size_t)r * nslots;
  const int* vv = corr_v + (size_t)r * nslots;
  for (int base = 0; base < nslots; base += 32) {
    const int i = base + lane;
    const float myr = i < nslots ? rr[i] : 0.f;
    unsigned live = __ballot_sync(0xffffffffu, myr != 0.f);
    while (live) {
      const int src = __ffs(live) - 1;
      live &= live - 1;
      const float coef = __shfl_sync(0xffffffffu, myr, src);
      const int v = vv[base + src];
      const __nv_bfloat16* w = Ws + (size_t)v * d_s;
      for (int j = lane; j < d_s; j += 32) out[j] = fmaf(coef, __bfloat162float(w[j]), out[j]);
    }
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_compact(const uint8_t* mask, int N, int* idx, int* n_eff, cudaStream_t s) {
  if (mask) k_compact<<<1, 1024, 0, s>>>(mask, N, idx, n_eff);
  else k_set_count<<<1, 1, 0, s>>>(n_eff, N);
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
                         long long rec_plane, const int* idx, int orig_rows, long long* nonfinite, cudaStream_t s) {
  k_merge_stats<<<(n_rows + 255) / 256, 256, 0, s>>>(part, plane, split_stride, n_split, n_rows, row0, n_eff, kind,
                                                      mode, fstats, loss, rec, rec_plane, idx, orig_rows, nonfinite);
  return cudaGetLastError();
}
cudaError_t launch_zero_records(const uint8_t* mask, int N, float* rec, long long plane, cudaStream_t s) {
  if (N > 0) k_zero_records<<<(N + 255) / 256, 256, 0, s>>>(mask, N, rec, plane);
  return cudaGetLastError();
}
cudaError_t launch_kfix(const float* kpart, int n_split, int n_rows, int row0, const int* n_eff, int kind, float beta,
                        float* kfin, float* loss, const int* idx, long long* nonfinite, const float* ga,
                        const float* gb, int g_ld, float scale, __nv_bfloat16* ghi, __nv_bfloat16* glo,
                        int num_sms, cudaStream_t s) {
  k_kfix_rows<<<(n_rows + 255) / 256, 256, 0, s>>>(kpart, n_split, n_rows, row0, n_eff, kind, beta, kfin, loss, idx,
                                                    nonfinite);
  k_kfix_apply<<<num_sms * 8, 256, 0, s>>>(ga, gb, kfin, g_ld, n_rows, row0, n_eff, scale, ghi, glo);
  return cudaGetLastError();
}
cudaError_t launch_corr_dh(const int* corr_v, const float* corr_r, int n_split, int n_rows, int row0,
                           const int* n_eff, const int* idx, const __nv_bfloat16* Ws, int d_s, float* dh, cudaStream_t s) {
  k_corr_dh<<<(n_rows + 7) / 8, 256, 0, s>>>(corr_v, corr_r, n_split, n_rows, row0, n_eff, idx, Ws, d_s, dh);
  return cudaGetLastError();
}
cudaError_t launch_reduce_dh(const float* part, long long split_stride, int k_split, int d_s, int n_rows, int row0,
                             const int* n_eff, const int* idx, float* dh, int num_sms, cudaStream_t s) {
  k_reduce_dh<<<num_sms * 8, 256, 0, s>>>(part, split_stride, k_split, d_s, n_rows, row0, n_eff, idx, dh);
  return cudaGetLastError();
}

}  // namespace kd
