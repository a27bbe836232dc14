// kd_stage.cu — the logit-gradient step of the STAGED variant.
//
// Default path: pass 2 recomputes both LM-head GEMMs (2V(d_t + d_s) flop/token) to turn the merged per-token
// LSEs into the logit gradient G.  Staged path: pass 1 also writes its raw fp32 logit tiles for the token chunk
// (Z_tᵀ, Z_sᵀ as [g_ld][Nc] planes, 8 B per (token, v) — only ONE chunk of Nc tokens exists at a time, never the
// [N × V] logits of the step), and this HBM-bound kernel produces G from them: 8 B read + 4 B written per (token, v)
// instead of a second sweep of the tensor cores.  The arithmetic is pass 2's, element for element (kd_pass.cu,
// p2chunk): same per-row constants from the merged statistics, same base-2 formulation, same split-bf16 planes,
// residual-fix slots and loss / (K, J) partials — so every downstream kernel (merge, loss rows, JSD/TVD fix-up,
// dh / dW GEMMs, reduce) is shared unchanged.
//
// Mapping: R consecutive token rows per thread, a warp = 32·R consecutive rows, so every load of a staged column
// and every store of a Gᵀ column is one contiguous run.  blockIdx.y = vocab slot s: the row's column steps
// [s·nst/S, (s+1)·nst/S) — slot s plays the role of pass 2's record slot.
#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

// R consecutive token rows per thread (R = 1, 2, 4), C vocab columns per step: every load of a staged
// column is an R-wide vector (a warp: one 128·R-byte run) and every Gᵀ store packs the R rows' bf16 (R = 4: 8 B).
// The arithmetic per element is independent of R.
template <int R>
__device__ __forceinline__ void ld_rows(const float* p, float (&v)[R]) {
  if constexpr (R == 1) {
    v[0] = __ldcs(p);
  } else if constexpr (R == 2) {
    const float2 x = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = x.x; v[1] = x.y;
  } else {
    const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
}
template <int R>
__device__ __forceinline__ void st_rows_f32(float* p, const float (&v)[R]) {
  if constexpr (R == 1) *p = v[0];
  else if constexpr (R == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  else *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
// R bf16 (packed pairs, row j in the low half of pair j/2) to consecutive addresses
template <int R>
__device__ __forceinline__ void st_rows_bf16(__nv_bfloat16* p, const uint32_t (&w)[(R + 1) / 2]) {
  if constexpr (R == 1) st_global_b16(p, (uint16_t)(w[0] & 0xFFFFu));
  else if constexpr (R == 2) *reinterpret_cast<uint32_t*>(p) = w[0];
  else *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
}

#ifndef KD_STAGE_ROWS
#define KD_STAGE_ROWS 4  // rows per thread of k_stage_grad (1, 2 or 4; A/B knob)
#endif
#ifndef KD_STAGE_COLS
#define KD_STAGE_COLS 4  // vocab columns per step (R x C elements per thread per step; A/B knob)
#endif

template <int KIND, int R>
__global__ void __launch_bounds__(128) k_stage_grad(const StageParams sp) {
  constexpr int C = KD_STAGE_COLS;  // vocab columns per step
  const int r0 = (blockIdx.x * 128 + threadIdx.x) * R;  // chunk-local rows r0 .. r0 + R - 1
  const int valid = min(sp.n_rows, *sp.n_eff - sp.row0);
  const int rows_pad = valid > 0 ? min(sp.n_rows, (valid + 255) / 256 * 256) : 0;
  if (r0 >= rows_pad) return;
  const int slot = blockIdx.y, n_slots = gridDim.y;
  const int nst = sp.g_ld / C;  // C-column steps of the scratch row
  const int c0 = (int)((long long)slot * nst / n_slots), c1 = (int)((long long)(slot + 1) * nst / n_slots);
  const float alpha = sp.alpha;
  bool row_ok[R];
  float Mt2[R], lSt[R], Ms2[R], lSs[R], iSt[R], iSs[R], dlr[R], dlr_lo[R], dlt[R];
  float2 cTS[R];
  // row totals (Kahan-compensated over steps): FKL loss L; JSD/TVD K and J
  float Ltot[R], cL[R], Ktot[R], cK[R], Jtot[R], cJ[R], cr0[R], cr1[R];
  int cv0[R], cv1[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = r0 + j;
    row_ok[j] = r < valid;
    Mt2[j] = lSt[j] = Ms2[j] = lSs[j] = dlr[j] = dlr_lo[j] = 0.f;
    iSt[j] = iSs[j] = 1.f;
    if (row_ok[j]) {
      Mt2[j] = sp.fstats[r];
      lSt[j] = sp.fstats[sp.n_rows + r];
      Ms2[j] = sp.fstats[2 * sp.n_rows + r];
      lSs[j] = sp.fstats[3 * sp.n_rows + r];
      if (KIND == KIND_RKL) {  // the RKL gradient offset as an fp64-exact hi + lo pair (k_merge_stats)
        dlr[j] = sp.fstats[5 * sp.n_rows + r];
        dlr_lo[j] = sp.fstats[6 * sp.n_rows + r];
      }
      iSt[j] = exp2f(-lSt[j]);
      iSs[j] = exp2f(-lSs[j]);
    }
    cTS[j] = make_float2(__fmul_rn(iSt[j], sp.gscale), __fmul_rn(iSs[j], sp.gscale));
    dlt[j] = lSt[j] - lSs[j];
    Ltot[j] = cL[j] = Ktot[j] = cK[j] = Jtot[j] = cJ[j] = cr0[j] = cr1[j] = 0.f;
    cv0[j] = cv1[j] = 0;
  }
  bool any_ok = false, all_ok = true;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    any_ok |= row_ok[j];
    all_ok &= row_ok[j];
  }
  const size_t plane = (size_t)sp.g_ld * sp.n_rows;
  for (int c = c0; c < c1; ++c) {
    const int v0 = c * C;
    const int nvalid = min(C, sp.V_r - v0);
    const size_t col0 = (size_t)v0 * sp.n_rows + r0;
    float zt[C][R], zs[C][R];
    float stepL[R], stepK[R], stepJ[R];  // this step's partial sums
#pragma unroll
    for (int j = 0; j < R; ++j) stepL[j] = stepK[j] = stepJ[j] = 0.f;
    if (any_ok && nvalid > 0) {
      const float* pzt = sp.zst + col0;
      const float* pzs = sp.zst + plane + col0;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        ld_rows<R>(pzt, zt[i]);
        ld_rows<R>(pzs, zs[i]);
        pzt += sp.n_rows;
        pzs += sp.n_rows;
      }
    } else {
#pragma unroll
      for (int i = 0; i < C; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) zt[i][j] = zs[i][j] = 0.f;
    }
    if (KIND == KIND_FKL || KIND == KIND_RKL) {
      const bool two = sp.g_lo != nullptr;
      // the step's gradient: every element first (no per-element control flow on the fast path)
      float g[C][R];
      float amax = 0.f;
      auto elem = [&](int i, int j, bool ok) {
        const float2 u = ffma2(make_float2(zt[i][j], zs[i][j]), make_float2(alpha, alpha),
                               make_float2(-Mt2[j], -Ms2[j]));
        const float2 e2 = make_float2(ex2(u.x), ex2(u.y));
        const float2 e = fmul2(e2, cTS[j]);  // (gscale·p, gscale·q)
        const float gi = KIND == KIND_FKL ? e.y - e.x : e.y * (((u.y - u.x) - dlr[j]) - dlr_lo[j]);
        g[i][j] = ok ? gi : 0.f;
        if (KIND == KIND_FKL) stepL[j] = fmaf(ok ? e2.x : 0.f, (u.x - u.y) - dlt[j], stepL[j]);
        amax = fmaxf(amax, fabsf(g[i][j]));
      };
      if (all_ok && nvalid == C) {  // every chunk but the vocab tail and the chunk's last rows
#pragma unroll
        for (int i = 0; i < C; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) elem(i, j, true);
      } else {
#pragma unroll
        for (int i = 0; i < C; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) elem(i, j, row_ok[j] && (i < nvalid));
      }
      // split-bf16 planes: hi = RNE(g), lo = RNE(g − hi); rows packed pairwise
      uint32_t hi[C][(R + 1) / 2], lo[C][(R + 1) / 2];
#pragma unroll
      for (int i = 0; i < C; ++i)
#pragma unroll
        for (int j = 0; j < R; j += 2) split2(g[i][j], (j + 1 < R) ? g[i][j + 1] : 0.f, hi[i][j / 2], lo[i][j / 2]);
      if (amax > kCorrThresh) {  // the two largest entries |g| > 2^-7 per (row, slot): extracted from the dh GEMM
#pragma unroll
        for (int i = 0; i < C; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const float gv = g[i][j];
            if (fabsf(gv) > kCorrThresh && fabsf(gv) > fabsf(cr1[j])) {
              if (fabsf(gv) > fabsf(cr0[j])) { cr1[j] = cr0[j]; cv1[j] = cv0[j]; cr0[j] = gv; cv0[j] = v0 + i; }
              else { cr1[j] = gv; cv1[j] = v0 + i; }
            }
          }
      }
      __nv_bfloat16* ph = sp.g_hi + col0;
      __nv_bfloat16* pl = two ? sp.g_lo + col0 : nullptr;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        st_rows_bf16<R>(ph, hi[i]);
        if (two) st_rows_bf16<R>(pl, lo[i]);
        ph += sp.n_rows;
        pl += sp.n_rows;
      }
    } else {  // JSD / TVD: the two fp32 planes (q·ℓ_v or q·sign, q) + partial (K, J), fixed up downstream
#pragma unroll
      for (int i = 0; i < C; ++i) {
        float ga[R], gb[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const float ut = fmaf(zt[i][j], alpha, -Mt2[j]), us = fmaf(zs[i][j], alpha, -Ms2[j]);
          const float pt = __fmul_rn(ex2(ut), iSt[j]), qs = __fmul_rn(ex2(us), iSs[j]);
          const float xt = ut - lSt[j];  // log2 p
          const float xs = us - lSs[j];  // log2 q
          const bool ok = row_ok[j] && (i < nvalid);
          if (KIND == KIND_JSD) {
            const float m = fmaxf(fmaf(sp.beta, pt, (1.f - sp.beta) * qs), 1.17549435e-38f);
            const float lm = lg2(m);
            ga[j] = ok ? qs * (xs - lm) : 0.f;  // q·log2(q/m)
            gb[j] = ok ? qs : 0.f;
            stepK[j] += ga[j];
            stepJ[j] += ok ? pt * (xt - lm) : 0.f;
          } else {
            const float d = qs - pt;
            const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
            ga[j] = ok ? qs * sgn : 0.f;
            gb[j] = ok ? qs : 0.f;
            stepK[j] += ga[j];
            stepJ[j] += ok ? fabsf(d) : 0.f;
          }
        }
        const size_t e = col0 + (size_t)i * sp.n_rows;
        st_rows_f32<R>(sp.g_a + e, ga);
        st_rows_f32<R>(sp.g_b + e, gb);
      }
    }
    // per-step partial sums enter the row totals Kahan-compensated (one step = C columns)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (KIND == KIND_FKL) kahan_add(Ltot[j], cL[j], stepL[j]);
      if (KIND == KIND_JSD || KIND == KIND_TVD) {
        kahan_add(Ktot[j], cK[j], stepK[j]);
        kahan_add(Jtot[j], cJ[j], stepJ[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (!row_ok[j]) continue;
    const int r = r0 + j;
    const size_t idx = (size_t)slot * sp.n_rows + r;
    if (KIND == KIND_JSD || KIND == KIND_TVD) {
      sp.kpart[idx] = Ktot[j] - cK[j];
      sp.kpart[(size_t)n_slots * sp.n_rows + idx] = Jtot[j] - cJ[j];
    } else {
      if (KIND == KIND_FKL) sp.kpart[idx] = __fmul_rn(Ltot[j] - cL[j], iSt[j]);  // FKL loss partial (bits)
      const size_t q = ((size_t)r * n_slots + slot) * kCorrSlots;
      sp.corr_v[q] = cv0[j];
      sp.corr_r[q] = cr0[j];
      sp.corr_v[q + 1] = cv1[j];
      sp.corr_r[q + 1] = cr1[j];
    }
  }
}

int stage_cols() { return KD_STAGE_COLS; }
int stage_rows() { return KD_STAGE_ROWS; }

// grid: (n_rows / (128·R)) x n_slots.
cudaError_t launch_stage_grad(int kind, const StageParams& sp, int n_slots, cudaStream_t s) {
  constexpr int R = KD_STAGE_ROWS;
  const dim3 grid((sp.n_rows + 128 * R - 1) / (128 * R), n_slots);
  switch (kind) {
    case KIND_FKL: k_stage_grad<KIND_FKL, R><<<grid, 128, 0, s>>>(sp); break;
    case KIND_RKL: k_stage_grad<KIND_RKL, R><<<grid, 128, 0, s>>>(sp); break;
    case KIND_JSD: k_stage_grad<KIND_JSD, R><<<grid, 128, 0, s>>>(sp); break;
    default: k_stage_grad<KIND_TVD, R><<<grid, 128, 0, s>>>(sp); break;
  }
  return cudaGetLastError();
}

}  // namespace kd
