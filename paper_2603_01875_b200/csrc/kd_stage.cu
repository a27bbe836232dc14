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
// Mapping: one thread per token row, a warp = 32 consecutive rows, so every load of a staged column and every
// store of a Gᵀ column is one contiguous run (128 B / 64 B per warp instruction).  blockIdx.y = vocab slot s:
// the row's 32-column chunks [s·nch/S, (s+1)·nch/S) — slot s plays the role of pass 2's record slot.
#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

template <int KIND>
__global__ void __launch_bounds__(128) k_stage_grad(const StageParams sp) {
  const int r = blockIdx.x * 128 + threadIdx.x;  // chunk-local row
  const int valid = min(sp.n_rows, *sp.n_eff - sp.row0);
  const int rows_pad = valid > 0 ? min(sp.n_rows, (valid + 255) / 256 * 256) : 0;
  if (r >= rows_pad) return;
  const bool row_ok = r < valid;
  const int slot = blockIdx.y, n_slots = gridDim.y;
  const int nch = sp.g_ld / 32;
  const int c0 = (int)((long long)slot * nch / n_slots), c1 = (int)((long long)(slot + 1) * nch / n_slots);
  const float alpha = sp.alpha;
  float Mt2 = 0.f, lSt = 0.f, Ms2 = 0.f, lSs = 0.f, ell2 = 0.f, iSt = 1.f, iSs = 1.f;
  if (row_ok) {
    Mt2 = sp.fstats[r];
    lSt = sp.fstats[sp.n_rows + r];
    Ms2 = sp.fstats[2 * sp.n_rows + r];
    lSs = sp.fstats[3 * sp.n_rows + r];
    ell2 = sp.fstats[4 * sp.n_rows + r];
    iSt = exp2f(-lSt);
    iSs = exp2f(-lSs);
  }
  const float2 negM2 = make_float2(-Mt2, -Ms2);
  const float2 cTS = make_float2(__fmul_rn(iSt, sp.gscale), __fmul_rn(iSs, sp.gscale));
  const float dlr = (lSs - lSt) + ell2;
  const float dlt = lSt - lSs;
  float Lacc = 0.f, cL = 0.f, Kacc = 0.f, cK = 0.f, Jacc = 0.f, cJ = 0.f;
  float cr0 = 0.f, cr1 = 0.f;
  int cv0 = 0, cv1 = 0;
  const size_t plane = (size_t)sp.g_ld * sp.n_rows;
  for (int c = c0; c < c1; ++c) {
    const int v0 = c * 32;
    const int nvalid = min(32, sp.V_r - v0);
    const size_t col0 = (size_t)v0 * sp.n_rows + r;
    float zt[32], zs[32];
    if (row_ok && nvalid > 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        zt[i] = __ldcs(sp.zst + col0 + (size_t)i * sp.n_rows);
        zs[i] = __ldcs(sp.zst + plane + col0 + (size_t)i * sp.n_rows);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) zt[i] = zs[i] = 0.f;
    }
    if (KIND == KIND_FKL || KIND == KIND_RKL) {
      float g[32];
      float la = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const bool ok = row_ok && (i < nvalid);
        const float2 u = ffma2(make_float2(zt[i], zs[i]), make_float2(alpha, alpha), negM2);
        const float2 e2 = make_float2(ex2(u.x), ex2(u.y));
        const float2 e = fmul2(e2, cTS);  // (gscale·p, gscale·q)
        const float gi = KIND == KIND_FKL ? e.y - e.x : e.y * ((u.y - u.x) - dlr);
        g[i] = ok ? gi : 0.f;
        if (KIND == KIND_FKL && ok) la = fmaf(e2.x, (u.x - u.y) - dlt, la);
      }
      if (KIND == KIND_FKL) kahan_add(Lacc, cL, la);
      uint32_t hi[16], lo[16];
      const bool two = sp.g_lo != nullptr;
#pragma unroll
      for (int i = 0; i < 16; ++i) split2(g[2 * i], g[2 * i + 1], hi[i], lo[i]);
      float amax = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(g[i]));
      if (amax > kCorrThresh) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float gv = g[2 * i + h];
            if (fabsf(gv) > kCorrThresh) {
              const float rep = h ? bf16hi_to_f32(hi[i]) + (two ? bf16hi_to_f32(lo[i]) : 0.f)
                                  : bf16lo_to_f32(hi[i]) + (two ? bf16lo_to_f32(lo[i]) : 0.f);
              const float rr = gv - rep;
              if (fabsf(rr) > fabsf(cr1)) {
                if (fabsf(rr) > fabsf(cr0)) { cr1 = cr0; cv1 = cv0; cr0 = rr; cv0 = v0 + 2 * i + h; }
                else { cr1 = rr; cv1 = v0 + 2 * i + h; }
              }
            }
          }
        }
      }
      __nv_bfloat16* ph = sp.g_hi + col0;
      __nv_bfloat16* pl = two ? sp.g_lo + col0 : nullptr;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        st_global_b16(ph, (uint16_t)(hi[i] & 0xFFFFu));
        st_global_b16(ph + sp.n_rows, (uint16_t)(hi[i] >> 16));
        ph += 2 * (size_t)sp.n_rows;
        if (two) {
          st_global_b16(pl, (uint16_t)(lo[i] & 0xFFFFu));
          st_global_b16(pl + sp.n_rows, (uint16_t)(lo[i] >> 16));
          pl += 2 * (size_t)sp.n_rows;
        }
      }
    } else {  // JSD / TVD: the two fp32 planes (q·ℓ_v or q·sign, q) + partial (K, J), fixed up downstream
      float kk = 0.f, jj = 0.f;
      float* pa = sp.g_a + col0;
      float* pb = sp.g_b + col0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float ut = fmaf(zt[i], alpha, -Mt2), us = fmaf(zs[i], alpha, -Ms2);
        const float pt = __fmul_rn(ex2(ut), iSt), qs = __fmul_rn(ex2(us), iSs);
        const float xt = ut - lSt;  // log2 p
        const float xs = us - lSs;  // log2 q
        const bool ok = row_ok && (i < nvalid);
        float ga, gb;
        if (KIND == KIND_JSD) {
          const float m = fmaxf(fmaf(sp.beta, pt, (1.f - sp.beta) * qs), 1.17549435e-38f);
          const float lm = lg2(m);
          const float a = qs * (xs - lm);  // q·log2(q/m)
          ga = ok ? a : 0.f;
          gb = ok ? qs : 0.f;
          kk += ga;
          jj += ok ? pt * (xt - lm) : 0.f;
        } else {
          const float d = qs - pt;
          const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
          ga = ok ? qs * sgn : 0.f;
          gb = ok ? qs : 0.f;
          kk += ga;
          jj += ok ? fabsf(d) : 0.f;
        }
        pa[(size_t)i * sp.n_rows] = ga;
        pb[(size_t)i * sp.n_rows] = gb;
      }
      kahan_add(Kacc, cK, kk);
      kahan_add(Jacc, cJ, jj);
    }
  }
  if (!row_ok) return;
  const size_t idx = (size_t)slot * sp.n_rows + r;
  if (KIND == KIND_JSD || KIND == KIND_TVD) {
    sp.kpart[idx] = Kacc - cK;
    sp.kpart[(size_t)n_slots * sp.n_rows + idx] = Jacc - cJ;
  } else {
    if (KIND == KIND_FKL) sp.kpart[idx] = __fmul_rn(Lacc - cL, iSt);  // FKL loss partial (bits)
    const size_t q = ((size_t)r * n_slots + slot) * kCorrSlots;
    sp.corr_v[q] = cv0;
    sp.corr_r[q] = cr0;
    sp.corr_v[q + 1] = cv1;
    sp.corr_r[q + 1] = cr1;
  }
}

// grid: (n_rows / 128) x n_slots (n_rows is a multiple of 128).
cudaError_t launch_stage_grad(int kind, const StageParams& sp, int n_slots, cudaStream_t s) {
  const dim3 grid(sp.n_rows / 128, n_slots);
  switch (kind) {
    case KIND_FKL: k_stage_grad<KIND_FKL><<<grid, 128, 0, s>>>(sp); break;
    case KIND_RKL: k_stage_grad<KIND_RKL><<<grid, 128, 0, s>>>(sp); break;
    case KIND_JSD: k_stage_grad<KIND_JSD><<<grid, 128, 0, s>>>(sp); break;
    default: k_stage_grad<KIND_TVD><<<grid, 128, 0, s>>>(sp); break;
  }
  return cudaGetLastError();
}

}  // namespace kd
