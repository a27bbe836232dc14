// kd_pass.cu — the fused vocabulary sweeps of the KD hot path (sm_100a).
//
// One persistent CTA per SM.  Per (128-token tile, 128-vocab tile) the CTA computes BOTH LM-head
// logit tiles with tcgen05 tensor-core MMAs into TMEM:
//     Z_t = H_t · W_tᵀ   (K = d_t)   and   Z_s = H_s · W_sᵀ   (K = d_s)
// ("recomputes the full logit distributions using the teacher's language model head";
//  the student's own LM head is fused the same way), and an epilogue consumes them straight from TMEM,
// so the [tokens × V] logits never reach HBM (BASELINE.json north_star).
//
//   pass 1 (PASS == 1): online base-2 log-sum-exp statistics per token over the unit's vocab range:
//       record (M_p, M_q, S_p, S_q, U) with u = α z_p, w = α z_q, α = log2(e)/T,
//       S_p = Σ 2^{u−M_p}, S_q = Σ 2^{w−M_q}, U = Σ 2^{u−M_p}((u−M_p) − (w−M_q)),
//       (p, q) = (teacher, student) for FKL / JSD / TVD and (student, teacher) for RKL.
//   pass 2 (PASS == 2): with the merged LSEs, the logit gradient g = ∂ℓ/∂z_s · loss_scale (R5)
//       FKL/RKL: written as a split-bf16 (hi + lo) pair for the backward GEMMs;
//       JSD/TVD: written as the two fp32 planes (q·ℓ_v, q) plus per-unit partial K, fixed up later.
//
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warps 4..7 = epilogue (thread i of warp 4+j owns token row 32j + i = TMEM lane 32j + i).
// TMEM: 2 accumulator buffers × (teacher 128 cols + student 128 cols) = 512 columns.
#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

constexpr int kTileBytes = kBM * kBK * 2;  // 16 KB: one 128x64 bf16 tile (A or B)
constexpr int kStageBytes = 2 * kTileBytes;
constexpr int kPassSmem = kPassStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct UnitRange {
  int m_tile, vt0, vt1;
};
__device__ __forceinline__ UnitRange unit_range(int u, int m_tiles, int n_split, int v_tiles) {
  UnitRange r;
  r.m_tile = u % m_tiles;
  const int s = u / m_tiles;
  r.vt0 = (int)((long long)s * v_tiles / n_split);
  r.vt1 = (int)((long long)(s + 1) * v_tiles / n_split);
  return r;
}

template <int PASS, int KIND>
__global__ void __launch_bounds__(kPassThreads, 1)
    kd_pass_kernel(const __grid_constant__ CUtensorMap tm_ht, const __grid_constant__ CUtensorMap tm_wt,
                   const __grid_constant__ CUtensorMap tm_hs, const __grid_constant__ CUtensorMap tm_ws,
                   const PassParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kPassStages * kTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kPassStages * kTileBytes);
  uint64_t* empty = full + kPassStages;
  uint64_t* tfull = empty + kPassStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_ht);
    tma_prefetch(&tm_wt);
    tma_prefetch(&tm_hs);
    tma_prefetch(&tm_ws);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kPassStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int valid_rows = min(p.n_rows, *p.n_eff - p.row0);
  const int m_tiles = valid_rows > 0 ? (valid_rows + kBM - 1) / kBM : 0;
  const int n_units = m_tiles * p.n_split;

  if (warp == 0) {
    // ================================================================ TMA producer
    uint32_t kit = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const UnitRange ur = unit_range(u, m_tiles, p.n_split, p.v_tiles);
      const int row = p.row0 + ur.m_tile * kBM;
      for (int vt = ur.vt0; vt < ur.vt1; ++vt) {
        const int vrow = vt * kBN;
        for (int kb = 0; kb < p.kb_t + p.kb_s; ++kb, ++kit) {
          const uint32_t st = kit % kPassStages, ph = (kit / kPassStages) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[st], kStageBytes);
            if (kb < p.kb_t) {
              tma_load_2d(&tm_ht, &full[st], sA + st * kTileBytes, kb * kBK, row);
              tma_load_2d(&tm_wt, &full[st], sB + st * kTileBytes, kb * kBK, vrow);
            } else {
              const int k = (kb - p.kb_t) * kBK;
              tma_load_2d(&tm_hs, &full[st], sA + st * kTileBytes, k, row);
              tma_load_2d(&tm_ws, &full[st], sB + st * kTileBytes, k, vrow);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (one thread)
    constexpr uint32_t idesc = idesc_bf16_f32(kBM, kBN, false, false);
    uint32_t kit = 0, it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const UnitRange ur = unit_range(u, m_tiles, p.n_split, p.v_tiles);
      for (int vt = ur.vt0; vt < ur.vt1; ++vt, ++it) {
        const uint32_t buf = it & 1, tph = (it >> 1) & 1;
        mbar_wait(&tempty[buf], tph ^ 1);
        tc_fence_after();
        const uint32_t d_t = tmem_base + buf * 256;
        const uint32_t d_s = d_t + 128;
        for (int kb = 0; kb < p.kb_t + p.kb_s; ++kb, ++kit) {
          const uint32_t st = kit % kPassStages, ph = (kit / kPassStages) & 1;
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const bool teacher = kb < p.kb_t;
            const int kb0 = teacher ? kb : kb - p.kb_t;
            const uint32_t d = teacher ? d_t : d_s;
            const uint32_t a_addr = smem_u32(sA + st * kTileBytes);
            const uint32_t b_addr = smem_u32(sB + st * kTileBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              umma_bf16(d, sdesc_sw128(a_addr + k * 32, 16, 1024), sdesc_sw128(b_addr + k * 32, 16, 1024), idesc,
                        (kb0 | k) != 0);
            }
            umma_commit(&empty[st]);
            if (kb == p.kb_t + p.kb_s - 1) umma_commit(&tfull[buf]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    // ================================================================ epilogue (one token row per thread)
    const uint32_t q4 = warp - 4;                   // TMEM lane quarter
    const int r_in_tile = q4 * 32 + lane;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const float alpha = p.alpha;
    uint32_t it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const UnitRange ur = unit_range(u, m_tiles, p.n_split, p.v_tiles);
      const int r_local = ur.m_tile * kBM + r_in_tile;  // row within the chunk
      const bool row_ok = r_local < valid_rows;
      const int split = u / m_tiles;
      // per-row state
      float Mp = -INFINITY, Mq = -INFINITY, Sp = 0.f, Sq = 0.f, U = 0.f;  // pass 1
      float L2t = 0.f, L2s = 0.f, ell2 = 0.f, Kacc = 0.f, Jacc = 0.f;     // pass 2
      if (PASS == 2 && row_ok) {
        L2t = p.fstats[r_local];
        L2s = p.fstats[p.n_rows + r_local];
        ell2 = p.fstats[2 * p.n_rows + r_local];
      }
      for (int vt = ur.vt0; vt < ur.vt1; ++vt, ++it) {
        const uint32_t buf = it & 1, tph = (it >> 1) & 1;
        mbar_wait(&tfull[buf], tph);
        tc_fence_after();
        const uint32_t t_addr = tmem_base + lane_addr + buf * 256;
        const int vbase = vt * kBN;
#pragma unroll 1
        for (int c = 0; c < kBN / 32; ++c) {
          float zt[32], zs[32];
          tmem_ld32(t_addr + c * 32, zt);
          tmem_ld32(t_addr + 128 + c * 32, zs);
          tmem_wait_ld();
          if (c == kBN / 32 - 1) {  // accumulator buffer fully drained -> hand it back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
          }
          const int v0 = vbase + c * 32;
          const int nvalid = min(32, p.V_r - v0);  // columns of this chunk inside [0, V_r)
          if (PASS == 1) {
            if (nvalid <= 0) continue;
            float* zp = (KIND == KIND_RKL) ? zs : zt;
            float* zq = (KIND == KIND_RKL) ? zt : zs;
            if (nvalid < 32) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i >= nvalid) { zp[i] = -1e30f; zq[i] = -1e30f; }
            }
            float cp = zp[0], cq = zq[0];
#pragma unroll
            for (int i = 1; i < 32; ++i) { cp = fmaxf(cp, zp[i]); cq = fmaxf(cq, zq[i]); }
            const float nMp = fmaxf(Mp, cp * alpha), nMq = fmaxf(Mq, cq * alpha);
            if (Sp == 0.f) {
              Mp = nMp; Mq = nMq;
            } else if (nMp > Mp || nMq > Mq) {
              const float dp = nMp - Mp, dq = nMq - Mq;
              const float fp = ex2(-dp);
              U = fp * (U - (dp - dq) * Sp);
              Sp *= fp;
              Sq *= ex2(-dq);
              Mp = nMp; Mq = nMq;
            }
            float sp[4] = {0.f, 0.f, 0.f, 0.f}, sq[4] = {0.f, 0.f, 0.f, 0.f}, uu[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float xp = fmaf(zp[i], alpha, -Mp);
              const float xq = fmaf(zq[i], alpha, -Mq);
              const float e = ex2(xp);
              sp[i & 3] += e;
              sq[i & 3] += ex2(xq);
              uu[i & 3] = fmaf(e, xp - xq, uu[i & 3]);
            }
            Sp += (sp[0] + sp[1]) + (sp[2] + sp[3]);
            Sq += (sq[0] + sq[1]) + (sq[2] + sq[3]);
            U += (uu[0] + uu[1]) + (uu[2] + uu[3]);
          } else {
            // ------------------------------------------------ pass 2: logit gradient
            if (v0 >= p.g_ld) continue;  // beyond the scratch row (only in the last tile)
            float g[32], gb[32];
            float kk[2] = {0.f, 0.f}, jj[2] = {0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float xt = fmaf(zt[i], alpha, -L2t);  // log2 p
              const float xs = fmaf(zs[i], alpha, -L2s);  // log2 q
              const float pt = ex2(xt), qs = ex2(xs);
              const bool ok = row_ok && (i < nvalid);
              if (KIND == KIND_FKL) {
                g[i] = ok ? p.gscale * (qs - pt) : 0.f;
              } else if (KIND == KIND_RKL) {
                g[i] = ok ? p.gscale * qs * ((xs - xt) - ell2) : 0.f;
              } else if (KIND == KIND_JSD) {
                const float m = fmaxf(fmaf(p.beta, pt, (1.f - p.beta) * qs), 1.17549435e-38f);
                const float lm = lg2(m);
                const float lv = xs - lm;  // log2(q/m)
                const float a = qs * lv;
                g[i] = ok ? a : 0.f;
                gb[i] = ok ? qs : 0.f;
                kk[i & 1] += ok ? a : 0.f;
                jj[i & 1] += ok ? pt * (xt - lm) : 0.f;
              } else {  // TVD
                const float d = qs - pt;
                const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
                g[i] = ok ? qs * sgn : 0.f;
                gb[i] = ok ? qs : 0.f;
                kk[i & 1] += ok ? qs * sgn : 0.f;
                jj[i & 1] += ok ? fabsf(d) : 0.f;
              }
            }
            const size_t off = (size_t)r_local * p.g_ld + v0;
            if (KIND == KIND_FKL || KIND == KIND_RKL) {
              uint32_t hi[16], lo[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) split2(g[2 * i], g[2 * i + 1], hi[i], lo[i]);
              uint8_t* ph = reinterpret_cast<uint8_t*>(p.g_hi + off);
              uint8_t* pl = reinterpret_cast<uint8_t*>(p.g_lo + off);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                st_global_v4(ph + 16 * i, hi[4 * i], hi[4 * i + 1], hi[4 * i + 2], hi[4 * i + 3]);
                st_global_v4(pl + 16 * i, lo[4 * i], lo[4 * i + 1], lo[4 * i + 2], lo[4 * i + 3]);
              }
            } else {
              float* pa = p.g_a + off;
              float* pb = p.g_b + off;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                st_global_v4(pa + 4 * i, __float_as_uint(g[4 * i]), __float_as_uint(g[4 * i + 1]),
                             __float_as_uint(g[4 * i + 2]), __float_as_uint(g[4 * i + 3]));
                st_global_v4(pb + 4 * i, __float_as_uint(gb[4 * i]), __float_as_uint(gb[4 * i + 1]),
                             __float_as_uint(gb[4 * i + 2]), __float_as_uint(gb[4 * i + 3]));
              }
              Kacc += kk[0] + kk[1];
              Jacc += jj[0] + jj[1];
            }
          }
        }
      }
      // ---- unit done: emit per-row partials (rows inside the chunk's valid range only)
      if (row_ok) {
        const size_t idx = (size_t)split * p.n_rows + r_local;
        if (PASS == 1) {
          p.part[idx] = Mp;
          p.part[p.part_plane + idx] = Mq;
          p.part[2 * p.part_plane + idx] = Sp;
          p.part[3 * p.part_plane + idx] = Sq;
          p.part[4 * p.part_plane + idx] = U;
        } else if (KIND == KIND_JSD || KIND == KIND_TVD) {
          const size_t plane = (size_t)p.n_split * p.n_rows;
          p.kpart[idx] = Kacc;
          p.kpart[plane + idx] = Jacc;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------------------------------------- host-side launchers
template <int PASS, int KIND>
static cudaError_t launch_pass_t(const CUtensorMap* maps, const PassParams& p, int grid, cudaStream_t stream) {
  auto kern = kd_pass_kernel<PASS, KIND>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPassSmem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kPassThreads, kPassSmem, stream>>>(maps[0], maps[1], maps[2], maps[3], p);
  return cudaGetLastError();
}

cudaError_t launch_pass(int pass, int kind, const CUtensorMap* maps, const PassParams& p, int grid,
                        cudaStream_t stream) {
  if (pass == 1) {
    // pass 1 only distinguishes which side is "primary" (RKL swaps the roles)
    return kind == KIND_RKL ? launch_pass_t<1, KIND_RKL>(maps, p, grid, stream)
                            : launch_pass_t<1, KIND_FKL>(maps, p, grid, stream);
  }
  switch (kind) {
    case KIND_FKL: return launch_pass_t<2, KIND_FKL>(maps, p, grid, stream);
    case KIND_RKL: return launch_pass_t<2, KIND_RKL>(maps, p, grid, stream);
    case KIND_JSD: return launch_pass_t<2, KIND_JSD>(maps, p, grid, stream);
    default: return launch_pass_t<2, KIND_TVD>(maps, p, grid, stream);
  }
}

int pass_smem_bytes() { return kPassSmem; }

}  // namespace kd
