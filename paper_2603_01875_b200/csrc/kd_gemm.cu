// kd_gemm.cu — tcgen05 GEMM for the backward products of the KD hot path (sm_100a).
//
//   dL/dh_s = G · W_s        ("backward passes"):  A = G [tokens, V], stored as Gᵀ [V][tokens] (MN-major),
//                                                         B = W_s [V, d_s]   (MN-major: d_s contiguous)
//   dL/dW_s = Gᵀ · H_s                                   A = Gᵀ [V][tokens] (K-major, K = tokens),
//                                                         B = H_s [tokens, d_s] (MN-major)
// G arrives as a split-bf16 pair (hi + lo, R11), so A is NUM_A = 2 planes that share every B
// tile: D += A_hi·Bᵀ + A_lo·Bᵀ  — one B load feeds two MMAs.
//
// 128 x 256 output tile per CTA (UMMA M=128, N=256, K=16), TMA 128B-swizzled operands, 3-4 stage
// mbarrier ring, double-buffered TMEM accumulator (2 x 256 columns), persistent grid.
// Epilogue: TMEM -> registers -> fp32 global (store into a split-K slab, or read-modify-write accumulate).
//
// Accumulation precision: tcgen05's fp32 accumulation loses bits on every MMA step (measured:
// scripts/probe_accum.py, probe_longk.py — error grows ~linearly with the steps per accumulator), and these
// GEMMs run K = V = 151936 long.  So a unit's K range is cut into pieces of <= kb_per_acc K blocks; each
// piece gets a fresh TMEM accumulator (the double buffer rotates per piece) and the epilogue adds it into
// the fp32 output with round-to-nearest CUDA-core adds ("promotion"), overlapped with the next piece's MMAs.
#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

template <int NUM_A>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;         // 16 KB per A plane
  static constexpr int kBBytes = kGemmBN * kBK * 2;     // 32 KB
  static constexpr int kStageBytes = NUM_A * kABytes + kBBytes;
  static constexpr int kStages = (NUM_A == 2) ? 3 : 4;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

template <bool A_MN, bool B_MN, int NUM_A, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    kd_gemm_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_a1,
                   const __grid_constant__ CUtensorMap tm_b, const GemmParams p) {
  using C = GemmCfg<NUM_A>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_a0);
    if (NUM_A == 2) tma_prefetch(&tm_a1);
    tma_prefetch(&tm_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  int M = p.M, K = p.K;
  if (p.dyn_dim == DYN_M) M = max(0, min(p.M, *p.dyn - p.dyn_base));
  if (p.dyn_dim == DYN_K) K = max(0, min(p.K, *p.dyn - p.dyn_base));
  const int m_tiles = (M + kBM - 1) / kBM;
  const int n_tiles = (p.N + kGemmBN - 1) / kGemmBN;
  const int kbs = (K + kBK - 1) / kBK;
  const int n_units = m_tiles * n_tiles * p.k_split;

  auto unit = [&](int u, int& m0, int& n0, int& kb0, int& kb1, int& ks) {
    const int nt = u % n_tiles;
    const int mt = (u / n_tiles) % m_tiles;
    ks = u / (n_tiles * m_tiles);
    m0 = mt * kBM;
    n0 = nt * kGemmBN;
    kb0 = (int)((long long)ks * kbs / p.k_split);
    kb1 = (int)((long long)(ks + 1) * kbs / p.k_split);
  };

  if (warp == 0) {
    // ================================================================ TMA producer
    uint32_t kit = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, n0, kb0, kb1, ks;
      unit(u, m0, n0, kb0, kb1, ks);
      for (int kb = kb0; kb < kb1; ++kb, ++kit) {
        const uint32_t st = kit % C::kStages, ph = (kit / C::kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        if (lane == 0) {
          uint8_t* s = smem + st * C::kStageBytes;
          mbar_arrive_expect_tx(&full[st], C::kStageBytes);
          const int k0 = kb * kBK;
#pragma unroll
          for (int a = 0; a < NUM_A; ++a) {
            const CUtensorMap* ma = a == 0 ? &tm_a0 : &tm_a1;
            uint8_t* sa = s + a * C::kABytes;
            if (A_MN) {  // [K rows][M cols]: two 64-wide M boxes
              tma_load_2d(ma, &full[st], sa, m0, k0);
              tma_load_2d(ma, &full[st], sa + 8192, m0 + 64, k0);
            } else {
              tma_load_2d(ma, &full[st], sa, k0, m0);
            }
          }
          uint8_t* sb = s + NUM_A * C::kABytes;
          if (B_MN) {  // [K rows][N cols]: four 64-wide N boxes
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_load_2d(&tm_b, &full[st], sb + j * 8192, n0 + 64 * j, k0);
          } else {
            tma_load_2d(&tm_b, &full[st], sb, k0, n0);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(kBM, kGemmBN, A_MN, B_MN);
    uint32_t kit = 0, it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, n0, kb0, kb1, ks;
      unit(u, m0, n0, kb0, kb1, ks);
      const int npieces = kb1 > kb0 ? (kb1 - kb0 + p.kb_per_acc - 1) / p.kb_per_acc : 1;
      for (int pc = 0; pc < npieces; ++pc, ++it) {
        const int pk0 = kb0 + pc * p.kb_per_acc, pk1 = min(kb1, pk0 + p.kb_per_acc);
        const uint32_t buf = it & 1, tph = (it >> 1) & 1;
        mbar_wait(&tempty[buf], tph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * kGemmBN;
        for (int kb = pk0; kb < pk1; ++kb, ++kit) {
          const uint32_t st = kit % C::kStages, ph = (kit / C::kStages) & 1;
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t s = smem_u32(smem + st * C::kStageBytes);
            const uint32_t sb = s + NUM_A * C::kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t bdesc =
                  B_MN ? sdesc_sw128(sb + k * 2048, 8192, 1024) : sdesc_sw128(sb + k * 32, 16, 1024);
#pragma unroll
              for (int a = 0; a < NUM_A; ++a) {
                const uint32_t sa = s + a * C::kABytes;
                const uint64_t adesc =
                    A_MN ? sdesc_sw128(sa + k * 2048, 8192, 1024) : sdesc_sw128(sa + k * 32, 16, 1024);
                umma_bf16(d, adesc, bdesc, idesc, (kb > pk0 || k > 0 || a > 0) ? 1u : 0u);
              }
            }
            umma_commit(&empty[st]);
          }
          __syncwarp();
        }
        if (lane == 0) umma_commit(&tfull[buf]);  // also fires for an empty K range
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ================================================================ epilogue
    const uint32_t q4 = warp - 4;
    const uint32_t lane_addr = (q4 * 32) << 16;
    uint32_t it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, n0, kb0, kb1, ks;
      unit(u, m0, n0, kb0, kb1, ks);
      const int npieces = kb1 > kb0 ? (kb1 - kb0 + p.kb_per_acc - 1) / p.kb_per_acc : 1;
      const int row = m0 + q4 * 32 + lane;
      const bool row_ok = row < M;
      const bool empty_k = kb1 <= kb0;
      float* orow = p.out + (size_t)ks * p.out_split_stride + (size_t)row * p.out_ld + n0;
      for (int pc = 0; pc < npieces; ++pc, ++it) {
      const uint32_t buf = it & 1, tph = (it >> 1) & 1;
      mbar_wait(&tfull[buf], tph);
      tc_fence_after();
      // first piece of an EPI_STORE unit stores; every other piece accumulates into what is there
      const bool accumulate = (EPI == EPI_ACCUM) || pc > 0;
#pragma unroll 1
      for (int c = 0; c < kGemmBN / 32; ++c) {
        float v[32];
        tmem_ld32_sync(tmem_base + lane_addr + buf * kGemmBN + c * 32, v);
        if (c == kGemmBN / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
        }
        if (!row_ok || n0 + c * 32 >= p.N) continue;
        float* o = orow + c * 32;
        if (accumulate) {
          if (empty_k) continue;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 prev = *reinterpret_cast<const float4*>(o + 4 * i);
            st_global_v4(o + 4 * i, __float_as_uint(prev.x + v[4 * i]), __float_as_uint(prev.y + v[4 * i + 1]),
                         __float_as_uint(prev.z + v[4 * i + 2]), __float_as_uint(prev.w + v[4 * i + 3]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float a = empty_k ? 0.f : v[4 * i], b = empty_k ? 0.f : v[4 * i + 1];
            const float c2 = empty_k ? 0.f : v[4 * i + 2], d2 = empty_k ? 0.f : v[4 * i + 3];
            st_global_v4(o + 4 * i, __float_as_uint(a), __float_as_uint(b), __float_as_uint(c2), __float_as_uint(d2));
          }
        }
      }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

template <bool A_MN, bool B_MN, int NUM_A, int EPI>
static cudaError_t launch_gemm_t(const CUtensorMap* a0, const CUtensorMap* a1, const CUtensorMap* b,
                                 const GemmParams& p, int grid, cudaStream_t stream) {
  auto kern = kd_gemm_kernel<A_MN, B_MN, NUM_A, EPI>;
  const int smem = GemmCfg<NUM_A>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kGemmThreads, smem, stream>>>(*a0, a1 ? *a1 : *a0, *b, p);
  return cudaGetLastError();
}

// Dispatch over the (major, planes, epilogue) combinations the library uses (+ the test-only ones).
cudaError_t launch_gemm(bool a_mn, bool b_mn, int num_a, int epi, const CUtensorMap* a0, const CUtensorMap* a1,
                        const CUtensorMap* b, const GemmParams& p, int grid, cudaStream_t stream) {
#define KD_GEMM_CASE(AM, BM_, NA, EP)                                              \
  if (a_mn == AM && b_mn == BM_ && num_a == NA && epi == EP)                       \
    return launch_gemm_t<AM, BM_, NA, EP>(a0, a1, b, p, grid, stream);
  KD_GEMM_CASE(false, false, 1, EPI_STORE)
  KD_GEMM_CASE(false, true, 1, EPI_STORE)
  KD_GEMM_CASE(true, false, 1, EPI_STORE)
  KD_GEMM_CASE(true, true, 1, EPI_STORE)
  KD_GEMM_CASE(true, true, 2, EPI_STORE)    // dh = [G_hi|G_lo] · W_s    (scratch holds Gᵀ: A MN-major)
  KD_GEMM_CASE(false, true, 2, EPI_ACCUM)   // dW += [G_hi|G_lo]ᵀ · H_s  (Gᵀ: A K-major)
  KD_GEMM_CASE(true, true, 1, EPI_ACCUM)
#undef KD_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace kd
