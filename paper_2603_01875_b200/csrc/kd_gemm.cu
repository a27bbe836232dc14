// kd_gemm.cu — tcgen05 GEMM for the backward products of the KD hot path (sm_100a).
//
//   dL/dh_s = G · W_s        ("backward passes"):  A = G [tokens, V], stored as Gᵀ [V][tokens] (MN-major),
//                                                         B = W_s [V, d_s]   (MN-major: d_s contiguous)
//   dL/dW_s = Gᵀ · H_s                                   A = Gᵀ [V][tokens] (K-major, K = tokens),
//                                                         B = H_s [tokens, d_s] (MN-major)
// G arrives as a split-bf16 pair (hi + lo, R11), so A is NUM_A = 2 planes that share every B
// tile: D += A_hi·Bᵀ + A_lo·Bᵀ  — one B load feeds two MMAs.
//
// Output tile 256 x 256 per SM pair (CG = 2: cluster of 2, tcgen05.mma.cta_group::2 with UMMA M=256, N=256; each
// CTA stages its own 128 rows of A and half of the B tile, so per-SM operand inflow is 48 B/clk at full tensor rate
// instead of the 64 B/clk of a single-SM 128 x 256 tile — the SM's L2->SMEM port caps near that; DESIGN.md
// "Kernel 3") or 128 x 256 per CTA (CG = 1, A/B experiments).  TMA 128B-swizzled operands, 192 KB mbarrier ring,
// double-buffered TMEM accumulator (2 x 256 columns), persistent grid.
// Epilogue: TMEM -> registers -> fp32 global (store into a split-K slab, or read-modify-write accumulate).
//
// Accumulation precision: tcgen05's fp32 accumulation loses bits on every MMA step (measured:
// scripts/probe_accum.py, probe_longk.py — error grows ~linearly with the steps per accumulator), and these
// GEMMs run K = V = 151936 long.  So a unit's K range is cut into pieces of <= kb_per_acc K blocks; each
// piece gets a fresh TMEM accumulator (the double buffer rotates per piece) and the epilogue adds it into
// the fp32 output with round-to-nearest CUDA-core adds ("promotion"), overlapped with the next piece's MMAs.
#include <atomic>

#include "kd_params.cuh"
#include "sm100.cuh"

namespace kd {

template <int NUM_A, int CG>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;                // 16 KB per A plane (this CTA's 128 rows)
  static constexpr int kBBytes = (kGemmBN / CG) * kBK * 2;     // this CTA's share of the B tile
  static constexpr int kStageBytes = NUM_A * kABytes + kBBytes;
  static constexpr int kStages = (192 * 1024) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

template <bool A_MN, bool B_MN, int NUM_A, int EPI, int CG>
__global__ void __launch_bounds__(kGemmThreads, 1)
    kd_gemm_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_a1,
                   const __grid_constant__ CUtensorMap tm_b, const GemmParams p) {
  using C = GemmCfg<NUM_A, CG>;
  constexpr int kBMt = kBM * CG;  // output rows per (pair) tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // 0 = leader (issues the MMAs)
  const int worker = blockIdx.x / CG, n_workers = gridDim.x / CG;
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
      mbar_init(&tempty[b], kGemmEpiWarps * CG);  // every epilogue warp of the group releases
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2) tmem_alloc_pair(tmem_slot, 512);
    else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  int M = p.M, K = p.K;
  if (p.dyn_dim == DYN_M) M = max(0, min(p.M, *p.dyn - p.dyn_base));
  if (p.dyn_dim == DYN_K) K = max(0, min(p.K, *p.dyn - p.dyn_base));
  const int m_tiles = (M + kBMt - 1) / kBMt;
  const int n_tiles = (p.N + kGemmBN - 1) / kGemmBN;
  const int kbs = (K + kBK - 1) / kBK;
  const int n_units = m_tiles * n_tiles * p.k_split;

  auto unit = [&](int u, int& m0, int& n0, int& kb0, int& kb1, int& ks) {
    const int nt = u % n_tiles;
    const int mt = (u / n_tiles) % m_tiles;
    ks = u / (n_tiles * m_tiles);
    m0 = mt * kBMt;
    n0 = nt * kGemmBN;
    kb0 = (int)((long long)ks * kbs / p.k_split);
    kb1 = (int)((long long)(ks + 1) * kbs / p.k_split);
  };

  if (warp == 0) {
    // ================================================================ TMA producer
    uint32_t kit = 0;
    for (int u = worker; u < n_units; u += n_workers) {
      int m0, n0, kb0, kb1, ks;
      unit(u, m0, n0, kb0, kb1, ks);
      const int mr = m0 + rank * kBM;               // this CTA's 128 rows of A
      const int nr = n0 + rank * (kGemmBN / CG);    // this CTA's share of the B tile
      for (int kb = kb0; kb < kb1; ++kb, ++kit) {
        const uint32_t st = kit % C::kStages, ph = (kit / C::kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        if (lane == 0) {
          uint8_t* s = smem + st * C::kStageBytes;
          // the leader's full barrier collects the bytes of the whole group
          if (rank == 0) mbar_arrive_expect_tx(&full[st], CG * C::kStageBytes);
          auto load = [&](const CUtensorMap* m, void* dst, int x, int y) {
            if (CG == 2) tma_load_2d_pair(m, &full[st], dst, x, y);
            else tma_load_2d(m, &full[st], dst, x, y);
          };
          const int k0 = kb * kBK;
#pragma unroll
          for (int a = 0; a < NUM_A; ++a) {
            const CUtensorMap* ma = a == 0 ? &tm_a0 : &tm_a1;
            uint8_t* sa = s + a * C::kABytes;
            if (A_MN) {  // [K rows][M cols]: two 64-wide M boxes
              load(ma, sa, mr, k0);
              load(ma, sa + 8192, mr + 64, k0);
            } else {
              load(ma, sa, k0, mr);
            }
          }
          uint8_t* sb = s + NUM_A * C::kABytes;
          if (B_MN) {  // [K rows][N cols]: 64-wide N boxes
#pragma unroll
            for (int j = 0; j < 4 / CG; ++j) load(&tm_b, sb + j * 8192, nr + 64 * j, k0);
          } else {
            load(&tm_b, sb, k0, nr);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ================================================================ MMA issuer (one thread of the leader)
    constexpr uint32_t idesc = idesc_bf16_f32(kBMt, kGemmBN, A_MN, B_MN);
    uint32_t kit = 0, it = 0;
    for (int u = worker; u < n_units; u += n_workers) {
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
                const uint32_t acc = (kb > pk0 || k > 0 || a > 0) ? 1u : 0u;
                if (CG == 2) umma_bf16_pair(d, adesc, bdesc, idesc, acc);
                else umma_bf16(d, adesc, bdesc, idesc, acc);
              }
            }
            if (CG == 2) umma_commit_pair(&empty[st], 0x3);
            else umma_commit(&empty[st]);
          }
          __syncwarp();
        }
        if (lane == 0) {  // also fires for an empty K range
          if (CG == 2) umma_commit_pair(&tfull[buf], 0x3);
          else umma_commit(&tfull[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ================================================================ epilogue
    // kGemmEpiWarps warps: (warp - 4) % 4 = TMEM lane quarter (one output row per thread), (warp - 4) / 4 = which
    // contiguous part of the tile's 32-column chunks.  A promotion piece's read-modify-write loads all eight float4 of
    // a chunk before the first add, so a warp keeps 8 L2 round trips in flight instead of one (with 16-block pieces
    // the RMW would otherwise outlast the piece's MMAs).
    constexpr int kParts = kGemmEpiWarps / 4, kChunks = kGemmBN / 32;
    const uint32_t q4 = (warp - 4) & 3;
    const int part = (int)(warp - 4) >> 2;
    const int c_beg = part * kChunks / kParts, c_end = (part + 1) * kChunks / kParts;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
#ifndef KD_X_NO_GEMM_SLAB_HINT
    const uint64_t pol_last = l2_policy_evict_last();
#endif
    uint32_t it = 0;
    for (int u = worker; u < n_units; u += n_workers) {
      int m0, n0, kb0, kb1, ks;
      unit(u, m0, n0, kb0, kb1, ks);
      const int npieces = kb1 > kb0 ? (kb1 - kb0 + p.kb_per_acc - 1) / p.kb_per_acc : 1;
      const int row = m0 + rank * kBM + q4 * 32 + lane;
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
        for (int c = c_beg; c < c_end; ++c) {
          float v[32];
          tmem_ld32_sync(tmem_base + lane_addr + buf * kGemmBN + c * 32, v);
          if (c == c_end - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader + buf * 8);
              else mbar_arrive_relaxed(&tempty[buf]);
            }
          }
          if (!row_ok || n0 + c * 32 >= p.N) continue;
          float* o = orow + c * 32;
#ifndef KD_X_NO_GEMM_SLAB_HINT
          // split-K slab tiles (EPI_STORE: the dh GEMM) are stored evict_last, so a unit's promotion pieces find their
          // tile in L2 instead of DRAM (ncu, c2 chunk: DRAM writes 603 -> 118 MB, reads 3.41 -> 2.94 GB per launch;
          // profiles/r02_ab.md).  dW (EPI_ACCUM, 1.2 GB of tiles re-read every chunk) stays unhinted.
          if (EPI == EPI_STORE) {
            if (accumulate) {
              if (empty_k) continue;
              float4 prev[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) prev[i] = __ldcg(reinterpret_cast<const float4*>(o + 4 * i));
#pragma unroll
              for (int i = 0; i < 8; ++i)
                st_global_f4_hint(o + 4 * i, make_float4(prev[i].x + v[4 * i], prev[i].y + v[4 * i + 1],
                                                         prev[i].z + v[4 * i + 2], prev[i].w + v[4 * i + 3]), pol_last);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                st_global_f4_hint(o + 4 * i, empty_k ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                     : make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]),
                                  pol_last);
            }
            continue;
          }
#endif
          if (accumulate) {
            if (empty_k) continue;
            float4 prev[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) prev[i] = __ldcg(reinterpret_cast<const float4*>(o + 4 * i));
#pragma unroll
            for (int i = 0; i < 8; ++i)
              st_global_v4(o + 4 * i, __float_as_uint(prev[i].x + v[4 * i]), __float_as_uint(prev[i].y + v[4 * i + 1]),
                           __float_as_uint(prev[i].z + v[4 * i + 2]), __float_as_uint(prev[i].w + v[4 * i + 3]));
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
  if (CG == 2) cluster_sync();  // neither CTA leaves while its partner may still signal its barriers
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (CG == 2) tmem_dealloc_pair(tmem_base, 512);
    else tmem_dealloc(tmem_base, 512);
  }
}

template <bool A_MN, bool B_MN, int NUM_A, int EPI, int CG>
static cudaError_t launch_gemm_t(const CUtensorMap* a0, const CUtensorMap* a1, const CUtensorMap* b,
                                 const GemmParams& p, int sms, cudaStream_t stream) {
  auto kern = kd_gemm_kernel<A_MN, B_MN, NUM_A, EPI, CG>;
  const int smem = GemmCfg<NUM_A, CG>::kSmem;
  // the shared-memory opt-in once per (instantiation, device): a driver call on every launch was measurable host
  // time for the per-chunk callers
  static std::atomic<uint64_t> smem_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(smem_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  const long long units = (long long)((p.M + kBM * CG - 1) / (kBM * CG)) * ((p.N + kGemmBN - 1) / kGemmBN) * p.k_split;
  const int workers = (int)(units < sms / CG ? units : sms / CG);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((workers > 0 ? workers : 1) * CG);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, *a0, a1 ? *a1 : *a0, *b, p);
}

// Dispatch over the (major, planes, epilogue) combinations the library uses (+ the test-only ones).
// cg: 2 = SM-pair tiles (B tensor maps with 128-row / 64-col boxes per CTA), 1 = single-SM tiles.
// sms: SMs available to the persistent grid.
cudaError_t launch_gemm(bool a_mn, bool b_mn, int num_a, int epi, int cg, const CUtensorMap* a0,
                        const CUtensorMap* a1, const CUtensorMap* b, const GemmParams& p, int sms,
                        cudaStream_t stream) {
#define KD_GEMM_CASE(AM, BM_, NA, EP)                                                           \
  if (a_mn == AM && b_mn == BM_ && num_a == NA && epi == EP)                                    \
    return cg == 2 ? launch_gemm_t<AM, BM_, NA, EP, 2>(a0, a1, b, p, sms, stream)               \
                   : launch_gemm_t<AM, BM_, NA, EP, 1>(a0, a1, b, p, sms, stream);
  KD_GEMM_CASE(false, false, 1, EPI_STORE)
  KD_GEMM_CASE(false, true, 1, EPI_STORE)
  KD_GEMM_CASE(true, false, 1, EPI_STORE)
  KD_GEMM_CASE(true, true, 1, EPI_STORE)
  KD_GEMM_CASE(true, true, 2, EPI_STORE)    // dh = [G_hi|G_lo] · W_s    (scratch holds Gᵀ: A MN-major)
  KD_GEMM_CASE(false, true, 2, EPI_ACCUM)   // dW += [G_hi|G_lo]ᵀ · H_s  (Gᵀ: A K-major)
  KD_GEMM_CASE(true, true, 1, EPI_ACCUM)
  KD_GEMM_CASE(false, true, 1, EPI_ACCUM)   // dW with a single bf16 G plane (KD_GRAD_BF16)
#undef KD_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace kd
