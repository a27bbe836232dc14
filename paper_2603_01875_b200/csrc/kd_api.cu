// kd_api.cu — host side of the C ABI declared in include/kdfused.h.
//
// Validation, the execution plan (token chunking, vocab-split and split-K choices sized to the SM
// count), workspace carving, TMA tensor-map encoding and the launch sequence on the caller's stream.
// Everything here is plain host C++; every floating-point step of the method runs in the kernels of
// kd_pass.cu / kd_gemm.cu / kd_aux.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/kdfused.h"
#include "kd_params.cuh"

namespace kd {
cudaError_t launch_pass(int pass, int kind, bool coupled, int cg, int bn, const CUtensorMap* maps, const PassParams& p,
                        int grid, cudaStream_t s);
cudaError_t launch_gemm(bool a_mn, bool b_mn, int num_a, int epi, int cg, const CUtensorMap* a0, const CUtensorMap* a1,
                        const CUtensorMap* b, const GemmParams& p, int sms, cudaStream_t stream);
cudaError_t launch_compact(const uint8_t* mask, int N, int* idx, int* n_eff, cudaStream_t s);
cudaError_t launch_gather(const __nv_bfloat16* src, long long src_ld, __nv_bfloat16* dst, int d, int N,
                          const int* idx, const int* n_eff, cudaStream_t s);
cudaError_t launch_zero_masked(const uint8_t* mask, int N, float* loss, float* dh, int d_s, cudaStream_t s);
cudaError_t launch_merge(const float* part, long long plane, long long split_stride, int n_split, int n_rows,
                         int row0, const int* n_eff, int kind, int mode, float* fstats, float* loss, float* rec,
                         long long rec_plane, const int* idx, int orig_rows, long long* nonfinite, int write_loss,
                         cudaStream_t s, const float* tstats_in = nullptr);
cudaError_t launch_loss_rows(const float* lpart, int n_slots, int n_rows, int row0, const int* n_eff, const RowDst& loss,
                             const int* idx, long long* nonfinite, cudaStream_t s);
cudaError_t launch_kfix(const float* kpart, int n_split, int n_rows, int row0, const int* n_eff, int kind, float beta,
                        float* kfin, float* loss, const int* idx, long long* nonfinite, const float* ga,
                        const float* gb, int g_ld, float scale, __nv_bfloat16* ghi, __nv_bfloat16* glo,
                        int num_sms, const float* kj_ranks, int n_ranks, long long N, cudaStream_t s);
cudaError_t launch_kj_rows(const float* kpart, int n_split, int n_rows, int row0, const int* n_eff, const int* idx,
                           float* kj, long long N, cudaStream_t s);
cudaError_t launch_stage_grad(int kind, const StageParams& sp, int n_slots, cudaStream_t s);
cudaError_t launch_die_probe(const unsigned* buf, const long long* line_off, int n_lines, int steps, unsigned* out,
                             int sms, int smem_bytes, cudaStream_t s);
int stage_rows();
int stage_cols();
cudaError_t launch_reduce_dh(const float* part, long long split_stride, int k_split, int d_s, int n_rows, int row0,
                             const int* n_eff, const int* idx, const RowDst& dh, const int* corr_v,
                             const float* corr_r, int n_slots, const __nv_bfloat16* Ws, cudaStream_t s,
                             const int* corr2_v = nullptr, const float* corr2_r = nullptr, int n_slots2 = 0);
cudaError_t launch_p2p_signal(const P2PFlags& f, cudaStream_t s);
cudaError_t launch_p2p_wait(const unsigned* ctr, int n, unsigned target, cudaStream_t s);
cudaError_t launch_p2p_combine(const P2PCombine& c, int num_sms, cudaStream_t s);
cudaError_t launch_p2p_copy(const P2PCopy& c, int num_sms, cudaStream_t s);
cudaError_t launch_zero_records(const uint8_t* mask, int N, float* rec, long long plane, cudaStream_t s);
cudaError_t launch_extract_zero(const int* corr_v, const float* corr_r, int n_slots, int n_rows, int row0,
                                const int* n_eff, __nv_bfloat16* ghi, __nv_bfloat16* glo, cudaStream_t s);
cudaError_t launch_topk_merge(const float* tk_val, const int* tk_idx, int n_slots, int n_rows, int row0,
                              const int* n_eff, const int* idx, int k, int v_base, int* out_idx, float* out_val,
                              cudaStream_t s);
cudaError_t launch_topk_fix(const __nv_bfloat16* hs, const __nv_bfloat16* Ws, int d_s, int V, int n_rows, int row0,
                            const int* n_eff, const int* idx, int k, const int* tk_i, const float* tk_v, float alpha,
                            const float* fstats, float gscale, __nv_bfloat16* ghi, __nv_bfloat16* glo, int* corr_v,
                            float* corr_r, int n_corr, int* tkr_v, float* tkr_r, float* loss, long long* nonfinite,
                            cudaStream_t s);
}  // namespace kd

using namespace kd;

// ------------------------------------------------------------------------------------ errors
static thread_local std::string g_err = "ok";
static thread_local int g_launches = 0;
static void* g_dbg_ptr = nullptr;  // device buffer for KD_EPI_TIMING builds (kd_debug_set_buffer)

static kd_status fail(kd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define KD_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail(KD_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
// ------------------------------------------------------------------------------------ live profiling
// When enabled, every launch is bracketed by two CUDA events on the launch stream; kd_profile_read()
// resolves them into per-kernel totals (bench.py uses this for the live roofline figure).
enum KernelId : int { K_COMPACT, K_GATHER, K_ZERO, K_PASS1, K_MERGE, K_PASS2, K_KFIX, K_GEMM_DH, K_REDUCE_DH,
                      K_GEMM_DW, K_GEMM, K_TOPK, K_STAGE_GRAD, K_P2P, K_NUM };
static const char* kKernelNames[K_NUM] = {"compact", "gather", "zero_masked", "pass1", "merge", "pass2",
                                          "kfix", "gemm_dh", "reduce_dh", "gemm_dW", "gemm", "topk",
                                          "stage_grad", "p2p"};
struct ProfRec { int id; cudaEvent_t a, b; };
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;
static std::mutex g_handoff_mu;
static std::unordered_map<void*, void*> g_handoff_bases;  // kd_handoff_open: returned pointer -> mapped base
static thread_local cudaStream_t g_cur_stream = nullptr;

static cudaEvent_t prof_event() {
  std::lock_guard<std::mutex> lk(g_prof_mu);  // kd_profile_read returns events to the pool from another thread
  if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Per-launch event brackets are recorded only outside stream capture: an event recorded into a graph
// is not something kd_profile_read could synchronise on later.
static bool prof_active() {
  if (!g_prof_on) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(g_cur_stream, &cs) != cudaSuccess) return false;
  return cs == cudaStreamCaptureStatusNone;
}

#define KD_LAUNCH(id, expr)                                                  \
  do {                                                                       \
    cudaEvent_t ea_ = nullptr, eb_ = nullptr;                                \
    const bool prof_ = prof_active();                                        \
    if (prof_) { ea_ = prof_event(); cudaEventRecord(ea_, g_cur_stream); }   \
    KD_CUDA(expr);                                                           \
    ++g_launches;                                                            \
    if (prof_) {                                                             \
      eb_ = prof_event();                                                    \
      cudaEventRecord(eb_, g_cur_stream);                                    \
      std::lock_guard<std::mutex> lk_(g_prof_mu);                            \
      g_prof.push_back({(id), ea_, eb_});                                    \
    }                                                                        \
  } while (0)

// ------------------------------------------------------------------------------------ TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static bool tma_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// bf16 2-D map: `inner` contiguous elements per row, `outer` rows of `row_bytes`; 128B-swizzled boxes.
static kd_status make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                          uint32_t box_inner, uint32_t box_outer) {
  if (!tma_encoder()) return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (outer == 0) outer = 1;  // never addressed when the extent is empty (kernels skip all tiles)
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu", (int)r,
                (unsigned long long)inner, (unsigned long long)outer);
  return KD_OK;
}

// ------------------------------------------------------------------------------------ plan
static int cta_group() {  // KD_CTA_GROUP=1 selects single-SM pass tiles (A/B experiments); default: SM pairs
  static int v = [] {
    const char* e = getenv("KD_CTA_GROUP");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return v;
}

static int gemm_cg() {  // KD_GEMM_CG=1 selects single-SM backward GEMM tiles (A/B experiments); default: SM pairs
  static int v = [] {
    const char* e = getenv("KD_GEMM_CG");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return v;
}

static int pass_bn() {  // KD_PASS_BN=128 selects 128-wide vocab tiles (A/B experiments); default 256
  static int v = [] {
    const char* e = getenv("KD_PASS_BN");
    return (e && atoi(e) == 128) ? 128 : 256;
  }();
  return v;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// Backward GEMMs flush their TMEM accumulator into the fp32 output every kKbPerAcc K blocks (see kd_gemm.cu).
// 64 (4096 K values per accumulator).  The dh GEMM's ill-conditioned outputs (the Zipf-bias column: results ~100x
// smaller than their terms) are protected by taking pass 2's largest entries out of its G instead (k_extract_zero):
// shorter pieces would cost a read-modify-write of the fp32 output per piece — 16 measured +18 ms per config-2 step.
constexpr int kKbPerAccDefault = 64;
static int kb_per_acc() {  // KD_KB_PER_ACC overrides the promotion period (precision experiments)
  static int v = [] {
    const char* e = getenv("KD_KB_PER_ACC");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : kKbPerAccDefault;
  }();
  return v;
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Plan {
  int N, d_t, d_s, V_r, kind;
  int Nc, n_chunks, m_tiles_c, v_tiles, n_split, g_ld, k_split, num_sms;
  int cg;  // CTA group of the fused passes: 2 = SM pairs (UMMA M=256), 1 = single SMs
  int bn;  // vocab tile of the fused passes (UMMA N): 256 or 128
  bool fix;  // JSD / TVD (two fp32 planes + K fix-up)
  int g_planes;  // bf16 planes of G fed to the backward GEMMs: 2 (split hi + lo) or 1 (KD_GRAD_BF16)
  bool stage;    // staged variant (kd_problem.stage_logits): pass 1 writes the chunk's logits, k_stage_grad makes G
  int n_gslots;  // per-row slots of the G step's partials (loss / (K, J) / residual fix): pass 2's n_split * parts,
                 // or the staged kernel's vocab slots
  // die-aware unit placement of the fused passes (PassParams::die_map): die_map != NULL when on; die_w0 = worker slots
  // of die 0; die_s0 = first vocab split of die 1
  const uint8_t* die_map;
  int die_w0, die_s0;
  size_t off_neff, off_nonfinite, off_idx, off_ht, off_hs, off_part, off_fstats, off_kpart, off_kfin, off_ghi,
      off_glo, off_ga, off_gb, off_dhp, off_corr_v, off_corr_r, off_zscr, off_tkv, off_tki, off_tkr_v, off_tkr_r,
      off_zst, off_sched, total;
};

// Static round-robin of units over a persistent grid: makespan in tiles (+ per-unit refill cost).
static double pass_makespan(int m_tiles, int s, int v_tiles, int sms) {
  const int units = m_tiles * s;
  const int grid = units < sms ? units : sms;
  double worst = 0;
  for (int c = 0; c < grid; ++c) {
    double t = 0;
    for (int u = c; u < units; u += grid) {
      const int sp = u / m_tiles;
      t += (double)((long long)(sp + 1) * v_tiles / s - (long long)sp * v_tiles / s) + 0.1;
    }
    if (t > worst) worst = t;
  }
  return worst;
}

// ------------------------------------------------------------------------------------ SM -> die map
// B200 has two dies, each with its own L2 partition.  The fused passes read every vocab tile of the heads once per
// token tile of the chunk; the token tiles of one vocab split run concurrently, so when their SM pairs sit on both
// dies each die's L2 misses on the same head rows and the heads come from DRAM ~2x (profiles/r01_ncu_full_final.md).
// The map is measured once per device (k_die_probe: per-SM L2 latency to lines homed on either partition; the two
// near-sets are the dies) and then steers each pair to a worker slot of its own die (PassParams::die_map).  A map
// that does not look like two equal halves of SM pairs is discarded (plain round-robin placement).  The probe
// allocates ~32 MB once per device at the first call (not on the hot path).  Opt-in (KD_DIE_SCHED=1): measured at
// config 2 it cuts pass 1's DRAM reads 3.5 -> 3.1 GB per launch (pass 2: 4.0 -> 3.8) with no change in step time
// (profiles/r02_die_sched.md), so the default keeps the plain round-robin placement.
namespace {
struct DieMap {
  bool tried = false;
  uint8_t* dev = nullptr;  // [256] die of each %smid, device memory
  int pairs0 = 0, pairs1 = 0;
};
}  // namespace
static std::mutex g_die_mu;
static DieMap g_die[64];

static void probe_die_map(DieMap& m, int sms) {
  constexpr int kLines = 16, kSteps = 256, kWords = (32 << 20) / 4;
  unsigned* buf = nullptr;
  long long* d_off = nullptr;
  unsigned* d_out = nullptr;
  cudaStream_t st = nullptr;
  std::vector<unsigned> out((size_t)sms * (kLines + 1));
  // every SM must be free for one probe CTA: drain the device first (first call only)
  bool ok = cudaDeviceSynchronize() == cudaSuccess &&
            cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&buf, (size_t)kWords * 4) == cudaSuccess &&
            cudaMalloc(&d_off, kLines * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&d_out, out.size() * 4) == cudaSuccess;
  if (ok) {
    long long off[kLines];
    for (int l = 0; l < kLines; ++l) off[l] = (long long)l * (kWords / kLines) + 32ll * (l * 7 % 16);
    ok = cudaMemsetAsync(buf, 0, (size_t)kWords * 4, st) == cudaSuccess &&
         cudaMemcpyAsync(d_off, off, sizeof off, cudaMemcpyHostToDevice, st) == cudaSuccess &&
         launch_die_probe(buf, d_off, kLines, kSteps, d_out, sms, 200 * 1024, st) == cudaSuccess &&
         cudaMemcpyAsync(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaStreamSynchronize(st) == cudaSuccess;
  }
  if (buf) cudaFree(buf);
  if (d_off) cudaFree(d_off);
  if (d_out) cudaFree(d_out);
  if (st) cudaStreamDestroy(st);
  if (!ok) {
    cudaGetLastError();
    return;
  }
  // each line: its near set = the half of the SMs with the lowest latency (the dies are equal halves; near / far
  // differ by ~10-15% of ~280 cycles, with a spread inside each die, so a median split rather than a gap);
  // lines are oriented against the first one and the SMs' memberships voted
  std::vector<int> smid(sms), vote(sms, 0);
  for (int b = 0; b < sms; ++b) smid[b] = (int)out[(size_t)b * (kLines + 1)];
  {
    std::vector<int> ids(smid);
    std::sort(ids.begin(), ids.end());
    if (std::unique(ids.begin(), ids.end()) != ids.end()) return;  // an SM ran two probe CTAs: not one per SM
  }
  std::vector<std::vector<char>> nears;
  for (int l = 0; l < kLines; ++l) {
    std::vector<int> order(sms);
    for (int b = 0; b < sms; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      return out[(size_t)x * (kLines + 1) + 1 + l] < out[(size_t)y * (kLines + 1) + 1 + l];
    });
    std::vector<char> near(sms, 0);
    for (int i = 0; i < sms / 2; ++i) near[order[i]] = 1;
    if (env_int("KD_DIE_DEBUG", 0) > 1)
      fprintf(stderr, "kd: die probe line %d: latency min %u median %u max %u\n", l,
              out[(size_t)order[0] * (kLines + 1) + 1 + l], out[(size_t)order[sms / 2] * (kLines + 1) + 1 + l],
              out[(size_t)order[sms - 1] * (kLines + 1) + 1 + l]);
    if (!nears.empty()) {
      int agree = 0;
      for (int b = 0; b < sms; ++b) agree += near[b] == nears[0][b];
      if (agree * 2 < sms)
        for (int b = 0; b < sms; ++b) near[b] ^= 1;
    }
    nears.push_back(near);
    for (int b = 0; b < sms; ++b) vote[b] += near[b] ? 1 : -1;
  }
  // lines must agree with the vote: a median split of a line homed evenly would be noise
  int used = 0;
  for (const auto& near : nears) {
    int agree = 0;
    for (int b = 0; b < sms; ++b) agree += (near[b] != 0) == (vote[b] > 0);
    used += agree * 10 >= sms * 9;  // >= 90% agreement
  }
  if (env_int("KD_DIE_DEBUG", 0)) fprintf(stderr, "kd: die probe: %d of %d lines split the SMs in two levels\n", used, kLines);
  if (used < 4) return;
  uint8_t table[256] = {0};
  int n0 = 0;
  for (int b = 0; b < sms; ++b) {
    if (smid[b] > 255) return;
    table[smid[b]] = vote[b] > 0 ? 0 : 1;
    n0 += vote[b] > 0;
  }
  // SM pairs (2k, 2k+1) run the clusters of two: they must share a die, and the dies must be equal halves
  for (int b = 0; b < sms; ++b)
    if ((smid[b] ^ 1) < 256 && table[smid[b]] != table[smid[b] ^ 1]) {
      bool partner_seen = false;
      for (int c = 0; c < sms; ++c) partner_seen |= smid[c] == (smid[b] ^ 1);
      if (partner_seen) return;
    }
  if (n0 % 2 || (sms - n0) % 2 || std::abs(n0 - (sms - n0)) > 8) return;
  uint8_t* d = nullptr;
  if (cudaMalloc(&d, 256) != cudaSuccess || cudaMemcpy(d, table, 256, cudaMemcpyHostToDevice) != cudaSuccess) {
    if (d) cudaFree(d);
    cudaGetLastError();
    return;
  }
  m.dev = d;
  m.pairs0 = n0 / 2;
  m.pairs1 = (sms - n0) / 2;
  if (env_int("KD_DIE_DEBUG", 0)) {
    fprintf(stderr, "kd: die map from %d/%d probe lines: %d + %d SMs; die of smid 0..%d:", used, kLines, n0, sms - n0,
            sms - 1);
    for (int i = 0; i < sms && i < 256; ++i) fprintf(stderr, "%d", table[i]);
    fprintf(stderr, "\n");
  }
}

// The device's die map (probed on first use), or NULL.  Not probed while `stream` is being captured into a graph
// (the probe allocates and synchronises); the capture then runs with plain placement.
static const DieMap* die_map_for(cudaStream_t stream, int sms) {
  static const int enabled = env_int("KD_DIE_SCHED", 0);
  if (!enabled) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_die_mu);
  DieMap& m = g_die[dev & 63];
  if (!m.tried) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    m.tried = true;
    probe_die_map(m, sms);
  }
  return m.dev ? &m : nullptr;
}

// Die-aware static makespan: die d's splits [d ? s0 : 0, d ? s : s0) over its w_d worker slots, token tiles of a split
// consecutive (the units the kernel deals to each die).
static double pass_makespan_die(int m_tiles, int s, int s0, int v_tiles, int w0, int w1) {
  double worst = 0;
  for (int d = 0; d < 2; ++d) {
    const int sb = d ? s0 : 0, se = d ? s : s0, W = d ? w1 : w0;
    const int units = (se - sb) * m_tiles;
    for (int c = 0; c < W && c < units; ++c) {
      double t = 0;
      for (int j = c; j < units; j += W) {
        const int sp = sb + j / m_tiles;
        t += (double)((long long)(sp + 1) * v_tiles / s - (long long)sp * v_tiles / s) + 0.1;
      }
      if (t > worst) worst = t;
    }
  }
  return worst;
}

static void choose_split_die(int m_tiles, int v_tiles, int w0, int w1, int& best_s, int& best_s0) {
  static std::mutex mu;
  static std::unordered_map<long long, long long> memo;
  const long long key = ((long long)m_tiles << 44) | ((long long)v_tiles << 20) | ((long long)w0 << 10) | w1;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) { best_s = (int)(it->second >> 20); best_s0 = (int)(it->second & 0xFFFFF); return; }
  }
  double best = 1e300;
  best_s = 2;
  best_s0 = 1;
  const int smax = v_tiles < 160 ? v_tiles : 160;
  for (int s = 2; s <= smax; ++s) {
    if ((long long)s * m_tiles < w0 + w1) continue;  // every worker slot of both dies gets a unit: the grid is all SMs
    const int base = (int)((long long)s * w0 / (w0 + w1));
    for (int s0 = std::max(1, base - 1); s0 <= std::min(s - 1, base + 1); ++s0) {
      const double c = pass_makespan_die(m_tiles, s, s0, v_tiles, w0, w1);
      if (c < best * 0.999) { best = c; best_s = s; best_s0 = s0; }
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  memo[key] = ((long long)best_s << 20) | best_s0;
}

static int choose_n_split_search(int m_tiles, int v_tiles, int sms);
// memoised: the makespan search is O(160² · m_tiles) host work (~2 ms at 32 token tiles), and every entry point plans
// twice per call (kd_workspace_size + the call)
static int choose_n_split(int m_tiles, int v_tiles, int sms) {
  static std::mutex mu;
  static std::unordered_map<long long, int> memo;
  const long long key = ((long long)m_tiles << 42) | ((long long)v_tiles << 16) | (long long)sms;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  const int best = choose_n_split_search(m_tiles, v_tiles, sms);
  std::lock_guard<std::mutex> lk(mu);
  memo[key] = best;
  return best;
}

static int choose_n_split_search(int m_tiles, int v_tiles, int sms) {
  int best = 1;
  double best_cost = 1e300;
  const int smax = v_tiles < 160 ? v_tiles : 160;
  for (int s = 1; s <= smax; ++s) {
    const double c = pass_makespan(m_tiles, s, v_tiles, sms);
    if (c < best_cost * 0.999) { best_cost = c; best = s; }
  }
  return best;
}

// Split-K factor of the dh GEMM: units = m_tiles * n_tiles * k over a persistent grid of `workers` (SMs or SM
// pairs).  Cost in K-block times (1024 cycles: one 64-deep K block of a full-rate tile): waves x (K blocks per
// unit + ~2 fill/drain) + the split-K reduction re-reading (k - 1) extra fp32 slabs of M x N (~3.4 MB per K-block
// time at HBM speed).  At c2 (64 tile units on 74 pairs) this picks k = 8: 7 full waves instead of one 86%-full one.
static int choose_k_split(int m_tiles, int n_tiles, int kbs, int workers, long long M, long long N) {
  int best = 1;
  double best_cost = 1e300;
  const double slab_kb = (double)M * (double)N * 4.0 / 3.4e6;
  for (int k = 1; k <= 16 && k <= kbs; ++k) {
    const long long units = (long long)m_tiles * n_tiles * k;
    const double waves = (double)((units + workers - 1) / workers);
    const double c = waves * ((double)((kbs + k - 1) / k) + 2.0) + slab_kb * (k - 1);
    if (c < best_cost * 0.999) { best_cost = c; best = k; }
  }
  return best;
}

static kd_status validate(const kd_problem* p, bool require_full_vocab) {
  if (!p) return fail(KD_ERR_INVALID_ARG, "problem is NULL");
  for (int i = 0; i < 3; ++i)
    if (p->reserved[i] != 0) return fail(KD_ERR_INVALID_ARG, "reserved fields must be zero");
  if (p->stage_logits != 0 && p->stage_logits != 1)
    return fail(KD_ERR_INVALID_ARG, "stage_logits must be 0 or 1 (got %d)", p->stage_logits);
  if (p->grad_precision != KD_GRAD_SPLIT_BF16 && p->grad_precision != KD_GRAD_BF16)
    return fail(KD_ERR_INVALID_ARG, "unknown grad_precision %d", p->grad_precision);
  if (!(p->temperature > 0.f) || !std::isfinite(p->temperature))
    return fail(KD_ERR_INVALID_ARG, "temperature must be finite and > 0 (got %g)", (double)p->temperature);
  if (p->kind < KD_FKL || p->kind > KD_TVD) return fail(KD_ERR_INVALID_ARG, "unknown divergence kind %d", p->kind);
  if (p->kind == KD_JSD && !(p->jsd_beta > 0.f && p->jsd_beta < 1.f))
    return fail(KD_ERR_INVALID_ARG, "jsd_beta must lie in (0,1) (got %g)", (double)p->jsd_beta);
  if (!std::isfinite(p->loss_scale)) return fail(KD_ERR_INVALID_ARG, "loss_scale must be finite");
  if (p->n_tokens < 0 || p->n_tokens > (1ll << 30)) return fail(KD_ERR_SHAPE, "n_tokens out of range");
  if (p->d_t < 64 || p->d_s < 64 || p->d_t % 64 || p->d_s % 64 || p->d_t > 65536 || p->d_s > 65536)
    return fail(KD_ERR_SHAPE, "d_t and d_s must be positive multiples of 64 (got %d, %d)", p->d_t, p->d_s);
  if (p->vocab < 1 || p->v_begin < 0 || p->v_end > p->vocab || p->v_end <= p->v_begin)
    return fail(KD_ERR_SHAPE, "bad vocabulary range [%lld, %lld) of %lld", (long long)p->v_begin,
                (long long)p->v_end, (long long)p->vocab);
  if (p->v_end - p->v_begin > (1ll << 26)) return fail(KD_ERR_SHAPE, "vocabulary shard too large");
  if (require_full_vocab && (p->v_begin != 0 || p->v_end != p->vocab))
    return fail(KD_ERR_SHAPE, "kd_fused_fwd_bwd needs the full vocabulary; use kd_vocab_* for shards");
  if (p->chunk_tokens < 0) return fail(KD_ERR_SHAPE, "chunk_tokens must be >= 0");
  return KD_OK;
}

// Entry points other than kd_fused_fwd_bwd: the staged variant is not implemented there (kdfused.h stage_logits).
static kd_status validate_unstaged(const kd_problem* p, bool require_full_vocab) {
  const kd_status st = validate(p, require_full_vocab);
  if (st != KD_OK) return st;
  if (p->stage_logits) return fail(KD_ERR_UNSUPPORTED, "stage_logits is implemented by kd_fused_fwd_bwd only");
  return KD_OK;
}

static Plan make_plan(const kd_problem* p) {
  Plan P{};
  P.N = (int)p->n_tokens;
  P.d_t = p->d_t;
  P.d_s = p->d_s;
  P.V_r = (int)(p->v_end - p->v_begin);
  P.kind = p->kind;
  P.fix = (p->kind == KD_JSD || p->kind == KD_TVD);
  P.g_planes = p->grad_precision == KD_GRAD_BF16 ? 1 : 2;
  P.num_sms = device_sms();
  P.cg = cta_group();
  P.bn = pass_bn();
  const int bmt = kBM * P.cg;  // token rows per fused-pass work tile
  // Default chunk: the fused passes re-read the chunk's hidden rows for every vocab tile, so they must stay
  // L2-resident next to the streaming heads, while every chunk streams both heads once per pass from DRAM.  ~36 MiB
  // of H_t|H_s per chunk, at most 4096 tokens: 3072 at configs 2/3/5, 4096 at config 4.  Measured with the pass-2
  // staging L2 hints (profiles/r02_ab.md, r02b_ab7/ab8): c2 3072 vs 2048 +0.8 / +2.3% on two boxes (2560 and 3584
  // lose: 80 / 112 dh-GEMM tiles quantise badly on 74 pair workers), c3 RKL +0.9%, c5 +1.4%; c4 4096 vs 5120 / 6144
  // +0.8 / +0.6%.  (Round 1, without the hints, preferred 24 MiB: c2 at 8192 tokens ran 12% slower than at 2048.)
  // KD_CHUNK_TOKENS overrides (experiments).
  static const int nc_env = env_int("KD_CHUNK_TOKENS", 0);
  int nc_default = (int)((36ll << 20) / ((long long)(P.d_t + P.d_s) * 2));
  nc_default = nc_default < 1024 ? 1024 : (nc_default > 4096 ? 4096 : nc_default);
  if (nc_env > 0) nc_default = nc_env;
  int nc = p->chunk_tokens > 0 ? p->chunk_tokens : nc_default;
  const int n_pad = ((P.N + bmt - 1) / bmt) * bmt;
  if (nc > n_pad) nc = n_pad;
  nc = ((nc + bmt - 1) / bmt) * bmt;
  if (nc < bmt) nc = bmt;
  P.Nc = nc;
  P.n_chunks = (P.N + nc - 1) / nc;
  P.m_tiles_c = nc / bmt;
  P.v_tiles = (P.V_r + P.bn - 1) / P.bn;
  {
    // vocab splits: die-aware placement needs both dies' worker slots filled (all SMs, an even number of pairs);
    // its split count is planned per die even when the map turns out unavailable at run time (the workspace depends
    // on n_split), where the same splits are then dealt round-robin
    static const int die_env = env_int("KD_DIE_SCHED", 0);
    const int workers = P.num_sms / P.cg;
    P.die_map = nullptr;
    if (die_env && P.cg == 2 && P.bn == 256 && workers % 2 == 0 && (long long)P.m_tiles_c * P.v_tiles >= 2ll * workers) {
      choose_split_die(P.m_tiles_c, P.v_tiles, workers / 2, workers / 2, P.n_split, P.die_s0);
      P.die_w0 = workers / 2;
    } else {
      P.n_split = choose_n_split(P.m_tiles_c, P.v_tiles, workers);
      P.die_s0 = P.n_split;
      P.die_w0 = 0;  // plain placement (pass_params: die_w0 = the grid's workers)
    }
  }
  P.g_ld = ((P.V_r + 63) / 64) * 64;
  P.stage = p->stage_logits != 0;
  {
    // staged G kernel: one 128-thread block per (128·R rows, vocab slot); ~8 blocks per SM in one wave
    const int R = stage_rows(), row_blocks = (P.Nc + 128 * R - 1) / (128 * R), nch = P.g_ld / stage_cols();
    static const int bps = env_int("KD_STAGE_BPS", 8);  // target resident blocks per SM (A/B knob)
    int s = (bps * P.num_sms + row_blocks - 1) / row_blocks;
    P.n_gslots = P.stage ? (s < 1 ? 1 : (s > nch ? nch : s)) : P.n_split * epi_parts(2, P.kind);
  }
  const int slots_max = std::max(P.n_gslots, P.n_split * epi_parts(2, P.kind));
  P.k_split = choose_k_split((P.Nc + kBM * gemm_cg() - 1) / (kBM * gemm_cg()), (P.d_s + kGemmBN - 1) / kGemmBN,
                             (P.V_r + kBK - 1) / kBK, P.num_sms / gemm_cg(), P.Nc, P.d_s);
  static const int ks_env = env_int("KD_DH_KSPLIT", 0);  // A/B override of the dh GEMM's split-K factor
  if (ks_env > 0) P.k_split = ks_env;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  P.off_neff = take(8);
  P.off_nonfinite = take(8);
  P.off_idx = take((size_t)P.N * 4);
  P.off_ht = take((size_t)P.N * P.d_t * 2);
  P.off_hs = take((size_t)P.N * P.d_s * 2);
  P.off_part = take((size_t)5 * P.n_split * epi_parts(1, P.kind) * P.Nc * 4);
  P.off_fstats = take((size_t)kFstatPlanes * P.Nc * 4);
  // JSD/TVD: K and J partials; FKL: the loss partials of pass 2 (plane 0)
  P.off_kpart = take((P.fix || P.kind == KD_FKL) ? (size_t)2 * slots_max * P.Nc * 4 : 0);
  P.off_kfin = take(P.fix ? (size_t)P.Nc * 4 : 0);
  P.off_ghi = take((size_t)P.Nc * P.g_ld * 2);
  P.off_glo = take(P.g_planes == 2 ? (size_t)P.Nc * P.g_ld * 2 : 0);
  P.off_ga = take(P.fix ? (size_t)P.Nc * P.g_ld * 4 : 0);
  P.off_gb = take(P.fix ? (size_t)P.Nc * P.g_ld * 4 : 0);
  P.off_dhp = take((size_t)P.k_split * P.Nc * P.d_s * 4);
  P.off_corr_v = take(P.fix ? 0 : (size_t)slots_max * kCorrSlots * P.Nc * 4);
  P.off_corr_r = take(P.fix ? 0 : (size_t)slots_max * kCorrSlots * P.Nc * 4);
  P.off_zscr = take((size_t)P.num_sms * P.bn * kBM * 4);  // decoupled pass 2 staging (19 MB: L2-resident)
  P.off_tkr_v = take((size_t)P.Nc * kTopK * 4);  // top-k baseline: residual slots of the k support entries
  P.off_tkr_r = take((size_t)P.Nc * kTopK * 4);
  P.off_zst = take(P.stage ? (size_t)2 * P.g_ld * P.Nc * 4 : 0);  // staged logits of one chunk (2.5 GB at c2)
  P.off_sched = take(16);  // die-aware placement counters (PassParams::sched), zeroed before each pass launch
  P.total = o;
  // kd_teacher_topk's candidate lists [n_split*parts][Nc][kTopK] (values, indices) reuse the G / dh scratch, which
  // that call does not touch (extended only if a tiny vocabulary makes the scratch smaller than the lists)
  const size_t tk_bytes = align256((size_t)P.n_split * epi_parts(1, KIND_TOPK) * P.Nc * kTopK * 4);
  P.off_tkv = P.off_ghi;
  P.off_tki = P.off_ghi + tk_bytes;
  if (P.off_tki + tk_bytes > P.total) P.total = P.off_tki + tk_bytes;
  return P;
}

static bool aligned16(const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; }

template <typename T>
static T* ws_at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// ------------------------------------------------------------------------------------ the call sequence
namespace {
struct Ctx {
  const kd_problem* p;
  Plan P;
  cudaStream_t s;
  void* ws;
  const __nv_bfloat16 *ht, *hs, *Wt, *Ws;  // possibly packed H
  const int* idx;                          // NULL = identity (no mask)
  int* n_eff;
  long long* nonfinite;
  CUtensorMap maps[4];
};
}  // namespace

// teacher_only (kd_teacher_lse): h_s / W_s are absent; the student maps alias the teacher's and are never read.
// student_only (kd_topk_fwd_bwd): h_t / W_t are absent; the teacher maps alias the student's and are never read.
static kd_status prologue(Ctx& c, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                          const uint8_t* mask, int64_t* n_nonfinite, bool teacher_only = false,
                          bool student_only = false) {
  const Plan& P = c.P;
  c.n_eff = ws_at<int>(c.ws, P.off_neff);
  c.nonfinite = n_nonfinite ? reinterpret_cast<long long*>(n_nonfinite) : ws_at<long long>(c.ws, P.off_nonfinite);
  KD_CUDA(cudaMemsetAsync(c.nonfinite, 0, sizeof(long long), c.s));
  c.Wt = static_cast<const __nv_bfloat16*>(W_t);
  c.Ws = static_cast<const __nv_bfloat16*>(W_s);
  if (mask) {
    int* idx = ws_at<int>(c.ws, P.off_idx);
    KD_LAUNCH(K_COMPACT, launch_compact(mask, P.N, idx, c.n_eff, c.s));
    auto* pt = ws_at<__nv_bfloat16>(c.ws, P.off_ht);
    auto* ps = ws_at<__nv_bfloat16>(c.ws, P.off_hs);
    if (!student_only)
      KD_LAUNCH(K_GATHER, launch_gather(static_cast<const __nv_bfloat16*>(h_t), P.d_t, pt, P.d_t, P.N, idx, c.n_eff, c.s));
    if (!teacher_only)
      KD_LAUNCH(K_GATHER, launch_gather(static_cast<const __nv_bfloat16*>(h_s), P.d_s, ps, P.d_s, P.N, idx, c.n_eff, c.s));
    c.ht = pt;
    c.hs = ps;
    c.idx = idx;
  } else {
    KD_LAUNCH(K_COMPACT, launch_compact(nullptr, P.N, nullptr, c.n_eff, c.s));
    c.ht = static_cast<const __nv_bfloat16*>(h_t);
    c.hs = static_cast<const __nv_bfloat16*>(h_s);
    c.idx = nullptr;
  }
  kd_status st;
  if (student_only) {
    if ((st = make_map(&c.maps[2], c.hs, P.d_s, P.N, (uint64_t)P.d_s * 2, kBK, kBM)) != KD_OK) return st;
    if ((st = make_map(&c.maps[3], c.Ws, P.d_s, P.V_r, (uint64_t)P.d_s * 2, kBK, P.bn / P.cg)) != KD_OK) return st;
    c.maps[0] = c.maps[2];
    c.maps[1] = c.maps[3];
    return KD_OK;
  }
  if ((st = make_map(&c.maps[0], c.ht, P.d_t, P.N, (uint64_t)P.d_t * 2, kBK, kBM)) != KD_OK) return st;
  if ((st = make_map(&c.maps[1], c.Wt, P.d_t, P.V_r, (uint64_t)P.d_t * 2, kBK, P.bn / P.cg)) != KD_OK) return st;
  if (teacher_only) {
    c.maps[2] = c.maps[0];
    c.maps[3] = c.maps[1];
    return KD_OK;
  }
  if ((st = make_map(&c.maps[2], c.hs, P.d_s, P.N, (uint64_t)P.d_s * 2, kBK, kBM)) != KD_OK) return st;
  if ((st = make_map(&c.maps[3], c.Ws, P.d_s, P.V_r, (uint64_t)P.d_s * 2, kBK, P.bn / P.cg)) != KD_OK) return st;
  return KD_OK;
}

static int pass_grid(const Plan& P) {  // CTAs (a multiple of the CTA group)
  const int units = P.m_tiles_c * P.n_split;
  const int workers = P.num_sms / P.cg;
  return (units < workers ? units : workers) * P.cg;
}

static PassParams pass_params(const Ctx& c, int row0) {
  const Plan& P = c.P;
  const kd_problem* p = c.p;
  PassParams pp{};
  pp.n_eff = c.n_eff;
  pp.row0 = row0;
  pp.n_rows = P.Nc;
  pp.kb_t = P.d_t / kBK;
  pp.kb_s = P.d_s / kBK;
  pp.v_tiles = P.v_tiles;
  pp.V_r = P.V_r;
  pp.n_split = P.n_split;
  pp.alpha = (float)(1.4426950408889634 / (double)p->temperature);
  pp.part = ws_at<float>(c.ws, P.off_part);
  pp.part_plane = (long long)P.n_split * epi_parts(1, P.kind) * P.Nc;
  pp.fstats = ws_at<float>(c.ws, P.off_fstats);
  const double cscale = (double)p->loss_scale / (double)p->temperature;
  pp.gscale = (float)(p->kind == KD_RKL ? cscale * 0.6931471805599453 : cscale);
  pp.beta = p->jsd_beta;
  pp.g_hi = ws_at<__nv_bfloat16>(c.ws, P.off_ghi);
  pp.g_lo = P.g_planes == 2 ? ws_at<__nv_bfloat16>(c.ws, P.off_glo) : nullptr;
  pp.g_a = P.fix ? ws_at<float>(c.ws, P.off_ga) : nullptr;
  pp.g_b = P.fix ? ws_at<float>(c.ws, P.off_gb) : nullptr;
  pp.g_ld = P.g_ld;
  pp.kpart = (P.fix || P.kind == KD_FKL) ? ws_at<float>(c.ws, P.off_kpart) : nullptr;
  pp.corr_v = P.fix ? nullptr : ws_at<int>(c.ws, P.off_corr_v);
  pp.corr_r = P.fix ? nullptr : ws_at<float>(c.ws, P.off_corr_r);
  pp.zscr = ws_at<float>(c.ws, P.off_zscr);
  pp.dbg = reinterpret_cast<unsigned long long*>(g_dbg_ptr);
  static const int l2_hints = env_int("KD_L2_HINTS", 0);  // measured neutral-to-negative (profiles/r01_ncu_pass_pair256.md)
  pp.l2_hints = l2_hints;
  pp.side_lo = 0;
  pp.side_hi = 2;
  pp.tk_val = ws_at<float>(c.ws, P.off_tkv);
  pp.tk_idx = ws_at<int>(c.ws, P.off_tki);
  pp.sched = ws_at<int>(c.ws, P.off_sched);
  pp.die_map = P.die_map;
  pp.die_w0 = P.die_map ? P.die_w0 : pass_grid(P) / P.cg;
  pp.die_s0 = P.die_map ? P.die_s0 : P.n_split;
  return pp;
}

// Die-aware placement for this call when the plan allows it and the device's map matches (PassParams::die_map).
static void attach_die(Ctx& c) {
  if (c.P.die_w0 <= 0) return;
  const DieMap* m = die_map_for(c.s, c.P.num_sms);
  if (m && m->pairs0 == c.P.die_w0 && m->pairs1 == c.P.num_sms / c.P.cg - c.P.die_w0 &&
      pass_grid(c.P) == c.P.num_sms)
    c.P.die_map = m->dev;
}

// RKL's pass 1: decoupled with the teacher half-tile staged (default) or the coupled form (KD_RKL_P1_COUPLED=1, A/B).
static bool rkl_p1_coupled() {
  static const bool v = env_int("KD_RKL_P1_COUPLED", 0) != 0;
  return v;
}

// One fused-pass launch (the die-aware placement counters are zeroed first).
static kd_status run_pass(Ctx& c, int pass, int kind, bool coupled, const PassParams& pp) {
  if (pp.die_map) KD_CUDA(cudaMemsetAsync(pp.sched, 0, 16, c.s));
  KD_LAUNCH(pass == 1 ? K_PASS1 : K_PASS2,
            launch_pass(pass, kind, coupled, c.P.cg, c.P.bn, c.maps, pp, pass_grid(c.P), c.s));
  return KD_OK;
}


// pass 2 for one chunk whose final per-token statistics are already in fstats: G (FKL/RKL) or the two JSD/TVD
// planes + partial K, J.
static kd_status grad_chunk(Ctx& c, int row0, int side_lo = 0) {
  const Plan& P = c.P;
  PassParams pp = pass_params(c, row0);
  pp.side_lo = side_lo;  // 1: student-only pass 2 (top-k baseline: G = gscale·q, the teacher put back afterwards)
  static const bool p2_coupled = env_int("KD_P2_COUPLED", 0) != 0;
  kd_status st = run_pass(c, 2, P.kind, p2_coupled && side_lo == 0, pp);
  if (st != KD_OK) return st;
  return KD_OK;
}

// After pass 2: [JSD/TVD fix-up with the local K partials, or with the P ranks' per-token totals kj_ranks]
// + dh GEMM (+ split-K reduce) + dW GEMM for one chunk.
static kd_status finish_chunk(Ctx& c, int row0, float* loss, const RowDst& dh, float* dW, const float* kj_ranks,
                              int n_ranks, int topk = 0, long long kj_plane = -1) {
  const Plan& P = c.P;
  const kd_problem* p = c.p;
  PassParams pp = pass_params(c, row0);
  if (P.fix) {
    const double cscale = (double)p->loss_scale / (double)p->temperature;
    const float scale = (float)(P.kind == KD_JSD ? cscale * (1.0 - (double)p->jsd_beta) * 0.6931471805599453
                                                 : 0.5 * cscale);
    KD_LAUNCH(K_KFIX, launch_kfix(pp.kpart, P.n_gslots, P.Nc, row0, c.n_eff, P.kind, p->jsd_beta,
                          ws_at<float>(c.ws, P.off_kfin), loss, c.idx, c.nonfinite, pp.g_a, pp.g_b, P.g_ld, scale,
                          pp.g_hi, pp.g_lo, P.num_sms, kj_ranks, n_ranks, kj_plane >= 0 ? kj_plane : (long long)P.N,
                          c.s));
  }
  kd_status st;
  if (dW) {
    // dW_s += Gᵀ · H_s first: it reads the full G, before the extracted entries are taken out for the dh GEMM
    CUtensorMap ma_hi, ma_lo, mh;
    // dW_s += Gᵀ · H_s: A = Gᵀ [g_ld][Nc] is K-major (K = tokens), B = H_s chunk MN-major
    if ((st = make_map(&ma_hi, pp.g_hi, P.Nc, P.g_ld, (uint64_t)P.Nc * 2, kBK, kBM)) != KD_OK) return st;
    if (P.g_planes == 2 && (st = make_map(&ma_lo, pp.g_lo, P.Nc, P.g_ld, (uint64_t)P.Nc * 2, kBK, kBM)) != KD_OK)
      return st;
    const int rows_left = P.N - row0;
    if ((st = make_map(&mh, c.hs + (size_t)row0 * P.d_s, P.d_s, rows_left, (uint64_t)P.d_s * 2, 64, kBK)) != KD_OK)
      return st;
    GemmParams wp{};
    wp.M = P.V_r;
    wp.N = P.d_s;
    wp.K = P.Nc;
    wp.dyn_dim = DYN_K;
    wp.dyn = c.n_eff;
    wp.dyn_base = row0;
    wp.k_split = 1;
    wp.kb_per_acc = kb_per_acc();
    wp.out = dW;
    wp.out_ld = P.d_s;
    wp.out_split_stride = 0;
    KD_LAUNCH(K_GEMM_DW, launch_gemm(false, true, P.g_planes, EPI_ACCUM, gemm_cg(), &ma_hi,
                                     P.g_planes == 2 ? &ma_lo : nullptr, &mh, wp, P.num_sms, c.s));
  }
  // FKL/RKL: pass 2's largest entries per (row, slot) leave the dh GEMM (restored exactly by k_reduce_dh)
  if (!P.fix)
    KD_LAUNCH(K_REDUCE_DH, launch_extract_zero(pp.corr_v, pp.corr_r, P.n_gslots * kCorrSlots, P.Nc, row0, c.n_eff,
                                               pp.g_hi, pp.g_lo, c.s));
  // dh_s rows of this chunk: [G_hi | G_lo] · W_s  (K = V_r); the scratch holds Gᵀ [g_ld][Nc], i.e. the A operand
  // [tokens, V] is MN-major; W_s [V_r, d_s] is the MN-major B operand.  Split-K slabs, then reduce + scatter.
  CUtensorMap mg_hi, mg_lo, mw;
  if ((st = make_map(&mg_hi, pp.g_hi, P.Nc, P.g_ld, (uint64_t)P.Nc * 2, 64, kBK)) != KD_OK) return st;
  if (P.g_planes == 2 && (st = make_map(&mg_lo, pp.g_lo, P.Nc, P.g_ld, (uint64_t)P.Nc * 2, 64, kBK)) != KD_OK)
    return st;
  if ((st = make_map(&mw, c.Ws, P.d_s, P.V_r, (uint64_t)P.d_s * 2, 64, kBK)) != KD_OK) return st;
  GemmParams gp{};
  gp.M = P.Nc;
  gp.N = P.d_s;
  gp.K = P.V_r;
  gp.dyn_dim = DYN_M;
  gp.dyn = c.n_eff;
  gp.dyn_base = row0;
  gp.k_split = P.k_split;
  gp.kb_per_acc = kb_per_acc();
  gp.out = ws_at<float>(c.ws, P.off_dhp);
  gp.out_ld = P.d_s;
  gp.out_split_stride = (long long)P.Nc * P.d_s;
  KD_LAUNCH(K_GEMM_DH, launch_gemm(true, true, P.g_planes, EPI_STORE, gemm_cg(), &mg_hi,
                                   P.g_planes == 2 ? &mg_lo : nullptr, &mw, gp, P.num_sms, c.s));
  KD_LAUNCH(K_REDUCE_DH, launch_reduce_dh(gp.out, gp.out_split_stride, P.k_split, P.d_s, P.Nc, row0, c.n_eff, c.idx, dh,
                                          P.fix ? nullptr : pp.corr_v, P.fix ? nullptr : pp.corr_r,
                                          P.n_gslots * kCorrSlots, c.Ws, c.s,
                                          topk ? ws_at<int>(c.ws, P.off_tkr_v) : nullptr,
                                          topk ? ws_at<float>(c.ws, P.off_tkr_r) : nullptr, topk));
  return KD_OK;
}

static kd_status backward_chunk(Ctx& c, int row0, float* loss, const RowDst& dh, float* dW) {
  kd_status st = grad_chunk(c, row0);
  if (st != KD_OK) return st;
  return finish_chunk(c, row0, loss, dh, dW, nullptr, 0);
}

static kd_status check_common(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                              const void* W_s, float* loss, float* dh, float* dW, void* ws, size_t ws_bytes,
                              const Plan& P, bool local_out = true) {
  // local_out = false: the peer exchange (kd_vocab_backward_p2p) sends dh / the FKL loss to the owners' slots
  if (P.N > 0 && (!h_t || !h_s || (local_out && (!loss || !dh))))
    return fail(KD_ERR_INVALID_ARG, "NULL input/output pointer");
  if (!W_t || !W_s) return fail(KD_ERR_INVALID_ARG, "NULL LM-head pointer");
  if (p->want_dW && !dW) return fail(KD_ERR_INVALID_ARG, "want_dW set but dW_s is NULL");
  const void* ptrs[] = {h_t, W_t, h_s, W_s, loss, dh, dW};
  for (const void* x : ptrs)
    if (x && !aligned16(x)) return fail(KD_ERR_ALIGNMENT, "pointers must be 16-byte aligned");
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace must be non-NULL and 256-byte aligned");
  if (ws_bytes < P.total)
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  return KD_OK;
}

extern "C" {

kd_status kd_check_problem(const kd_problem* p) { return validate(p, false); }

size_t kd_workspace_size(const kd_problem* p) {
  if (validate(p, false) != KD_OK) return 0;
  return make_plan(p).total;
}

// The whole path on one GPU.  lse_t != NULL: the teacher's per-token base-2 LSE record [2][N] (kd_teacher_lse) is
// supplied, so pass 1 sweeps the student head only.
static kd_status fused_impl(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                            const uint8_t* mask, const float* lse_t, float* loss, float* dh_s, float* dW_s,
                            int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = validate(p, true);
  if (st != KD_OK) return st;
  if (lse_t && p->kind == KD_RKL)
    return fail(KD_ERR_UNSUPPORTED, "kd_fused_fwd_bwd_lse: RKL's gradient needs its loss (a cross term of both heads) "
                                    "before pass 2, so pass 1 cannot skip the teacher head");
  if (lse_t && !aligned16(lse_t)) return fail(KD_ERR_ALIGNMENT, "lse_t must be 16-byte aligned");
  if (lse_t && p->stage_logits)
    return fail(KD_ERR_UNSUPPORTED, "stage_logits needs the teacher logits from pass 1; kd_fused_fwd_bwd_lse skips them");
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  float* dW = p->want_dW ? dW_s : nullptr;
  if ((st = check_common(p, h_t, W_t, h_s, W_s, loss, dh_s, dW, workspace, workspace_bytes, c.P)) != KD_OK)
    return st;
  const Plan& P = c.P;
  if (dW && !p->accumulate_dW) KD_CUDA(cudaMemsetAsync(dW, 0, (size_t)P.V_r * P.d_s * 4, c.s));
  if (P.N == 0) {
    if (n_nonfinite) KD_CUDA(cudaMemsetAsync(n_nonfinite, 0, 8, c.s));
    return KD_OK;
  }
  if ((st = prologue(c, h_t, W_t, h_s, W_s, mask, n_nonfinite)) != KD_OK) return st;
  if (mask) KD_LAUNCH(K_ZERO, launch_zero_masked(mask, P.N, loss, dh_s, P.d_s, c.s));
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    PassParams pp = pass_params(c, row0);
    // decoupled pass 1 (independent teacher / student LSEs) for FKL/JSD/TVD; RKL needs its loss (the cross term U,
    // both logits per element) in pass 2: decoupled with the teacher half staged (default) or coupled
    const bool coupled = P.kind == KD_RKL;
    if (lse_t) pp.side_lo = 1;  // student half-tiles only
    if (P.stage) pp.zst = ws_at<float>(c.ws, P.off_zst);
    if ((st = run_pass(c, 1, P.kind, coupled && rkl_p1_coupled(), pp)) != KD_OK) return st;
    KD_LAUNCH(K_MERGE, launch_merge(pp.part, pp.part_plane, P.Nc, P.n_split * epi_parts(1, P.kind), P.Nc, row0, c.n_eff, P.kind, 0,
                           ws_at<float>(c.ws, P.off_fstats), loss, nullptr, (long long)P.N, c.idx, 0, c.nonfinite,
                           coupled ? 1 : 0, c.s, lse_t));
    if (P.stage) {
      // staged variant: G from the chunk's staged logits (HBM-bound) instead of pass 2's second tensor sweep
      StageParams sp{};
      sp.n_eff = c.n_eff;
      sp.row0 = row0;
      sp.n_rows = P.Nc;
      sp.V_r = P.V_r;
      sp.g_ld = P.g_ld;
      sp.alpha = pp.alpha;
      sp.gscale = pp.gscale;
      sp.beta = pp.beta;
      sp.zst = pp.zst;
      sp.fstats = pp.fstats;
      sp.g_hi = pp.g_hi;
      sp.g_lo = pp.g_lo;
      sp.g_a = pp.g_a;
      sp.g_b = pp.g_b;
      sp.kpart = pp.kpart;
      sp.corr_v = pp.corr_v;
      sp.corr_r = pp.corr_r;
      KD_LAUNCH(K_STAGE_GRAD, launch_stage_grad(P.kind, sp, P.n_gslots, c.s));
      if ((st = finish_chunk(c, row0, loss, local_rows(dh_s, P.d_s), dW, nullptr, 0)) != KD_OK) return st;
    } else if ((st = backward_chunk(c, row0, loss, local_rows(dh_s, P.d_s), dW)) != KD_OK) {
      return st;
    }
    if (P.kind == KD_FKL)
      KD_LAUNCH(K_MERGE, launch_loss_rows(pp.kpart, P.n_gslots, P.Nc, row0, c.n_eff, local_rows(loss, 1), c.idx,
                                          c.nonfinite, c.s));
  }
  return KD_OK;
}

kd_status kd_fused_fwd_bwd(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                           const void* W_s, const uint8_t* mask, float* loss, float* dh_s, float* dW_s,
                           int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, void* stream) {
  return fused_impl(p, h_t, W_t, h_s, W_s, mask, nullptr, loss, dh_s, dW_s, n_nonfinite, workspace, workspace_bytes,
                    stream);
}

kd_status kd_fused_fwd_bwd_lse(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                               const void* W_s, const uint8_t* mask, const float* lse_t, float* loss, float* dh_s,
                               float* dW_s, int64_t* n_nonfinite, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (p && p->n_tokens > 0 && !lse_t) return fail(KD_ERR_INVALID_ARG, "lse_t is NULL");
  return fused_impl(p, h_t, W_t, h_s, W_s, mask, p && p->n_tokens > 0 ? lse_t : nullptr, loss, dh_s, dW_s,
                    n_nonfinite, workspace, workspace_bytes, stream);
}

kd_status kd_teacher_lse(const kd_problem* p, const void* h_t, const void* W_t, const uint8_t* mask, float* lse_t,
                         void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = validate_unstaged(p, true);
  if (st != KD_OK) return st;
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  const Plan& P = c.P;
  if (P.N > 0 && (!h_t || !lse_t)) return fail(KD_ERR_INVALID_ARG, "NULL h_t / lse_t");
  if (!W_t) return fail(KD_ERR_INVALID_ARG, "NULL W_t");
  const void* ptrs[] = {h_t, W_t, lse_t};
  for (const void* x : ptrs)
    if (x && !aligned16(x)) return fail(KD_ERR_ALIGNMENT, "pointers must be 16-byte aligned");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255) || workspace_bytes < P.total)
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace must be 256-byte aligned and >= %zu bytes", P.total);
  if (P.N == 0) return KD_OK;
  if ((st = prologue(c, h_t, W_t, nullptr, nullptr, mask, nullptr, true)) != KD_OK) return st;
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    PassParams pp = pass_params(c, row0);
    pp.side_hi = 1;  // teacher half-tiles only (the same sweep as the teacher side of the fused decoupled pass 1)
    if ((st = run_pass(c, 1, KD_FKL, false, pp)) != KD_OK) return st;
    KD_LAUNCH(K_MERGE, launch_merge(pp.part, pp.part_plane, P.Nc, P.n_split * epi_parts(1, KD_FKL), P.Nc, row0,
                                    c.n_eff, KD_FKL, 2, nullptr, nullptr, lse_t, (long long)P.N, c.idx, 0,
                                    c.nonfinite, 0, c.s));
  }
  return KD_OK;
}

kd_status kd_teacher_topk(const kd_problem* p, const void* h_t, const void* W_t, const uint8_t* mask, int32_t k,
                          int32_t* topk_idx, float* topk_val, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = validate_unstaged(p, true);
  if (st != KD_OK) return st;
  if (k < 1 || k > p->vocab) return fail(KD_ERR_INVALID_ARG, "k must lie in [1, vocab] (got %d)", k);
  if (k > kTopK) return fail(KD_ERR_UNSUPPORTED, "k = %d > %d (the register lists of the top-k pass)", k, kTopK);
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  const Plan& P = c.P;
  if (P.N > 0 && (!h_t || !topk_idx || !topk_val)) return fail(KD_ERR_INVALID_ARG, "NULL h_t / topk_idx / topk_val");
  if (!W_t) return fail(KD_ERR_INVALID_ARG, "NULL W_t");
  if ((h_t && !aligned16(h_t)) || !aligned16(W_t)) return fail(KD_ERR_ALIGNMENT, "h_t / W_t must be 16-byte aligned");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255) || workspace_bytes < P.total)
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace must be 256-byte aligned and >= %zu bytes", P.total);
  if (P.N == 0) return KD_OK;
  if ((st = prologue(c, h_t, W_t, nullptr, nullptr, mask, nullptr, true)) != KD_OK) return st;
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    PassParams pp = pass_params(c, row0);
    pp.side_hi = 1;  // teacher half-tiles only
    if ((st = run_pass(c, 1, KIND_TOPK, false, pp)) != KD_OK) return st;
    KD_LAUNCH(K_TOPK, launch_topk_merge(pp.tk_val, pp.tk_idx, P.n_split * epi_parts(1, KIND_TOPK), P.Nc, row0,
                                        c.n_eff, c.idx, k, (int)p->v_begin, topk_idx, topk_val, c.s));
  }
  return KD_OK;
}

kd_status kd_topk_fwd_bwd(const kd_problem* p, const void* h_s, const void* W_s, const uint8_t* mask, int32_t k,
                          const int32_t* topk_idx, const float* topk_val, float* loss, float* dh_s, float* dW_s,
                          int64_t* n_nonfinite, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = validate_unstaged(p, true);
  if (st != KD_OK) return st;
  if (p->kind != KD_FKL)
    return fail(KD_ERR_UNSUPPORTED, "kd_topk_fwd_bwd is forward KL only: RKL against a truncated teacher is +inf "
                                    "off the support (DESIGN.md R17)");
  if (k < 1 || k > p->vocab) return fail(KD_ERR_INVALID_ARG, "k must lie in [1, vocab] (got %d)", k);
  if (k > kTopK) return fail(KD_ERR_UNSUPPORTED, "k = %d > %d", k, kTopK);
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  float* dW = p->want_dW ? dW_s : nullptr;
  // h_t / W_t are not inputs of the top-k student: the student's own tensors stand in for the pointer checks
  if ((st = check_common(p, h_s, W_s, h_s, W_s, loss, dh_s, dW, workspace, workspace_bytes, c.P)) != KD_OK) return st;
  const Plan& P = c.P;
  if (P.N > 0 && (!topk_idx || !topk_val)) return fail(KD_ERR_INVALID_ARG, "NULL topk_idx / topk_val");
  if (dW && !p->accumulate_dW) KD_CUDA(cudaMemsetAsync(dW, 0, (size_t)P.V_r * P.d_s * 4, c.s));
  if (P.N == 0) {
    if (n_nonfinite) KD_CUDA(cudaMemsetAsync(n_nonfinite, 0, 8, c.s));
    return KD_OK;
  }
  if ((st = prologue(c, nullptr, nullptr, h_s, W_s, mask, n_nonfinite, false, true)) != KD_OK) return st;
  if (mask) KD_LAUNCH(K_ZERO, launch_zero_masked(mask, P.N, loss, dh_s, P.d_s, c.s));
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    PassParams pp = pass_params(c, row0);
    pp.side_lo = 1;  // student half-tiles only: LSE_s (the teacher's part of the record mirrors it, unused)
    if ((st = run_pass(c, 1, KD_FKL, false, pp)) != KD_OK) return st;
    KD_LAUNCH(K_MERGE, launch_merge(pp.part, pp.part_plane, P.Nc, P.n_split * epi_parts(1, P.kind), P.Nc, row0,
                                    c.n_eff, P.kind, 0, ws_at<float>(c.ws, P.off_fstats), loss, nullptr, 0, c.idx, 0,
                                    c.nonfinite, 0, c.s));
    if ((st = grad_chunk(c, row0, 1)) != KD_OK) return st;
    KD_LAUNCH(K_TOPK, launch_topk_fix(c.hs, c.Ws, P.d_s, P.V_r, P.Nc, row0, c.n_eff, c.idx, k, topk_idx, topk_val,
                                      pp.alpha, pp.fstats, pp.gscale, pp.g_hi, pp.g_lo, pp.corr_v, pp.corr_r,
                                      P.n_split * epi_parts(2, P.kind) * kCorrSlots, ws_at<int>(c.ws, P.off_tkr_v),
                                      ws_at<float>(c.ws, P.off_tkr_r), loss, c.nonfinite, c.s));
    if ((st = finish_chunk(c, row0, loss, local_rows(dh_s, P.d_s), dW, nullptr, 0, k)) != KD_OK) return st;
  }
  return KD_OK;
}

// A wait of the peer exchange to enqueue after an entry point's argument checks, before its first kernel.
struct P2PWaitArg {
  const unsigned* ctr = nullptr;  // counters [n], one per source rank
  int n = 0;
  unsigned target = 0;
};

// Stats of one shard into `rec` (plane stride rec_plane >= N): kd_vocab_stats (local) and kd_vocab_stats_p2p
// (straight into this rank's slot of the arena's record set).
static kd_status vocab_stats_impl(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                  const void* W_s, const uint8_t* mask, float* rec, long long rec_plane,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  kd_status st = validate_unstaged(p, false);
  if (st != KD_OK) return st;
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  if (c.P.N > 0 && !rec) return fail(KD_ERR_INVALID_ARG, "rec is NULL");
  if (rec && !aligned16(rec)) return fail(KD_ERR_ALIGNMENT, "rec must be 16-byte aligned");
  if ((st = check_common(p, h_t, W_t, h_s, W_s, rec, rec, nullptr, workspace, workspace_bytes, c.P)) != KD_OK)
    return st;
  const Plan& P = c.P;
  if (P.N == 0) return KD_OK;
  if ((st = prologue(c, h_t, W_t, h_s, W_s, mask, nullptr)) != KD_OK) return st;
  if (mask) KD_LAUNCH(K_ZERO, launch_zero_records(mask, P.N, rec, rec_plane, c.s));
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    PassParams pp = pass_params(c, row0);
    // RKL shards need the cross term U in the record: the RKL value enters the gradient, so it must be merged
    // before pass 2.  FKL (loss partials from pass 2, summed over the shards) needs the two LSEs only: the
    // decoupled pass 1, as the fused path
    const bool coupled = P.kind == KD_RKL;
    if ((st = run_pass(c, 1, P.kind, coupled && rkl_p1_coupled(), pp)) != KD_OK) return st;
    KD_LAUNCH(K_MERGE, launch_merge(pp.part, pp.part_plane, P.Nc, P.n_split * epi_parts(1, P.kind), P.Nc, row0, c.n_eff,
                           P.kind, 1, nullptr, nullptr, rec, rec_plane, c.idx, 0, c.nonfinite, 0, c.s));
  }
  return KD_OK;
}

kd_status kd_vocab_stats(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                         const uint8_t* mask, float* rec, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  if (!p) return fail(KD_ERR_INVALID_ARG, "problem is NULL");
  return vocab_stats_impl(p, h_t, W_t, h_s, W_s, mask, rec, (long long)p->n_tokens, workspace, workspace_bytes,
                          stream);
}

// The FKL/RKL shard backward behind kd_vocab_backward (dh / FKL loss rows into local buffers) and
// kd_vocab_backward_p2p (the same rows stored straight into the owning ranks' receive slots, RowDst).
static kd_status vocab_backward_impl(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                     const void* W_s, const uint8_t* mask, const float* recs, long long rec_plane,
                                     long long rec_rank_stride, int32_t n_ranks,
                                     float* loss, float* dh_local, const RowDst& dh_dst, const RowDst& floss_dst,
                                     float* dW_s, int64_t* n_nonfinite, void* workspace, size_t workspace_bytes,
                                     void* stream, bool p2p, const P2PWaitArg& pre = P2PWaitArg{}) {
  kd_status st = validate_unstaged(p, false);
  if (st != KD_OK) return st;
  if (p->kind != KD_FKL && p->kind != KD_RKL)
    return fail(KD_ERR_UNSUPPORTED, "JSD/TVD vocab shards need the K exchange: use kd_vocab_partials + kd_vocab_finish");
  if (n_ranks < 1) return fail(KD_ERR_INVALID_ARG, "n_ranks must be >= 1");
  Ctx c{};
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  float* dW = p->want_dW ? dW_s : nullptr;
  if ((st = check_common(p, h_t, W_t, h_s, W_s, loss, dh_local, dW, workspace, workspace_bytes, c.P,
                         !p2p)) != KD_OK)
    return st;
  if (c.P.N > 0 && !recs) return fail(KD_ERR_INVALID_ARG, "recs is NULL");
  const Plan& P = c.P;
  if (dW && !p->accumulate_dW) KD_CUDA(cudaMemsetAsync(dW, 0, (size_t)P.V_r * P.d_s * 4, c.s));
  if (P.N == 0) {
    if (n_nonfinite) KD_CUDA(cudaMemsetAsync(n_nonfinite, 0, 8, c.s));
    return KD_OK;
  }
  // the peer exchange's wait for the records (after every argument check, before the first kernel)
  if (pre.ctr) KD_LAUNCH(K_P2P, launch_p2p_wait(pre.ctr, pre.n, pre.target, c.s));
  if ((st = prologue(c, h_t, W_t, h_s, W_s, mask, n_nonfinite)) != KD_OK) return st;
  // masked rows: local outputs zeroed here; in the peer exchange the owner writes their zeros (k_p2p_combine)
  if (mask && (loss || dh_local)) KD_LAUNCH(K_ZERO, launch_zero_masked(mask, P.N, loss, dh_local, P.d_s, c.s));
  for (int ch = 0; ch < P.n_chunks; ++ch) {
    const int row0 = ch * P.Nc;
    // rank records [n_ranks][5][N] indexed by ORIGINAL row, merged in rank order
    KD_LAUNCH(K_MERGE, launch_merge(recs, rec_plane, rec_rank_stride, n_ranks, P.Nc, row0, c.n_eff, P.kind, 0,
                           ws_at<float>(c.ws, P.off_fstats), loss, nullptr, 0, c.idx, 1, c.nonfinite,
                           P.kind == KD_RKL ? 1 : 0, c.s));
    if ((st = backward_chunk(c, row0, loss, dh_dst, dW)) != KD_OK) return st;
    if (P.kind == KD_FKL)  // this shard's partial FKL: Σ over its vocab rows of p (ln p − ln q), global LSEs
      KD_LAUNCH(K_MERGE, launch_loss_rows(pass_params(c, row0).kpart, P.n_gslots, P.Nc, row0, c.n_eff, floss_dst,
                                          c.idx, c.nonfinite, c.s));
  }
  return KD_OK;
}

kd_status kd_vocab_backward(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                            const uint8_t* mask, const float* recs, int32_t n_ranks, float* loss,
                            float* dh_s_partial, float* dW_s, int64_t* n_nonfinite, void* workspace,
                            size_t workspace_bytes, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  if (!p) return fail(KD_ERR_INVALID_ARG, "problem is NULL");
  return vocab_backward_impl(p, h_t, W_t, h_s, W_s, mask, recs, (long long)p->n_tokens, 5ll * p->n_tokens, n_ranks,
                             loss, dh_s_partial,
                             local_rows(dh_s_partial, p->d_s), local_rows(loss, 1), dW_s, n_nonfinite,
                             workspace, workspace_bytes, stream, false);
}

// ------------------------------------------------------------------------------------ peer exchange (§8, kd_p2p)
namespace {
// counter block [0, 256) of an arena: one u32 per SOURCE rank and kind, each written by that rank only — a wait
// needs every source to have reached the chunk (a shared sum could be satisfied by a rank running ahead)
constexpr long long kCtrArrivals = 0, kCtrDone = 32, kCtrRecords = 64, kCtrKJ = 96;
struct P2PLayout {
  long long R, rplane, set_bytes, lset_bytes, rset_bytes, kjset_bytes, off_slots, off_lslots, off_recs, off_kj, off_dh,
      off_loss, total;
};
long long align256(long long x) { return (x + 255) / 256 * 256; }
P2PLayout p2p_layout(int world, long long max_rows, long long max_tokens, int d_s) {
  P2PLayout L{};
  L.R = world > 0 ? (max_rows + world - 1) / world : 0;
  L.set_bytes = align256((long long)world * L.R * d_s * 4);
  L.lset_bytes = align256((long long)world * L.R * 4);
  L.off_slots = 256;
  L.off_lslots = L.off_slots + kP2PSets * L.set_bytes;
  L.rplane = (max_rows + 3) / 4 * 4;                               // record plane stride (16-B aligned planes)
  L.rset_bytes = align256((long long)world * 5 * L.rplane * 4);   // records [world][5][rplane]
  L.kjset_bytes = align256((long long)world * 2 * L.rplane * 4);  // JSD/TVD (K, J) partials [world][2][rplane]
  L.off_recs = L.off_lslots + kP2PSets * L.lset_bytes;
  L.off_kj = L.off_recs + kP2PSets * L.rset_bytes;
  L.off_dh = L.off_kj + kP2PSets * L.kjset_bytes;
  L.off_loss = L.off_dh + align256(max_tokens * d_s * 4);
  L.total = L.off_loss + align256(max_tokens * 4);
  return L;
}
kd_status check_p2p(const kd_p2p* x) {
  if (!x) return fail(KD_ERR_INVALID_ARG, "kd_p2p is NULL");
  if (x->world < 1 || x->world > kP2PMaxRanks) return fail(KD_ERR_INVALID_ARG, "kd_p2p.world must be in [1, 8]");
  if (x->rank < 0 || x->rank >= x->world) return fail(KD_ERR_INVALID_ARG, "kd_p2p.rank outside [0, world)");
  if (x->d_s <= 0 || x->d_s % 4 || x->max_rows < 0 || x->max_tokens < 0)
    return fail(KD_ERR_SHAPE, "kd_p2p: d_s must be a positive multiple of 4, capacities >= 0");
  for (int j = 0; j < x->world; ++j)
    if (!x->arena[j] || (reinterpret_cast<uintptr_t>(x->arena[j]) & 255))
      return fail(KD_ERR_ALIGNMENT, "kd_p2p.arena[%d] must be non-NULL and 256-byte aligned", j);
  return KD_OK;
}
uint8_t* arena_at(const kd_p2p* x, int j, long long off) { return static_cast<uint8_t*>(x->arena[j]) + off; }
}  // namespace

size_t kd_p2p_arena_bytes(int32_t world, int64_t max_rows, int64_t max_tokens, int32_t d_s) {
  if (world < 1 || world > kP2PMaxRanks || max_rows < 0 || max_tokens < 0 || d_s <= 0) return 0;
  return (size_t)p2p_layout(world, max_rows, max_tokens, d_s).total;
}

kd_status kd_p2p_outputs(const kd_p2p* x, float** dh_out, float** loss_out) {
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  if (!dh_out || !loss_out) return fail(KD_ERR_INVALID_ARG, "NULL output pointer");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  *dh_out = reinterpret_cast<float*>(arena_at(x, x->rank, L.off_dh));
  *loss_out = reinterpret_cast<float*>(arena_at(x, x->rank, L.off_loss));
  return KD_OK;
}

// The all-gather of a per-rank block ([planes][rplane] f32 at byte offset `slot` of every arena): copy this rank's
// block into every peer's, then raise counter `ctr` [rank] in every arena.
static kd_status p2p_allgather(const kd_p2p* x, long long slot, int planes, long long rows, long long plane,
                               long long ctr, cudaStream_t s) {
  P2PCopy cp{};
  cp.src = reinterpret_cast<const float*>(arena_at(x, x->rank, slot));
  cp.n_dst = 0;
  for (int t = 0; t < x->world; ++t)
    if (t != x->rank) cp.dst[cp.n_dst++] = reinterpret_cast<float*>(arena_at(x, t, slot));
  cp.planes = planes;
  cp.rows = rows;
  cp.plane = plane;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cp.n_dst > 0 && rows > 0) KD_LAUNCH(K_P2P, launch_p2p_copy(cp, sms, s));
  P2PFlags f{};
  f.n = x->world;
  for (int t = 0; t < x->world; ++t) f.f[t] = reinterpret_cast<unsigned*>(arena_at(x, t, ctr + 4 * x->rank));
  KD_LAUNCH(K_P2P, launch_p2p_signal(f, s));
  return KD_OK;
}

static RowDst p2p_dh_dst(const kd_p2p* x, const P2PLayout& L, int set, long long n_tokens, bool loss) {
  RowDst d{};
  const long long R = (n_tokens + x->world - 1) / x->world;  // rows per owner in this exchange chunk
  for (int j = 0; j < x->world; ++j)
    d.base[j] = reinterpret_cast<float*>(
        arena_at(x, j, loss ? L.off_lslots + set * L.lset_bytes : L.off_slots + set * L.set_bytes));
  d.rows_per_owner = R > 0 ? R : 1;
  d.src_row = (long long)x->rank * R;
  d.ld = loss ? 1 : x->d_s;
  d.sys_fence = 1;
  return d;
}

kd_status kd_vocab_stats_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                             const uint8_t* mask, void* workspace, size_t workspace_bytes, const kd_p2p* x,
                             int32_t set, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  if (!p) return fail(KD_ERR_INVALID_ARG, "problem is NULL");
  if (set < 0 || set >= kP2PSets) return fail(KD_ERR_INVALID_ARG, "set must be in [0, %d)", kP2PSets);
  if (p->n_tokens > x->max_rows) return fail(KD_ERR_SHAPE, "n_tokens exceeds the arena's max_rows");
  if (p->d_s != x->d_s) return fail(KD_ERR_SHAPE, "problem d_s != kd_p2p.d_s");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  const long long slot = L.off_recs + set * L.rset_bytes + (long long)x->rank * 5 * L.rplane * 4;
  float* own = reinterpret_cast<float*>(arena_at(x, x->rank, slot));
  if ((st = vocab_stats_impl(p, h_t, W_t, h_s, W_s, mask, own, L.rplane, workspace, workspace_bytes, stream)) !=
      KD_OK)
    return st;
  // all-gather: this rank's record into every peer's slot [rank] of the set, then their record counters + 1
  return p2p_allgather(x, slot, 5, p->n_tokens, L.rplane, kCtrRecords, static_cast<cudaStream_t>(stream));
}

kd_status kd_vocab_backward_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                const void* W_s, const uint8_t* mask, const float* recs, int32_t n_ranks,
                                float* loss, float* dW_s, int64_t* n_nonfinite, void* workspace,
                                size_t workspace_bytes, const kd_p2p* x, int32_t set, uint32_t records_target,
                                void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  if (!p) return fail(KD_ERR_INVALID_ARG, "problem is NULL");
  if (set < 0 || set >= kP2PSets) return fail(KD_ERR_INVALID_ARG, "set must be in [0, %d)", kP2PSets);
  if (n_ranks != x->world) return fail(KD_ERR_INVALID_ARG, "n_ranks (%d) != kd_p2p.world (%d)", n_ranks, x->world);
  if (p->d_s != x->d_s) return fail(KD_ERR_SHAPE, "problem d_s != kd_p2p.d_s");
  if (p->n_tokens > x->max_rows) return fail(KD_ERR_SHAPE, "n_tokens exceeds the arena's max_rows");
  if (p->kind == KD_RKL && p->n_tokens > 0 && !loss) return fail(KD_ERR_INVALID_ARG, "RKL needs the local loss buffer");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  const RowDst dh = p2p_dh_dst(x, L, set, p->n_tokens, false), fl = p2p_dh_dst(x, L, set, p->n_tokens, true);
  long long rec_plane = p->n_tokens, rec_rank = 5ll * p->n_tokens;
  P2PWaitArg pre{};
  if (!recs) {  // the records all-gathered into this rank's arena by kd_vocab_stats_p2p: wait for all of them
    recs = reinterpret_cast<const float*>(arena_at(x, x->rank, L.off_recs + set * L.rset_bytes));
    rec_plane = L.rplane;
    rec_rank = 5ll * L.rplane;
    pre.ctr = reinterpret_cast<const unsigned*>(arena_at(x, x->rank, kCtrRecords));
    pre.n = x->world;
    pre.target = records_target;
  }
  if ((st = vocab_backward_impl(p, h_t, W_t, h_s, W_s, mask, recs, rec_plane, rec_rank, n_ranks,
                                p->kind == KD_RKL ? loss : nullptr, nullptr, dh, fl, dW_s, n_nonfinite, workspace,
                                workspace_bytes, stream, true, pre)) != KD_OK)
    return st;
  // publish: every owner's arrival counter + 1 (one per rank per exchange chunk, also for an empty chunk)
  P2PFlags f{};
  f.n = x->world;
  for (int j = 0; j < x->world; ++j) f.f[j] = reinterpret_cast<unsigned*>(arena_at(x, j, kCtrArrivals + 4 * x->rank));
  KD_LAUNCH(K_P2P, launch_p2p_signal(f, static_cast<cudaStream_t>(stream)));
  return KD_OK;
}

kd_status kd_p2p_combine(const kd_p2p* x, int32_t set, int64_t n_rows, int64_t row0, const uint8_t* mask,
                         int32_t with_loss, uint32_t arrivals_target, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  if (set < 0 || set >= kP2PSets) return fail(KD_ERR_INVALID_ARG, "set must be in [0, %d)", kP2PSets);
  if (n_rows < 0 || n_rows > x->max_rows) return fail(KD_ERR_SHAPE, "n_rows outside [0, max_rows]");
  if (row0 < 0 || row0 + n_rows > x->max_tokens) return fail(KD_ERR_SHAPE, "rows [row0, row0 + n_rows) exceed max_tokens");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  P2PCombine c{};
  c.slots = reinterpret_cast<const float*>(arena_at(x, x->rank, L.off_slots + set * L.set_bytes));
  c.lslots = with_loss ? reinterpret_cast<const float*>(arena_at(x, x->rank, L.off_lslots + set * L.lset_bytes))
                       : nullptr;
  for (int t = 0; t < x->world; ++t) {
    c.out[t] = reinterpret_cast<float*>(arena_at(x, t, L.off_dh)) + row0 * x->d_s;
    c.lout[t] = with_loss ? reinterpret_cast<float*>(arena_at(x, t, L.off_loss)) + row0 : nullptr;
  }
  c.mask = mask;
  c.arrivals = reinterpret_cast<const unsigned*>(arena_at(x, x->rank, kCtrArrivals));
  c.target = arrivals_target;
  c.P = x->world;
  c.me = x->rank;
  c.d_s = x->d_s;
  c.R = (n_rows + x->world - 1) / x->world;
  c.n_rows = n_rows;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  KD_LAUNCH(K_P2P, launch_p2p_combine(c, sms, s));
  P2PFlags f{};
  f.n = x->world;
  for (int t = 0; t < x->world; ++t) f.f[t] = reinterpret_cast<unsigned*>(arena_at(x, t, kCtrDone + 4 * x->rank));
  KD_LAUNCH(K_P2P, launch_p2p_signal(f, s));
  return KD_OK;
}

kd_status kd_p2p_wait(const kd_p2p* x, uint32_t done_target, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  KD_LAUNCH(K_P2P, launch_p2p_wait(reinterpret_cast<const unsigned*>(arena_at(x, x->rank, kCtrDone)), x->world, done_target,
                                   static_cast<cudaStream_t>(stream)));
  return KD_OK;
}

// JSD/TVD vocab shards (C2 exchange): one token chunk per call pair, the workspace carrying the chunk's G planes
// from kd_vocab_partials to kd_vocab_finish.
static kd_status vocab_fix_setup(Ctx& c, const kd_problem* p, void* workspace, size_t workspace_bytes, void* stream,
                                 int32_t n_ranks) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  kd_status st = validate_unstaged(p, false);
  if (st != KD_OK) return st;
  if (p->kind != KD_JSD && p->kind != KD_TVD)
    return fail(KD_ERR_UNSUPPORTED, "kd_vocab_partials/finish are the JSD/TVD shard path; FKL/RKL use kd_vocab_backward");
  if (n_ranks < 1) return fail(KD_ERR_INVALID_ARG, "n_ranks must be >= 1");
  c.p = p;
  c.P = make_plan(p);
  c.s = static_cast<cudaStream_t>(stream);
  c.ws = workspace;
  attach_die(c);
  if (c.P.n_chunks > 1)
    return fail(KD_ERR_SHAPE, "JSD/TVD vocab shards run one token chunk per call: n_tokens (%d) must be <= the chunk (%d)",
                c.P.N, c.P.Nc);
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace must be non-NULL and 256-byte aligned");
  if (workspace_bytes < c.P.total)
    return fail(KD_ERR_WORKSPACE_TOO_SMALL, "workspace %zu bytes < required %zu", workspace_bytes, c.P.total);
  return KD_OK;
}

static kd_status vocab_partials_impl(Ctx& c, const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                     const void* W_s, const uint8_t* mask, const float* recs, long long rec_plane,
                                     long long rec_rank, int32_t n_ranks, float* kj, long long kj_plane,
                                     void* workspace, size_t workspace_bytes, const P2PWaitArg& pre = P2PWaitArg{}) {
  const Plan& P = c.P;
  if (P.N == 0) return KD_OK;
  if (!recs || !kj) return fail(KD_ERR_INVALID_ARG, "recs / kj is NULL");
  if (!aligned16(kj) || !aligned16(recs)) return fail(KD_ERR_ALIGNMENT, "recs / kj must be 16-byte aligned");
  // the same input checks as every other entry point (pointers, alignment, workspace), before any launch; dW_s is
  // kd_vocab_finish's output, not this call's
  kd_problem q = *p;
  q.want_dW = 0;
  kd_status st;
  if ((st = check_common(&q, h_t, W_t, h_s, W_s, kj, kj, nullptr, workspace, workspace_bytes, P)) != KD_OK) return st;
  if (pre.ctr) KD_LAUNCH(K_P2P, launch_p2p_wait(pre.ctr, pre.n, pre.target, c.s));
  if ((st = prologue(c, h_t, W_t, h_s, W_s, mask, nullptr)) != KD_OK) return st;
  KD_CUDA(cudaMemsetAsync(kj, 0, (size_t)2 * kj_plane * sizeof(float), c.s));
  KD_LAUNCH(K_MERGE, launch_merge(recs, rec_plane, rec_rank, n_ranks, P.Nc, 0, c.n_eff, P.kind, 0,
                                  ws_at<float>(c.ws, P.off_fstats), nullptr, nullptr, 0, c.idx, 1, c.nonfinite, 0, c.s));
  if ((st = grad_chunk(c, 0)) != KD_OK) return st;
  PassParams pp = pass_params(c, 0);
  KD_LAUNCH(K_KFIX, launch_kj_rows(pp.kpart, P.n_split * epi_parts(2, P.kind), P.Nc, 0, c.n_eff, c.idx, kj, kj_plane,
                                   c.s));
  return KD_OK;
}

kd_status kd_vocab_partials(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                            const uint8_t* mask, const float* recs, int32_t n_ranks, float* kj, void* workspace,
                            size_t workspace_bytes, void* stream) {
  Ctx c{};
  kd_status st = vocab_fix_setup(c, p, workspace, workspace_bytes, stream, n_ranks);
  if (st != KD_OK) return st;
  return vocab_partials_impl(c, p, h_t, W_t, h_s, W_s, mask, recs, c.P.N, 5ll * c.P.N, n_ranks, kj, c.P.N, workspace,
                             workspace_bytes);
}

static kd_status vocab_finish_impl(Ctx& c, const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                   const void* W_s, const uint8_t* mask, const float* kj_all, long long kj_plane,
                                   int32_t n_ranks, float* loss, float* dh_local, const RowDst& dh, float* dW_s,
                                   int64_t* n_nonfinite, void* workspace, size_t workspace_bytes,
                                   const P2PWaitArg& pre = P2PWaitArg{}) {
  const Plan& P = c.P;
  float* dW = p->want_dW ? dW_s : nullptr;
  kd_status st;
  if ((st = check_common(p, h_t, W_t, h_s, W_s, loss, dh_local, dW, workspace, workspace_bytes, P,
                         dh_local != nullptr)) != KD_OK)
    return st;
  if (P.N > 0 && !loss) return fail(KD_ERR_INVALID_ARG, "NULL loss pointer");
  if (dW && !p->accumulate_dW) KD_CUDA(cudaMemsetAsync(dW, 0, (size_t)P.V_r * P.d_s * 4, c.s));
  if (P.N == 0) {
    if (n_nonfinite) KD_CUDA(cudaMemsetAsync(n_nonfinite, 0, 8, c.s));
    return KD_OK;
  }
  if (!kj_all) return fail(KD_ERR_INVALID_ARG, "kj_all is NULL");
  if (pre.ctr) KD_LAUNCH(K_P2P, launch_p2p_wait(pre.ctr, pre.n, pre.target, c.s));
  // the prologue is deterministic in the inputs: it rebuilds the same row compaction / packed rows that
  // kd_vocab_partials used, leaving the chunk's G planes in the workspace untouched
  if ((st = prologue(c, h_t, W_t, h_s, W_s, mask, n_nonfinite)) != KD_OK) return st;
  if (mask) KD_LAUNCH(K_ZERO, launch_zero_masked(mask, P.N, loss, dh_local, P.d_s, c.s));
  return finish_chunk(c, 0, loss, dh, dW, kj_all, n_ranks, 0, kj_plane);
}

kd_status kd_vocab_finish(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                          const uint8_t* mask, const float* kj_all, int32_t n_ranks, float* loss,
                          float* dh_s_partial, float* dW_s, int64_t* n_nonfinite, void* workspace,
                          size_t workspace_bytes, void* stream) {
  Ctx c{};
  kd_status st = vocab_fix_setup(c, p, workspace, workspace_bytes, stream, n_ranks);
  if (st != KD_OK) return st;
  if (c.P.N > 0 && !dh_s_partial) return fail(KD_ERR_INVALID_ARG, "NULL input/output pointer");
  return vocab_finish_impl(c, p, h_t, W_t, h_s, W_s, mask, kj_all, c.P.N, n_ranks, loss, dh_s_partial,
                           local_rows(dh_s_partial, c.P.d_s), dW_s, n_nonfinite, workspace, workspace_bytes);
}

// JSD/TVD shards with the peer exchange: records and (K, J) partials through the arena, dh to the owners.
kd_status kd_vocab_partials_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s,
                                const void* W_s, const uint8_t* mask, void* workspace, size_t workspace_bytes,
                                const kd_p2p* x, int32_t set, uint32_t records_target, void* stream) {
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  Ctx c{};
  if ((st = vocab_fix_setup(c, p, workspace, workspace_bytes, stream, x->world)) != KD_OK) return st;
  if (set < 0 || set >= kP2PSets) return fail(KD_ERR_INVALID_ARG, "set must be in [0, %d)", kP2PSets);
  if (p->n_tokens > x->max_rows) return fail(KD_ERR_SHAPE, "n_tokens exceeds the arena's max_rows");
  if (p->d_s != x->d_s) return fail(KD_ERR_SHAPE, "problem d_s != kd_p2p.d_s");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  P2PWaitArg pre{};
  pre.ctr = reinterpret_cast<const unsigned*>(arena_at(x, x->rank, kCtrRecords));
  pre.n = x->world;
  pre.target = records_target;
  const float* recs = reinterpret_cast<const float*>(arena_at(x, x->rank, L.off_recs + set * L.rset_bytes));
  const long long kslot = L.off_kj + set * L.kjset_bytes + (long long)x->rank * 2 * L.rplane * 4;
  float* kj = reinterpret_cast<float*>(arena_at(x, x->rank, kslot));
  if ((st = vocab_partials_impl(c, p, h_t, W_t, h_s, W_s, mask, recs, L.rplane, 5ll * L.rplane, x->world, kj,
                                L.rplane, workspace, workspace_bytes, pre)) != KD_OK)
    return st;
  return p2p_allgather(x, kslot, 2, p->n_tokens, L.rplane, kCtrKJ, s);
}

kd_status kd_vocab_finish_p2p(const kd_problem* p, const void* h_t, const void* W_t, const void* h_s, const void* W_s,
                              const uint8_t* mask, float* loss, float* dW_s, int64_t* n_nonfinite, void* workspace,
                              size_t workspace_bytes, const kd_p2p* x, int32_t set, uint32_t kj_target,
                              void* stream) {
  kd_status st = check_p2p(x);
  if (st != KD_OK) return st;
  Ctx c{};
  if ((st = vocab_fix_setup(c, p, workspace, workspace_bytes, stream, x->world)) != KD_OK) return st;
  if (set < 0 || set >= kP2PSets) return fail(KD_ERR_INVALID_ARG, "set must be in [0, %d)", kP2PSets);
  if (p->n_tokens > x->max_rows) return fail(KD_ERR_SHAPE, "n_tokens exceeds the arena's max_rows");
  if (p->d_s != x->d_s) return fail(KD_ERR_SHAPE, "problem d_s != kd_p2p.d_s");
  const P2PLayout L = p2p_layout(x->world, x->max_rows, x->max_tokens, x->d_s);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  P2PWaitArg pre{};
  pre.ctr = reinterpret_cast<const unsigned*>(arena_at(x, x->rank, kCtrKJ));
  pre.n = x->world;
  pre.target = kj_target;
  const float* kj_all = reinterpret_cast<const float*>(arena_at(x, x->rank, L.off_kj + set * L.kjset_bytes));
  if ((st = vocab_finish_impl(c, p, h_t, W_t, h_s, W_s, mask, kj_all, L.rplane, x->world, loss, nullptr,
                              p2p_dh_dst(x, L, set, p->n_tokens, false), dW_s, n_nonfinite, workspace,
                              workspace_bytes, pre)) != KD_OK)
    return st;
  // publish: every owner's arrival counter [rank] + 1 (also for an empty chunk)
  P2PFlags f{};
  f.n = x->world;
  for (int j = 0; j < x->world; ++j) f.f[j] = reinterpret_cast<unsigned*>(arena_at(x, j, kCtrArrivals + 4 * x->rank));
  KD_LAUNCH(K_P2P, launch_p2p_signal(f, s));
  return KD_OK;
}

kd_status kd_gemm_bf16_f32(const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                           int32_t a_mn_major, int32_t b_mn_major, void* stream) {
  g_launches = 0;
  g_cur_stream = static_cast<cudaStream_t>(stream);
  if (!A || !B || !D) return fail(KD_ERR_INVALID_ARG, "NULL pointer");
  if (M < 1 || N < 1 || K < 1) return fail(KD_ERR_SHAPE, "M, N, K must be >= 1");
  if (N % 32) return fail(KD_ERR_SHAPE, "N must be a multiple of 32");
  if ((!a_mn_major && K % 8) || (a_mn_major && M % 8) || (!b_mn_major && K % 8) || (b_mn_major && N % 8))
    return fail(KD_ERR_SHAPE, "contiguous extents must be multiples of 8 (16-byte rows)");
  if (!aligned16(A) || !aligned16(B) || !aligned16(D)) return fail(KD_ERR_ALIGNMENT, "pointers must be 16B aligned");
  CUtensorMap ma, mb;
  kd_status st;
  if (a_mn_major) st = make_map(&ma, A, M, K, (uint64_t)M * 2, 64, kBK);
  else st = make_map(&ma, A, K, M, (uint64_t)K * 2, kBK, kBM);
  if (st != KD_OK) return st;
  if (b_mn_major) st = make_map(&mb, B, N, K, (uint64_t)N * 2, 64, kBK);
  else st = make_map(&mb, B, K, N, (uint64_t)K * 2, kBK, kGemmBN / gemm_cg());  // each CTA of a pair: half the tile
  if (st != KD_OK) return st;
  GemmParams gp{};
  gp.M = M;
  gp.N = N;
  gp.K = K;
  gp.dyn_dim = DYN_NONE;
  gp.k_split = 1;
  gp.kb_per_acc = 1 << 30;  // plain GEMM: one accumulator per output tile
  gp.out = D;
  gp.out_ld = N;
  KD_LAUNCH(K_GEMM, launch_gemm(a_mn_major != 0, b_mn_major != 0, 1, EPI_STORE, gemm_cg(), &ma, nullptr, &mb, gp,
                                device_sms(), static_cast<cudaStream_t>(stream)));
  return KD_OK;
}

// ------------------------------------------------------------------------------------ hand-off (NEXT-4)
namespace {
struct HandoffWire {  // the KD_HANDOFF_HANDLE_BYTES bytes a handle occupies
  uint32_t magic;     // 'KDH1'
  uint32_t version;
  uint64_t offset;    // exported range: [base + offset, base + offset + bytes)
  uint64_t bytes;
  uint64_t pad;
  cudaIpcMemHandle_t ipc;  // 64 B: the allocation holding the range
};
static_assert(sizeof(HandoffWire) == KD_HANDOFF_HANDLE_BYTES, "wire size");
constexpr uint32_t kHandoffMagic = 0x3148444bu;
}  // namespace

kd_status kd_handoff_export(const void* dev_ptr, uint64_t bytes, void* handle) {
  if (!dev_ptr || !handle) return fail(KD_ERR_INVALID_ARG, "kd_handoff_export: NULL pointer");
  // driver entry point resolved at run time (the library keeps no link-time dependency on libcuda)
  static PFN_cuMemGetAddressRange_v3020 get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) ? reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn) : nullptr;
  }();
  if (!get_range) return fail(KD_ERR_CUDA, "kd_handoff_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(KD_ERR_CUDA, "kd_handoff_export: not a device allocation");
  const uint64_t off = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
  if (off + bytes > size) return fail(KD_ERR_INVALID_ARG, "kd_handoff_export: range exceeds its allocation");
  HandoffWire w{};
  w.magic = kHandoffMagic;
  w.version = KDFUSED_ABI_VERSION;
  w.offset = off;
  w.bytes = bytes;
  KD_CUDA(cudaIpcGetMemHandle(&w.ipc, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &w, sizeof w);
  return KD_OK;
}

kd_status kd_handoff_open(const void* handle, void** dev_ptr, uint64_t* bytes) {
  if (!handle || !dev_ptr || !bytes) return fail(KD_ERR_INVALID_ARG, "kd_handoff_open: NULL pointer");
  HandoffWire w;
  std::memcpy(&w, handle, sizeof w);
  if (w.magic != kHandoffMagic) return fail(KD_ERR_INVALID_ARG, "kd_handoff_open: not a kd_handoff_export handle");
  void* base = nullptr;
  KD_CUDA(cudaIpcOpenMemHandle(&base, w.ipc, cudaIpcMemLazyEnablePeerAccess));
  {
    std::lock_guard<std::mutex> lk(g_handoff_mu);
    g_handoff_bases[static_cast<char*>(base) + w.offset] = base;
  }
  *dev_ptr = static_cast<char*>(base) + w.offset;
  *bytes = w.bytes;
  return KD_OK;
}

kd_status kd_handoff_close(void* dev_ptr) {
  if (!dev_ptr) return fail(KD_ERR_INVALID_ARG, "kd_handoff_close: NULL pointer");
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_handoff_mu);
    auto it = g_handoff_bases.find(dev_ptr);
    if (it == g_handoff_bases.end()) return fail(KD_ERR_INVALID_ARG, "kd_handoff_close: not from kd_handoff_open");
    base = it->second;
    g_handoff_bases.erase(it);
  }
  KD_CUDA(cudaIpcCloseMemHandle(base));
  return KD_OK;
}

int32_t kd_last_launch_count(void) { return g_launches; }

// Undocumented debug hook (not in kdfused.h): device buffer the KD_EPI_TIMING build accumulates into.
void kd_debug_set_buffer(void* p) { g_dbg_ptr = p; }

int32_t kd_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int32_t prev = g_prof_on ? 1 : 0;
  g_prof_on = on != 0;
  return prev;
}

int32_t kd_profile_read(int32_t* launches, double* total_ms, int32_t max_kernels) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int n = max_kernels < K_NUM ? max_kernels : K_NUM;
  for (int i = 0; i < n; ++i) { launches[i] = 0; total_ms[i] = 0.0; }
  int32_t rc = K_NUM;
  for (const ProfRec& r : g_prof) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) rc = -1;
    if (r.id < n) { launches[r.id] += 1; total_ms[r.id] += ms; }
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof.clear();
  return rc;
}

const char* kd_profile_kernel_name(int32_t id) { return (id >= 0 && id < K_NUM) ? kKernelNames[id] : "?"; }
const char* kd_last_error(void) { return g_err.c_str(); }
int32_t kd_abi_version(void) { return KDFUSED_ABI_VERSION; }

}  // extern "C"
