// Probe (round-2 groundwork, DESIGN.md §10 item 2): which SMs share an L2 partition (die) on this B200.
// One CTA per SM (large dynamic smem forces 1/SM). For each of several small buffers (each fits L2 easily), every
// SM times a dependent chase on one line (the same address) after warming it: the latency is lower from the die whose L2
// partition homes (or caches) the lines.  Prints one line per SM: smid, mean cycles per load for each buffer.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int kBuffers = 16;
constexpr int kElems = 1;  // one line per buffer: its L2 home decides the latency
constexpr int kSteps = 2048;

__global__ void probe(const unsigned* const* bufs, unsigned* out) {
  extern __shared__ unsigned char big[];
  if (threadIdx.x != 0) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  out[blockIdx.x * (kBuffers + 1)] = smid;
  for (int b = 0; b < kBuffers; ++b) {
    const unsigned* p = bufs[b];
    unsigned i = 0;
    for (int s = 0; s < 256; ++s) i = __ldcg(p + i);  // warm (L2 only)
    long long t0 = clock64();
    for (int s = 0; s < kSteps; ++s) i = __ldcg(p + i);
    long long t1 = clock64();
    out[blockIdx.x * (kBuffers + 1) + 1 + b] = (unsigned)((t1 - t0) / kSteps) + (i == 0xFFFFFFFFu);
  }
  big[0] = 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<unsigned*> d(kBuffers);
  std::vector<unsigned> h(kElems);
  for (int b = 0; b < kBuffers; ++b) {
    // a random cyclic permutation (stride-free chase); buffers 64 MB apart so they hash to different slices
    for (int i = 0; i < kElems; ++i) h[i] = i;
    for (int i = kElems - 1; i > 0; --i) { int j = rand() % i; std::swap(h[i], h[j]); }
    std::vector<unsigned> nxt(kElems);
    for (int i = 0; i < kElems; ++i) nxt[h[i]] = h[(i + 1) % kElems];
    unsigned* p;
    cudaMalloc(&p, 64ull << 20);
    cudaMemcpy(p, nxt.data(), kElems * 4, cudaMemcpyHostToDevice);
    d[b] = p;
  }
  unsigned** dd;
  cudaMalloc(&dd, sizeof(unsigned*) * kBuffers);
  cudaMemcpy(dd, d.data(), sizeof(unsigned*) * kBuffers, cudaMemcpyHostToDevice);
  unsigned* out;
  cudaMalloc(&out, sms * (kBuffers + 1) * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<sms, 32, 200 * 1024>>>(dd, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<unsigned> r(sms * (kBuffers + 1));
  cudaMemcpy(r.data(), out, r.size() * 4, cudaMemcpyDeviceToHost);
  printf("smid");
  for (int b = 0; b < kBuffers; ++b) printf(" buf%d", b);
  printf("\n");
  for (int s = 0; s < sms; ++s) {
    printf("%u", r[s * (kBuffers + 1)]);
    for (int b = 0; b < kBuffers; ++b) printf(" %u", r[s * (kBuffers + 1) + 1 + b]);
    printf("\n");
  }
  return 0;
}
