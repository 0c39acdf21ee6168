// nvlink_probe.cu -- measures SM-issued NVLink traffic patterns between two
// GPUs, both directions at once (what a symmetric all-reduce round does) and
// one direction alone: 16-B peer loads, 16-B peer stores, and bulk async
// (TMA-engine) peer->smem copies.  Informs the exchange design of the
// one-shot all-reduce.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_read(const uint4* __restrict__ src, uint64_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

__global__ void k_write(uint4* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((unsigned)i, 1u, 2u, 3u);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}

constexpr int STAGES = 4;
constexpr unsigned TB = 16384;
__global__ void k_tma_read(const char* src, uint64_t ntiles, uint4* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  char* st = reinterpret_cast<char*>(sm + 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < STAGES; ++s) {
      uint64_t t = blockIdx.x + (uint64_t)s * gridDim.x;
      if (t < ntiles) { mbar_expect(&bars[s], TB); bulk(st + s * TB, src + t * TB, TB, &bars[s]); }
    }
  }
  __syncthreads();
  unsigned acc = 0;
  for (uint64_t j = 0;; ++j) {
    uint64_t t = blockIdx.x + j * gridDim.x;
    if (t >= ntiles) break;
    int s = j % STAGES;
    mbar_wait(&bars[s], (j / STAGES) & 1);
    acc ^= reinterpret_cast<const unsigned*>(st + s * TB)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t nt = blockIdx.x + (j + STAGES) * gridDim.x;
      if (nt < ntiles) { mbar_expect(&bars[s], TB); bulk(st + s * TB, src + nt * TB, TB, &bars[s]); }
    }
  }
  if (acc == 0x12345678u) sink[0] = make_uint4(acc, 0, 0, 0);
}

// bulk async shared->global stores into peer memory (the TMA engine writing
// over NVLink): each CTA stores a 16-KB smem tile to consecutive peer tiles.
__global__ void k_tma_write(char* dst, uint64_t ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  char* st = reinterpret_cast<char*>(sm + 128);
  for (unsigned i = threadIdx.x; i < TB / 4; i += blockDim.x) reinterpret_cast<unsigned*>(st)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    int inflight = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(dst + t * TB), "r"((unsigned)__cvta_generic_to_shared(st)), "r"(TB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight > 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// local HBM streaming (read 2 streams, write 1: the shape of an update kernel)
__global__ void k_local(const uint4* __restrict__ a, const uint4* __restrict__ b,
                        uint4* __restrict__ c, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 x = a[i], y = b[i];
    c[i] = make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w);
  }
}

// Concurrency: does SM-issued NVLink traffic slow a co-running HBM kernel?
int interference(void* const* buf, uint4* const* sink) {
  const uint64_t lb = 400ull << 20;  // 400 MB per local array
  void *a, *b, *c;
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&a, lb)); CK(cudaMalloc(&b, lb)); CK(cudaMalloc(&c, lb));
  cudaStream_t s0, s1; CK(cudaStreamCreate(&s0)); CK(cudaStreamCreate(&s1));
  cudaEvent_t ev[4]; for (auto& x : ev) CK(cudaEventCreate(&x));
  const uint64_t nl = lb / 16, np = (100ull << 20) / 16;
  void* cebuf;
  CK(cudaMalloc(&cebuf, 100ull << 20));
  for (int mode = 0; mode < 8; ++mode) {  // 0 local, 1 peer ld, 2 both, 3 peer st, 4 local+st, 5 local+bulk rd, 6 CE peer copy, 7 local + CE
    float bl = 1e9f, bp = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaDeviceSynchronize());
      if (mode != 1 && mode != 3 && mode != 6) {
        CK(cudaEventRecord(ev[0], s0));
        k_local<<<148 * 4, 512, 0, s0>>>((const uint4*)a, (const uint4*)b, (uint4*)c, nl);
        CK(cudaEventRecord(ev[1], s0));
      }
      if (mode >= 1) {
        CK(cudaEventRecord(ev[2], s1));
        if (mode == 1 || mode == 2) k_read<<<148 * 2, 512, 0, s1>>>((const uint4*)buf[1], np, sink[0]);
        if (mode == 3 || mode == 4) k_write<<<148 * 2, 512, 0, s1>>>((uint4*)buf[1], np);
        if (mode >= 6) CK(cudaMemcpyAsync(cebuf, buf[1], 100ull << 20, cudaMemcpyDefault, s1));
        if (mode == 5) k_tma_read<<<148, 512, 128 + STAGES * TB, s1>>>((const char*)buf[1], (100ull << 20) / TB, sink[0]);
        CK(cudaEventRecord(ev[3], s1));
      }
      CK(cudaDeviceSynchronize());
      float ms;
      if (mode != 1 && mode != 3 && mode != 6) { CK(cudaEventElapsedTime(&ms, ev[0], ev[1])); if (ms < bl) bl = ms; }
      if (mode >= 1) { CK(cudaEventElapsedTime(&ms, ev[2], ev[3])); if (ms < bp) bp = ms; }
    }
    const char* nm[] = {"local alone", "peer ld alone", "local + peer ld", "peer st alone",
                        "local + peer st", "local + bulk peer rd", "CE peer copy alone",
                        "local + CE peer copy"};
    printf("%-22s", nm[mode]);
    if (mode != 1 && mode != 3 && mode != 6) printf("  local %.1f us (%.0f GB/s)", bl * 1e3, 3.0 * lb / (bl * 1e6));
    if (mode >= 1) printf("  peer %.1f us (%.0f GB/s)", bp * 1e3, (100ull << 20) / (bp * 1e6));
    printf("\n");
  }
  return 0;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  const uint64_t bytes = 100ull << 20;
  void* buf[2]; uint4* sink[2]; cudaStream_t s[2]; cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMemset(buf[g], 1, bytes));
    CK(cudaMalloc(&sink[g], 64));
    CK(cudaStreamCreate(&s[g]));
    CK(cudaEventCreate(&e0[g])); CK(cudaEventCreate(&e1[g]));
    CK(cudaFuncSetAttribute(k_tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + STAGES * TB));
    CK(cudaFuncSetAttribute(k_tma_write, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + TB));
  }
  const char* names[] = {"ld16 peer read", "st16 peer write", "bulk peer read (16KB x4)",
                         "bulk peer write (16KB)"};
  for (int kind = 0; kind < 4; ++kind)
    for (int both = 0; both < 2; ++both)
      for (int bps : {1, 2, 4}) {
        float best[2] = {1e9f, 1e9f};
        for (int rep = 0; rep < 5; ++rep) {
          for (int g = 0; g <= both; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventRecord(e0[g], s[g]));
            const uint64_t n16 = bytes / 16;
            const int grid = 148 * bps;
            if (kind == 0) k_read<<<grid, 512, 0, s[g]>>>((const uint4*)buf[1 - g], n16, sink[g]);
            if (kind == 1) k_write<<<grid, 512, 0, s[g]>>>((uint4*)buf[1 - g], n16);
            if (kind == 3) k_tma_write<<<grid, 128, 128 + TB, s[g]>>>((char*)buf[1 - g], bytes / TB);
            if (kind == 2) k_tma_read<<<grid, 512, 128 + STAGES * TB, s[g]>>>((const char*)buf[1 - g], bytes / TB, sink[g]);
            CK(cudaEventRecord(e1[g], s[g]));
          }
          for (int g = 0; g <= both; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventSynchronize(e1[g]));
            float ms; CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
            if (ms < best[g]) best[g] = ms;
          }
        }
        printf("%-26s %-14s ctas/sm=%d  gpu0 %.1f GB/s%s", names[kind], both ? "bidirectional" : "one-way", bps,
               bytes / (best[0] * 1e6), both ? "" : "\n");
        if (both) printf("  gpu1 %.1f GB/s\n", bytes / (best[1] * 1e6));
      }
  if (interference(buf, sink)) return 1;
  // spatial split: local stream on L SMs, peer loads on the other 148 - L
  // (one CTA per SM each, forced by a large dynamic smem reservation)
  {
    CK(cudaSetDevice(0));
    const uint64_t lb = 400ull << 20;
    void *a, *b, *c;
    CK(cudaMalloc(&a, lb)); CK(cudaMalloc(&b, lb)); CK(cudaMalloc(&c, lb));
    cudaStream_t s0, s1; CK(cudaStreamCreate(&s0)); CK(cudaStreamCreate(&s1));
    cudaEvent_t ev[4]; for (auto& x : ev) CK(cudaEventCreate(&x));
    const int big = 160 * 1024;
    CK(cudaFuncSetAttribute(k_local, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_read, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    for (int L : {148, 120, 100, 74}) {
      float bl = 1e9f, bp = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(ev[0], s0));
        k_local<<<L, 1024, big, s0>>>((const uint4*)a, (const uint4*)b, (uint4*)c, lb / 16);
        CK(cudaEventRecord(ev[1], s0));
        if (L < 148) {
          CK(cudaEventRecord(ev[2], s1));
          k_read<<<148 - L, 1024, big, s1>>>((const uint4*)buf[1], (100ull << 20) / 16, sink[0]);
          CK(cudaEventRecord(ev[3], s1));
        }
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, ev[0], ev[1])); if (ms < bl) bl = ms;
        if (L < 148) { CK(cudaEventElapsedTime(&ms, ev[2], ev[3])); if (ms < bp) bp = ms; }
      }
      printf("split: local on %3d SMs %.1f us (%.0f GB/s)", L, bl * 1e3, 3.0 * lb / (bl * 1e6));
      if (L < 148) printf("  peer ld on %3d SMs %.1f us (%.0f GB/s)", 148 - L, bp * 1e3, (100ull << 20) / (bp * 1e6));
      printf("\n");
    }
    // peer loads alone on the small SM sets
    for (int P : {28, 48, 74}) {
      float bp = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(ev[2], s1));
        k_read<<<P, 1024, big, s1>>>((const uint4*)buf[1], (100ull << 20) / 16, sink[0]);
        CK(cudaEventRecord(ev[3], s1));
        CK(cudaDeviceSynchronize());
        float ms; CK(cudaEventElapsedTime(&ms, ev[2], ev[3])); if (ms < bp) bp = ms;
      }
      printf("peer ld alone on %3d SMs: %.0f GB/s\n", P, (100ull << 20) / (bp * 1e6));
    }
  }
  // both GPUs at once: each streams its own HBM and pulls 100 MB from the
  // other with a copy engine (the shape of a CE-exchange all-reduce round)
  {
    const uint64_t lb = 400ull << 20;
    void *a[2], *b[2], *c[2], *ce[2];
    cudaStream_t sl[2], sc[2];
    cudaEvent_t ev[2][4];
    for (int g = 0; g < 2; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&a[g], lb)); CK(cudaMalloc(&b[g], lb)); CK(cudaMalloc(&c[g], lb));
      CK(cudaMalloc(&ce[g], 100ull << 20));
      CK(cudaStreamCreate(&sl[g])); CK(cudaStreamCreate(&sc[g]));
      for (auto& x : ev[g]) CK(cudaEventCreate(&x));
    }
    for (int with_local = 0; with_local < 2; ++with_local) {
      float bl[2] = {1e9f, 1e9f}, bp[2] = {1e9f, 1e9f};
      for (int rep = 0; rep < 5; ++rep) {
        for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          if (with_local) {
            CK(cudaEventRecord(ev[g][0], sl[g]));
            k_local<<<148 * 4, 512, 0, sl[g]>>>((const uint4*)a[g], (const uint4*)b[g], (uint4*)c[g], lb / 16);
            CK(cudaEventRecord(ev[g][1], sl[g]));
          }
          CK(cudaEventRecord(ev[g][2], sc[g]));
          CK(cudaMemcpyAsync(ce[g], buf[1 - g], 100ull << 20, cudaMemcpyDefault, sc[g]));
          CK(cudaEventRecord(ev[g][3], sc[g]));
        }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize());
          float ms;
          if (with_local) { CK(cudaEventElapsedTime(&ms, ev[g][0], ev[g][1])); if (ms < bl[g]) bl[g] = ms; }
          CK(cudaEventElapsedTime(&ms, ev[g][2], ev[g][3])); if (ms < bp[g]) bp[g] = ms;
        }
      }
      for (int g = 0; g < 2; ++g) {
        printf("bidirectional CE%s gpu%d:", with_local ? " + local" : "", g);
        if (with_local) printf("  local %.1f us (%.0f GB/s)", bl[g] * 1e3, 3.0 * lb / (bl[g] * 1e6));
        printf("  CE %.1f us (%.0f GB/s)\n", bp[g] * 1e3, (100ull << 20) / (bp[g] * 1e6));
      }
    }
  }
  return 0;
}
