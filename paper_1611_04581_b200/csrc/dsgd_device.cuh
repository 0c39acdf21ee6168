// dsgd_device.cuh -- device-side building blocks of the B200 update path.
//
// * Reference-order arithmetic: every operation of the reference update
//   rules (protocols.cpp, core.cpp:101, param_vec.cpp) is one explicitly
//   rounded IEEE op (__fadd_rn/__dmul_rn ...), so nvcc can never contract
//   a*b+c into an FMA.  The fp64 instantiation therefore reproduces the
//   reference bit-for-bit and the fp32 one is the same operation order in
//   binary32 (checked against oracle/ in tests/).
// * 128-bit vector access (float4 / double2) for the streaming kernels.
// * Cross-GPU flags: acquire/release at system scope over NVLink-mapped
//   peer memory, bounded by %globaltimer so a dead peer turns into
//   DSGD_ETIMEOUT instead of a hung GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dsgd {

constexpr int kMaxLocal = 32;  // == DSGD_MAX_LOCAL_NODES
constexpr int kMaxWait = 16;
constexpr int kBlock = 256;
constexpr uint32_t kNormSlots = 1024;  // rounds of grad-norm sums between folds

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------------------ 128-bit vectors
template <typename T>
struct Vec {
  static constexpr int N = 16 / sizeof(T);
  union {
    uint4 u;
    T t[N];
  };
};

template <typename T>
__device__ __forceinline__ Vec<T> ld_vec(const T* p) {  // coherent load (may be written elsewhere)
  Vec<T> v;
  v.u = *reinterpret_cast<const uint4*>(p);
  return v;
}
template <typename T>
__device__ __forceinline__ Vec<T> ld_vec_stream(const T* p) {  // read-once input, evict first
  Vec<T> v;
  v.u = __ldcs(reinterpret_cast<const uint4*>(p));
  return v;
}
template <typename T>
__device__ __forceinline__ Vec<T> ld_vec_ro(const T* p) {  // read-only for the kernel
  Vec<T> v;
  v.u = __ldg(reinterpret_cast<const uint4*>(p));
  return v;
}
template <typename T>
__device__ __forceinline__ void st_vec(T* p, const Vec<T>& v) {
  *reinterpret_cast<uint4*>(p) = v.u;
}

// ------------------------------------------------------- cross-GPU flags
struct WaitSpec {
  const unsigned long long* ptr[kMaxWait];
  unsigned long long val[kMaxWait];
  int n;
  unsigned long long timeout_ns;
  unsigned int* error;
  unsigned long long* trace;    // DSGD_TRACE: [0] entry, [1] after the wait (CTA 0)
};

struct SignalSpec {
  unsigned long long* counter;  // own round counter (IPC-visible); null: no signal
  unsigned long long value;
  unsigned int* arrive;         // grid arrival counter (own device memory)
  unsigned long long* trace;    // DSGD_TRACE: [2] last CTA done
  // 1: the kernel writes only this GPU's memory (peers read it through our
  // L2), so each CTA's arrival is a gpu-scope release and only the last CTA
  // issues the system-scope release of the counter (DSGD_SIGNAL_GPU=0: the
  // per-CTA system fence everywhere)
  int local_only;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread per CTA polls the flags; the barrier then orders every thread's
// later peer loads after the acquire.  Returns false on timeout (the error
// flag is raised and the CTA must skip its work).
__device__ __forceinline__ bool wait_flag(const unsigned long long* p, unsigned long long need,
                                          unsigned long long timeout_ns, unsigned int* error) {
  if (ld_acquire_sys(p) >= need) return true;
  const unsigned long long t0 = globaltimer();
  unsigned ns = 32;
  while (ld_acquire_sys(p) < need) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicExch(error, 1u);
      return false;
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
  return true;
}

// wait_flag for a flag written on this GPU (gpu-scope acquire).
__device__ __forceinline__ bool wait_flag_gpu(const unsigned long long* p, unsigned long long need,
                                              unsigned long long timeout_ns, unsigned int* error) {
  if (ld_acquire_gpu(p) >= need) return true;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_gpu(p) < need) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicExch(error, 1u);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

__device__ __forceinline__ bool block_wait(const WaitSpec& w) {
  // programmatic dependent launch: a kernel that starts with block_wait may
  // be launched while the previous kernel of its stream drains; nothing of
  // it touches global memory before that grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool tr = w.trace && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr) w.trace[0] = globaltimer();
  if (w.n == 0) {
    if (tr) w.trace[1] = globaltimer();
    return true;
  }
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int good = 1;
    for (int i = 0; i < w.n && good; ++i) good = wait_flag(w.ptr[i], w.val[i], w.timeout_ns, w.error);
    // the peers published their buffers with generic-proxy stores; this
    // thread next reads them with cp.async.bulk (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    ok = good;
    if (tr) w.trace[1] = globaltimer();
  }
  __syncthreads();
  return ok != 0;
}

// Every CTA fences its writes at system scope and arrives; the last one to
// arrive publishes the round counter with a release store.
__device__ __forceinline__ void block_signal(const SignalSpec& s) {
  if (s.counter == nullptr) {
    // nothing to publish (single context); the tracer stamps CTA 0's end
    if (s.trace && blockIdx.x == 0) {
      __syncthreads();
      if (threadIdx.x == 0) s.trace[2] = globaltimer();
    }
    return;
  }
  __syncthreads();
  if (s.local_only && threadIdx.x == 0) {
    // release at gpu scope (cumulative over the CTA's writes, ordered by the
    // barrier); the last arrival acquires every CTA's writes and publishes
    // them to the peers with one system-scope release
    const unsigned total = gridDim.x * gridDim.y;
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(s.arrive)
                 : "memory");
    if (prev == total - 1) {
      atomicExch(s.arrive, 0u);
      st_release_sys(s.counter, s.value);
      if (s.trace) s.trace[2] = globaltimer();
    }
    return;
  }
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y;
    const unsigned prev = atomicAdd(s.arrive, 1u);
    if (prev == total - 1) {
      atomicExch(s.arrive, 0u);
      __threadfence_system();
      st_release_sys(s.counter, s.value);
      if (s.trace) s.trace[2] = globaltimer();
    }
  }
}

// ------------------------------------------- async bulk copies (TMA engine)
// cp.async.bulk global -> shared with mbarrier completion: a single thread
// keeps many KB of (NVLink peer) reads in flight without holding registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// shared -> global bulk copy (bulk async-group completion); the destination
// may be a peer GPU's memory (NVLink)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all but the N most recent bulk groups complete (writes done)
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// all but the N most recent bulk groups have read their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy shared-memory writes -> a following bulk copy reads them
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ void block_add_double(double v, double* out) {
  if (out == nullptr) return;
  __shared__ double part[kBlock / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) part[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) atomicAdd(out, v);
  }
  __syncthreads();  // part[] is reused by the next call
}

}  // namespace dsgd
