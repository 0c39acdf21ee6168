// dsgd_kernels.cu -- sm_100a kernels of the B200 aggregation/update path.
//
// All kernels are HBM-streaming, elementwise-parallel over the parameter
// dimension d (the work is 0.3-0.5 flop/byte, so tensor cores are
// irrelevant): 128-bit vectorised coalesced loads/stores, grid-stride over a
// grid sized to the SM count, every reference pass of a round fused into one
// sweep over HBM.  The per-element arithmetic is written once (sgd_delta,
// mix) in the reference's exact operation order; see dsgd_device.cuh.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "dsgd_kernels.cuh"

namespace dsgd {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: one process
// may drive several GPUs (in-process rank groups), so remember what was set
// for every (kernel, current device) pair.
template <typename K>
void smem_attr(K* kernel, size_t smem) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(m);
  size_t& have = set[{(const void*)kernel, dev}];
  if (have < smem) {
    cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    have = smem;
  }
}

// Programmatic dependent launch (DSGD_PDL, default on): the kernel may be
// scheduled while the previous kernel of the stream drains; the kernel
// itself executes griddepcontrol.wait before touching global memory.
static bool pdl_enabled() {
  static const bool pdl = [] {  // DSGD_PDL=0: plain stream-ordered launches
    const char* e = getenv("DSGD_PDL");
    return !(e && e[0] == '0');
  }();
  return pdl;
}

template <typename K, typename A>
cudaError_t launch_pdl(K* kernel, uint32_t grid, uint32_t block, size_t smem, cudaStream_t s,
                       const A& args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args);
}

// Kernels issued by this thread (tail launches included): dsgd_launch_count.
// (the file is compiled once per dtype, DSGD_KERNEL_DTYPE = 32 / 64, in
// parallel; the counter lives in the fp32 object)
#if !defined(DSGD_KERNEL_DTYPE) || DSGD_KERNEL_DTYPE == 32
thread_local uint64_t g_launches = 0;
uint64_t launches_issued() { return g_launches; }
#else
extern thread_local uint64_t g_launches;
#endif
#define DSGD_COUNTED(...) \
  do {                    \
    ++g_launches;         \
    __VA_ARGS__;          \
  } while (0)

// a counted launch with programmatic dependent launch (the kernel must start
// with griddepcontrol.wait -- block_wait does -- before any global access)
#define DSGD_PDL_LAUNCH(kernel, grid, block, smem, stream, args)                    \
  do {                                                                              \
    ++g_launches;                                                                   \
    const cudaError_t e_ = launch_pdl(kernel, grid, block, smem, stream, args);     \
    if (e_ != cudaSuccess) return e_;                                               \
  } while (0)

// compute_local_delta protocols.cpp:85-100 for one coordinate:
//   la = mu != 0 ? theta + mu*delta_prev : theta          (92-93)
//   g  = obj.stochastic_gradient(la)                       (30; quadratic: objectives.cpp:75)
//   g += wd*la  if wd > 0                                  (31-33)
//   g += xi     (the zero noise kind still adds +0)        (98)
//   delta = mu*delta_prev - alpha*g                        (core.cpp:101)
template <typename T>
__device__ __forceinline__ T sgd_delta(T x, T dp, T gb, T s, T o, T xi, T alpha, T mu, T wd,
                                       int mu_nz, int wd_pos, int quad, bool norm, double& nacc) {
  const T la = mu_nz ? radd(x, rmul(mu, dp)) : x;
  T g = quad ? rmul(s, rsub(la, o)) : gb;
  if (wd_pos) g = radd(g, rmul(wd, la));
  if (norm) nacc += (double)g * (double)g;
  g = radd(g, xi);
  return rsub(rmul(mu, dp), rmul(alpha, g));
}

// mix_toward protocols.cpp:42-51: own + beta*(other - own), centred so that
// other == own leaves own bit-exactly unchanged.
template <typename T>
__device__ __forceinline__ T mix(T own, T other, T beta) {
  return radd(own, rmul(beta, rsub(other, own)));
}

// ---------------------------------------------- synthetic gradient source
// Philox4x32-10 counter-based generator + Box-Muller: N(0, sigma^2) synthetic
// gradients / noise on the device (bench inputs; not bit-compatible with the
// host mt19937_64 streams, which the parity path uses instead).
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Device-side gradient noise (F1): N(0, sigma^2) per coordinate from
// Philox(counter = (k / 4, t), key = (seed, node)), Box-Muller on pairs.
// Deterministic in (seed, node, t, k) whatever the vector width; not the
// host mt19937_64 stream (the parity path draws those on the host).
template <int W>
__device__ __forceinline__ void dev_normals(uint64_t key, uint64_t ctr, uint64_t k, float (&z)[W]) {
  const uint64_t q = k >> 2;
  const uint4 r = philox(make_uint4((uint32_t)q, (uint32_t)(q >> 32), (uint32_t)ctr,
                                    (uint32_t)(ctr >> 32)),
                         make_uint2((uint32_t)key, (uint32_t)(key >> 32)));
  const uint32_t lane0 = (uint32_t)(k & 3);
#pragma unroll
  for (int l = 0; l < W; ++l) {
    const uint32_t lane = lane0 + l;
    const uint32_t ua = lane < 2 ? r.x : r.z, ub = lane < 2 ? r.y : r.w;
    const float u1 = ((ua >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = ((ub >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float rad = sqrtf(-2.0f * __logf(u1));
    float sn, cs;
    __sincosf(6.2831853071795864f * u2, &sn, &cs);
    z[l] = (lane & 1) ? rad * sn : rad * cs;
  }
}

// ------------------------------------------------------------------ loads
template <typename T, bool VEC>
struct Lanes {
  static constexpr int W = VEC ? Vec<T>::N : 1;
  T v[W];
};

template <typename T, bool VEC>
__device__ __forceinline__ void ld(Lanes<T, VEC>& r, const T* p, uint64_t k) {
  if constexpr (VEC) {
    Vec<T> t = ld_vec(p + k);
#pragma unroll
    for (int l = 0; l < Vec<T>::N; ++l) r.v[l] = t.t[l];
  } else {
    r.v[0] = p[k];
  }
}
template <typename T, bool VEC>
__device__ __forceinline__ void ld_stream(Lanes<T, VEC>& r, const T* p, uint64_t k) {
  if constexpr (VEC) {
    Vec<T> t = ld_vec_stream(p + k);
#pragma unroll
    for (int l = 0; l < Vec<T>::N; ++l) r.v[l] = t.t[l];
  } else {
    r.v[0] = __ldcs(p + k);
  }
}
template <typename T, bool VEC>
__device__ __forceinline__ void ld_ro(Lanes<T, VEC>& r, const T* p, uint64_t k) {
  if constexpr (VEC) {
    Vec<T> t = ld_vec_ro(p + k);
#pragma unroll
    for (int l = 0; l < Vec<T>::N; ++l) r.v[l] = t.t[l];
  } else {
    r.v[0] = __ldg(p + k);
  }
}
template <typename T, bool VEC>
__device__ __forceinline__ void st(T* p, uint64_t k, const Lanes<T, VEC>& r) {
  if constexpr (VEC) {
    Vec<T> t;
#pragma unroll
    for (int l = 0; l < Vec<T>::N; ++l) t.t[l] = r.v[l];
    st_vec(p + k, t);
  } else {
    p[k] = r.v[0];
  }
}
template <typename T, bool VEC>
__device__ __forceinline__ void zero(Lanes<T, VEC>& r) {
#pragma unroll
  for (int l = 0; l < Lanes<T, VEC>::W; ++l) r.v[l] = T(0);
}

// Gradient-source inputs of one coordinate group.
template <typename T, bool VEC>
__device__ __forceinline__ void ld_grad_inputs(Lanes<T, VEC>& gb, Lanes<T, VEC>& s,
                                               Lanes<T, VEC>& o, Lanes<T, VEC>& xi,
                                               const NodeIO<T>& n, const T* spec, const T* opt,
                                               int quad, uint64_t k) {
  if (quad) {
    ld_ro(s, spec, k);
    ld_ro(o, opt, k);
  } else {
    ld_stream(gb, n.grad, k);
  }
  if (n.noise != nullptr) {
    ld_stream(xi, n.noise, k);
  } else if (n.nsigma != T(0)) {
    constexpr int W = Lanes<T, VEC>::W;
    float z[W];
    dev_normals<W>(n.nkey, n.nctr, n.nbase + k, z);
#pragma unroll
    for (int l = 0; l < W; ++l) xi.v[l] = rmul(n.nsigma, (T)z[l]);
  } else {
    zero(xi);
  }
}

template <typename T>
__device__ __forceinline__ T noise_at(const NodeIO<T>& n, uint64_t k) {
  if (n.noise) return n.noise[k];
  if (n.nsigma == T(0)) return T(0);
  float z[1];
  dev_normals<1>(n.nkey, n.nctr, n.nbase + k, z);
  return rmul(n.nsigma, (T)z[0]);
}

// ------------------------------------------------- fused gossip-family step
// Inputs of one coordinate group, loaded before any store of the iteration
// so two groups per thread are in flight (the compiler cannot hoist loads
// above stores through possibly aliasing pointers).
template <typename T, bool VEC>
struct StepIn {
  Lanes<T, VEC> x, dp, gb, s, o, xi, xj, ax;
};

template <typename T, int MODE, bool VEC>
__device__ __forceinline__ void step_load(const StepArgs<T>& a, const NodeIO<T>& n, uint64_t k,
                                          StepIn<T, VEC>& in) {
  auto& x = in.x;
  auto& dp = in.dp;
  auto& gb = in.gb;
  auto& s = in.s;
  auto& o = in.o;
  auto& xi = in.xi;
  auto& xj = in.xj;
  auto& ax = in.ax;
  ld(x, n.theta_in, k);
  if constexpr (MODE == kModePull || MODE == kModeStale || MODE == kModeMix || MODE == kModeAsync)
    ld(xj, n.partner, k);
  if constexpr (MODE == kModeApply) ld(ax, n.aux, k);
  if constexpr (MODE == kModeApplyDelta) ld(ax, n.partner ? n.partner : n.aux, k);  // avg_t
  if constexpr (MODE == kModeStep || MODE == kModePull || MODE == kModeStale ||
                MODE == kModeArDelta || MODE == kModeLookahead) {
    ld(dp, n.delta, k);
  } else if constexpr (MODE == kModeApplyDelta) {
    if (a.agg)
      dp = ax;             // aggregate scope: delta_prev is the average itself
    else
      ld(dp, n.delta, k);  // per-node scope: own delta_prev
  }
  if constexpr (MODE != kModeMix && MODE != kModeApply && MODE != kModeLookahead)
    ld_grad_inputs(gb, s, o, xi, n, a.spec, a.opt, a.quad, k);
}

template <typename T, int MODE, bool VEC>
__device__ __forceinline__ void step_store(const StepArgs<T>& a, const NodeIO<T>& n, uint64_t k,
                                           const StepIn<T, VEC>& in, bool norm, double& nacc) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  const auto& x = in.x;
  const auto& dp = in.dp;
  const auto& gb = in.gb;
  const auto& s = in.s;
  const auto& o = in.o;
  const auto& xi = in.xi;
  const auto& xj = in.xj;
  const auto& ax = in.ax;
  L out_t, out_d;
#pragma unroll
  for (int l = 0; l < W; ++l) {
    if constexpr (MODE == kModeStep) {
      const T dl = sgd_delta(x.v[l], dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu,
                             a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
      out_d.v[l] = dl;
      out_t.v[l] = radd(x.v[l], dl);  // theta += delta_prev  (param_vec.hpp:49)
    } else if constexpr (MODE == kModePull) {
      const T m = mix(x.v[l], xj.v[l], a.beta);
      const T dl = sgd_delta(m, dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu, a.wd,
                             a.mu_nz, a.wd_pos, a.quad, norm, nacc);
      out_d.v[l] = dl;
      out_t.v[l] = radd(m, dl);
    } else if constexpr (MODE == kModeStale) {
      const T dl = sgd_delta(x.v[l], dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu,
                             a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
      out_d.v[l] = dl;
      out_t.v[l] = radd(mix(x.v[l], xj.v[l], a.beta), dl);
    } else if constexpr (MODE == kModeMix) {
      out_t.v[l] = mix(x.v[l], xj.v[l], a.beta);
    } else if constexpr (MODE == kModeArDelta) {
      out_d.v[l] = sgd_delta(x.v[l], dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu,
                             a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
    } else if constexpr (MODE == kModeApply) {
      out_t.v[l] = radd(x.v[l], ax.v[l]);
    } else if constexpr (MODE == kModeLookahead) {
      // la = theta; la.axpy(mu, delta_prev)  (protocols.cpp:92-93)
      out_t.v[l] = a.mu_nz ? radd(x.v[l], rmul(a.mu, dp.v[l])) : x.v[l];
    } else if constexpr (MODE == kModeApplyDelta) {
      // theta_{t+1} = theta_t + avg_t  (protocols.cpp:126), then round t+1's
      // compute_local_delta at theta_{t+1}, in one pass
      const T x1 = radd(x.v[l], ax.v[l]);
      out_t.v[l] = x1;
      out_d.v[l] = sgd_delta(x1, dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu, a.wd,
                             a.mu_nz, a.wd_pos, a.quad, norm, nacc);
    } else {  // kModeAsync: no lookahead, no momentum; y = x + (-alpha)*g
      T g = a.quad ? rmul(s.v[l], rsub(x.v[l], o.v[l])) : gb.v[l];
      if (a.wd_pos) g = radd(g, rmul(a.wd, x.v[l]));
      if (norm) nacc += (double)g * (double)g;
      g = radd(g, xi.v[l]);
      const T y = radd(x.v[l], rmul(n.alpha, g));  // alpha carries the sign (-alpha)
      out_t.v[l] = mix(y, xj.v[l], a.beta);
    }
  }
  if constexpr (MODE == kModeArDelta) {
    st(n.aux, k, out_d);
    if (n.aux != n.delta) st(n.delta, k, out_d);  // per-node scope keeps the own delta
  } else if constexpr (MODE == kModeApplyDelta) {
    st(n.theta_out, k, out_t);
    st(n.aux, k, out_d);
    if (!a.agg) st(n.delta, k, out_d);
  } else {
    st(n.theta_out, k, out_t);
    if constexpr (MODE == kModeStep || MODE == kModePull || MODE == kModeStale)
      st(n.delta, k, out_d);
  }
}

template <typename T, int MODE, bool VEC>
__device__ __forceinline__ void step_group(const StepArgs<T>& a, const NodeIO<T>& n, uint64_t k,
                                           bool norm, double& nacc) {
  StepIn<T, VEC> in;
  step_load<T, MODE, VEC>(a, n, k, in);
  step_store<T, MODE, VEC>(a, n, k, in, norm, nacc);
}

template <typename T, int MODE, bool VEC>
__global__ void __launch_bounds__(kBlock) k_step(const __grid_constant__ StepArgs<T> a) {
  if (!block_wait(a.wait)) return;
  const uint32_t node = blockIdx.x / a.blocks_per_node;
  const uint32_t bid = blockIdx.x - node * a.blocks_per_node;
  const NodeIO<T>& n = a.node[node];
  const bool norm = n.norm != nullptr;
  double nacc = 0.0;
  constexpr int W = Lanes<T, VEC>::W;
  const uint64_t nv = a.d / W;
  const uint64_t stride = (uint64_t)a.blocks_per_node * blockDim.x;
  const uint64_t first = (uint64_t)bid * blockDim.x + threadIdx.x;
  // two independent groups per iteration keep 2x the bytes in flight
  uint64_t v = first;
  for (; v + stride < nv; v += 2 * stride) {
    step_group<T, MODE, VEC>(a, n, v * W, norm, nacc);
    step_group<T, MODE, VEC>(a, n, (v + stride) * W, norm, nacc);
  }
  if (v < nv) step_group<T, MODE, VEC>(a, n, v * W, norm, nacc);
  if constexpr (VEC) {
    for (uint64_t k = nv * W + first; k < a.d; k += stride)
      step_group<T, MODE, false>(a, n, k, norm, nacc);
  }
  block_add_double(nacc, n.norm);
  block_signal(a.signal);
}

// Gossip-family step of ONE node whose partner snapshot lives in a peer GPU:
// the partner tiles are staged through shared memory by cp.async.bulk
// (kOsStages ahead, mbarrier completion) so the NVLink read stream keeps many
// KB in flight per SM without registers; the local streams use LDG.
constexpr int kStStages = 4;
template <typename T>
__host__ __device__ constexpr uint64_t st_tile() {
  return (uint64_t)kBlock * Vec<T>::N * 2;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kBlock) k_step_tma(const __grid_constant__ StepArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = st_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  if (!block_wait(a.wait)) return;
  const NodeIO<T>& n = a.node[0];
  const uint64_t nt = a.d / TILE;
  const bool norm = n.norm != nullptr;
  double nacc = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    for (int s = 0; s < kStStages; ++s) {
      const uint64_t tile = blockIdx.x + (uint64_t)s * gridDim.x;
      if (tile < nt) {
        mbar_expect_tx(&bars[s], TB);
        bulk_g2s(stage + (uint64_t)s * TILE, n.partner + tile * TILE, TB, &bars[s]);
      }
    }
  }
  __syncthreads();
  for (uint64_t j = 0;; ++j) {
    const uint64_t tile = blockIdx.x + j * gridDim.x;
    if (tile >= nt) break;
    const int s = (int)(j % kStStages);
    const uint32_t parity = (uint32_t)((j / kStStages) & 1);
    const uint64_t k0 = tile * TILE + (uint64_t)threadIdx.x * W;
    const uint64_t k1 = k0 + (uint64_t)kBlock * W;
    StepIn<T, true> i0, i1;
    // local streams (theta, delta, gradient, noise); the partner comes from smem
    ld(i0.x, n.theta_in, k0);
    ld(i1.x, n.theta_in, k1);
    if constexpr (MODE != kModeMix) {
      ld(i0.dp, n.delta, k0);
      ld(i1.dp, n.delta, k1);
      ld_grad_inputs(i0.gb, i0.s, i0.o, i0.xi, n, a.spec, a.opt, a.quad, k0);
      ld_grad_inputs(i1.gb, i1.s, i1.o, i1.xi, n, a.spec, a.opt, a.quad, k1);
    }
    mbar_wait(&bars[s], parity);
    const T* src = stage + (uint64_t)s * TILE + (uint64_t)threadIdx.x * W;
    Vec<T> t0, t1;
    t0.u = *reinterpret_cast<const uint4*>(src);
    t1.u = *reinterpret_cast<const uint4*>(src + (uint64_t)kBlock * W);
#pragma unroll
    for (int l = 0; l < W; ++l) {
      i0.xj.v[l] = t0.t[l];
      i1.xj.v[l] = t1.t[l];
    }
    __syncthreads();  // stage s consumed by every thread
    if (threadIdx.x == 0) {
      const uint64_t nxt = blockIdx.x + (j + kStStages) * gridDim.x;
      if (nxt < nt) {
        mbar_expect_tx(&bars[s], TB);
        bulk_g2s(stage + (uint64_t)s * TILE, n.partner + nxt * TILE, TB, &bars[s]);
      }
    }
    step_store<T, MODE, true>(a, n, k0, i0, norm, nacc);
    step_store<T, MODE, true>(a, n, k1, i1, norm, nacc);
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t kk = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < a.d;
       kk += stride)
    step_group<T, MODE, false>(a, n, kk, norm, nacc);
  block_add_double(nacc, n.norm);
  block_signal(a.signal);
}

// Gossip-family step with EVERY stream (partner snapshot -- local, or a
// peer GPU's over NVLink --, theta, delta, gradient / s+opt, noise) staged
// through shared memory by cp.async.bulk, kStages tiles ahead, for any
// number of local nodes: the tiles of all nodes form one work list
// (node-major), so p workers on one GPU stream as one (configs[1]/[2]
// single-GPU shapes) and one node per GPU gets deep NVLink pipelines.
template <int MODE>
struct StepSlots {
  static constexpr bool kPartner =
      MODE == kModePull || MODE == kModeStale || MODE == kModeMix || MODE == kModeAsync;
  static constexpr bool kGrad = MODE != kModeMix;
  static constexpr bool kDelta = kGrad && MODE != kModeAsync;  // async: no momentum term
};

template <typename T, int MODE>
__host__ __device__ inline int step_nslots(int quad, bool noise) {
  using S = StepSlots<MODE>;
  return (S::kPartner ? 1 : 0) + 1 + (S::kDelta ? 1 : 0) +
         (S::kGrad ? (quad ? 2 : 1) + (noise ? 1 : 0) : 0);
}

template <typename T, int MODE, int kStages>
__global__ void __launch_bounds__(kBlock) k_step_tma2(const __grid_constant__ StepArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using S = StepSlots<MODE>;
  constexpr uint64_t TILE = st_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  // programmatic dependent launch: the next launch may be scheduled now;
  // this one touches no global memory before the previous grid is done
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!block_wait(a.wait)) return;
  const bool noise = a.node[0].noise != nullptr;  // the same for every node of a launch
  // slot layout (identical for every node)
  int q = 0;
  const int s_p = S::kPartner ? q++ : -1;
  const int s_x = q++;
  const int s_dp = S::kDelta ? q++ : -1;
  const int s_g = S::kGrad ? q : -1;
  if (S::kGrad) q += a.quad ? 2 : 1;
  const int s_nz = (S::kGrad && noise) ? q++ : -1;
  const int nsl = q;
  const uint64_t nt = a.d / TILE;
  const uint64_t total = nt * a.n_local;
  auto issue = [&](uint64_t work, int sg) {
    const uint32_t node = (uint32_t)(work / nt);
    const uint64_t off = (work - (uint64_t)node * nt) * TILE;
    const NodeIO<T>& n = a.node[node];
    T* dst = stage + (uint64_t)sg * nsl * TILE;
    mbar_expect_tx(&bars[sg], TB * nsl);
    if (S::kPartner) bulk_g2s(dst + (uint64_t)s_p * TILE, n.partner + off, TB, &bars[sg]);
    bulk_g2s(dst + (uint64_t)s_x * TILE, n.theta_in + off, TB, &bars[sg]);
    if (S::kDelta) bulk_g2s(dst + (uint64_t)s_dp * TILE, n.delta + off, TB, &bars[sg]);
    if (S::kGrad) {
      if (a.quad) {
        bulk_g2s(dst + (uint64_t)s_g * TILE, a.spec + off, TB, &bars[sg]);
        bulk_g2s(dst + (uint64_t)(s_g + 1) * TILE, a.opt + off, TB, &bars[sg]);
      } else {
        bulk_g2s(dst + (uint64_t)s_g * TILE, n.grad + off, TB, &bars[sg]);
      }
      if (noise) bulk_g2s(dst + (uint64_t)s_nz * TILE, n.noise + off, TB, &bars[sg]);
    }
  };
  if (threadIdx.x == 0) {
    for (int sg = 0; sg < kStages; ++sg) mbar_init(&bars[sg], 1);
    fence_mbar_init();
    for (int sg = 0; sg < kStages; ++sg) {
      const uint64_t work = blockIdx.x + (uint64_t)sg * gridDim.x;
      if (work < total) issue(work, sg);
    }
  }
  __syncthreads();
  double nacc = 0.0;
  uint32_t cur = 0xffffffffu;  // node of the running norm accumulator
  for (uint64_t j = 0;; ++j) {
    const uint64_t work = blockIdx.x + j * gridDim.x;
    if (work >= total) break;
    const uint32_t node = (uint32_t)(work / nt);
    const uint64_t tile = work - (uint64_t)node * nt;
    if (node != cur) {  // CTA-uniform: flush the previous node's sum of g^2
      if (cur != 0xffffffffu) block_add_double(nacc, a.node[cur].norm);
      nacc = 0.0;
      cur = node;
    }
    const NodeIO<T>& n = a.node[node];
    const bool norm = n.norm != nullptr;
    const int sg = (int)(j % kStages);
    mbar_wait(&bars[sg], (uint32_t)((j / kStages) & 1));
    const T* base = stage + (uint64_t)sg * nsl * TILE + (uint64_t)threadIdx.x * W;
    StepIn<T, true> in[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t off = (uint64_t)u * kBlock * W;
      auto rd = [&](int slot, Lanes<T, true>& dst) {
        Vec<T> v;
        v.u = *reinterpret_cast<const uint4*>(base + (uint64_t)slot * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) dst.v[l] = v.t[l];
      };
      if (S::kPartner) rd(s_p, in[u].xj);
      rd(s_x, in[u].x);
      if (S::kDelta) rd(s_dp, in[u].dp);
      if (S::kGrad) {
        if (a.quad) {
          rd(s_g, in[u].s);
          rd(s_g + 1, in[u].o);
        } else {
          rd(s_g, in[u].gb);
        }
        if (noise) {
          rd(s_nz, in[u].xi);
        } else if (n.nsigma != T(0)) {
          float z[W];
          dev_normals<W>(n.nkey, n.nctr, n.nbase + tile * TILE + (uint64_t)threadIdx.x * W + off, z);
#pragma unroll
          for (int l = 0; l < W; ++l) in[u].xi.v[l] = rmul(n.nsigma, (T)z[l]);
        } else {
#pragma unroll
          for (int l = 0; l < W; ++l) in[u].xi.v[l] = T(0);
        }
      }
    }
    __syncthreads();  // stage sg consumed by every thread
    if (threadIdx.x == 0) {
      const uint64_t nxt = blockIdx.x + (j + kStages) * gridDim.x;
      if (nxt < total) issue(nxt, sg);
    }
    const uint64_t k0 = tile * TILE + (uint64_t)threadIdx.x * W;
    step_store<T, MODE, true>(a, n, k0, in[0], norm, nacc);
    step_store<T, MODE, true>(a, n, k0 + (uint64_t)kBlock * W, in[1], norm, nacc);
  }
  if (cur != 0xffffffffu) block_add_double(nacc, a.node[cur].norm);
  // ragged tails [nt * TILE, d) of every node: the scalar path
  const uint64_t tail = a.d - nt * TILE;
  if (tail) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint32_t node = 0; node < a.n_local; ++node) {
      const NodeIO<T>& n = a.node[node];
      double tacc = 0.0;
      for (uint64_t kk = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < a.d;
           kk += stride)
        step_group<T, MODE, false>(a, n, kk, n.norm != nullptr, tacc);
      block_add_double(tacc, n.norm);
    }
  }
  block_signal(a.signal);
}

template <typename T, int MODE, int ST>
cudaError_t launch_step_staged_st(const StepArgs<T>& a, cudaStream_t s) {
  const int nsl = step_nslots<T, MODE>(a.quad, a.node[0].noise != nullptr);
  const size_t smem = 128 + (size_t)ST * nsl * st_tile<T>() * sizeof(T);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  smem_attr(k_step_tma2<T, MODE, ST>, smem);
  int resident = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_step_tma2<T, MODE, ST>, kBlock, smem);
  if (resident < 1) resident = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t work = a.d / st_tile<T>() * a.n_local;
  uint32_t g = (uint32_t)sms * (uint32_t)resident;
  if (work < g) g = (uint32_t)(work ? work : 1);
  ++g_launches;
  return launch_pdl(k_step_tma2<T, MODE, ST>, g, kBlock, smem, s, a);
}

template <typename T, int MODE>
cudaError_t launch_step_staged(const StepArgs<T>& a, cudaStream_t s) {
  static const int stages = [] {  // DSGD_STEP_STAGES: 2, 3 (default) or 4 stages in flight
    const char* e = getenv("DSGD_STEP_STAGES");
    const int v = e ? atoi(e) : 3;
    return v <= 2 ? 2 : (v >= 4 ? 4 : 3);
  }();
  if (stages == 2) return launch_step_staged_st<T, MODE, 2>(a, s);
  if (stages == 4) return launch_step_staged_st<T, MODE, 4>(a, s);
  return launch_step_staged_st<T, MODE, 3>(a, s);
}

// Partner-only staging (DSGD_GOSSIP_STAGE_ALL=0), one node per GPU.
template <typename T, int MODE>
cudaError_t launch_step_tma(const StepArgs<T>& a, cudaStream_t s) {
  const size_t smem = 128 + (size_t)kStStages * st_tile<T>() * sizeof(T);
  smem_attr(k_step_tma<T, MODE>, smem);
  static int resident = 0;
  if (!resident) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_step_tma<T, MODE>, kBlock, smem);
    if (resident < 1) resident = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = a.d / st_tile<T>();
  uint32_t g = (uint32_t)sms * (uint32_t)resident;
  if (tiles < g) g = (uint32_t)(tiles ? tiles : 1);
  DSGD_COUNTED(k_step_tma<T, MODE><<<g, kBlock, smem, s>>>(a));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_step(int mode, const StepArgs<T>& a, int vec, uint32_t grid, cudaStream_t s) {
  static const bool staged = [] {  // DSGD_STEP_STAGED=0: the LDG kernels
    const char* e = getenv("DSGD_STEP_STAGED");
    return !(e && e[0] == '0');
  }();
  static const bool all_staged = [] {  // DSGD_GOSSIP_STAGE_ALL=0: stage the peer partner only
    const char* e = getenv("DSGD_GOSSIP_STAGE_ALL");
    return !(e && e[0] == '0');
  }();
  // the staged kernel needs every node's streams 16-B aligned and a whole
  // tile; one node per GPU whose partner is remote always stages it
  const bool tiles = a.d >= st_tile<T>();
  if (vec && tiles && (staged || a.tma_partner) && (all_staged || !a.tma_partner)) {
    switch (mode) {
      case kModeStep: return launch_step_staged<T, kModeStep>(a, s);
      case kModePull: return launch_step_staged<T, kModePull>(a, s);
      case kModeStale: return launch_step_staged<T, kModeStale>(a, s);
      case kModeMix: return launch_step_staged<T, kModeMix>(a, s);
      case kModeAsync: return launch_step_staged<T, kModeAsync>(a, s);
      default: break;
    }
  }
  if (a.tma_partner && vec && a.n_local == 1 && a.blocks_per_node == grid) {
    if (mode == kModePull) return launch_step_tma<T, kModePull>(a, s);
    if (mode == kModeStale) return launch_step_tma<T, kModeStale>(a, s);
    if (mode == kModeMix) return launch_step_tma<T, kModeMix>(a, s);
  }
#define DSGD_STEP_CASE(M)                                                   \
  case M:                                                                   \
    if (vec)                                                                \
      DSGD_COUNTED(k_step<T, M, true><<<grid, kBlock, 0, s>>>(a));                        \
    else                                                                    \
      DSGD_COUNTED(k_step<T, M, false><<<grid, kBlock, 0, s>>>(a));                       \
    break;
  switch (mode) {
    DSGD_STEP_CASE(kModeStep)
    DSGD_STEP_CASE(kModePull)
    DSGD_STEP_CASE(kModeStale)
    DSGD_STEP_CASE(kModeMix)
    DSGD_STEP_CASE(kModeArDelta)
    DSGD_STEP_CASE(kModeApply)
    DSGD_STEP_CASE(kModeAsync)
    DSGD_STEP_CASE(kModeApplyDelta)
    DSGD_STEP_CASE(kModeLookahead)
    default:
      return cudaErrorInvalidValue;
  }
#undef DSGD_STEP_CASE
  return cudaGetLastError();
}

// ----------------------------------------- multi-GPU reduce + all-gather
template <typename T, bool VEC>
__device__ __forceinline__ void ar_reduce_group(const ArReduceArgs<T>& a, uint64_t k) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  L acc, v;
  ld(acc, a.x[a.slice], k);
  for (uint32_t s = 1; s < a.p; ++s) {
    uint32_t node = a.slice + s;
    if (node >= a.p) node -= a.p;
    ld(v, a.x[node], k);
#pragma unroll
    for (int l = 0; l < W; ++l) acc.v[l] = radd(acc.v[l], v.v[l]);
  }
  const T pt = T(a.p);
#pragma unroll
  for (int l = 0; l < W; ++l) acc.v[l] = rdiv(acc.v[l], pt);
  for (uint32_t r = 0; r < a.p; ++r) st(a.avg[r], k, acc);
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_ar_reduce(const __grid_constant__ ArReduceArgs<T> a) {
  if (!block_wait(a.wait)) return;
  constexpr uint64_t W = Vec<T>::N;
  // aligned vector body [vlo, vhi), scalar head/tail
  uint64_t vlo = (a.lo + W - 1) / W * W;
  uint64_t vhi = a.hi / W * W;
  if (vlo > vhi) vlo = vhi = a.hi;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = vlo / W + tid; v < vhi / W; v += stride) ar_reduce_group<T, true>(a, v * W);
  for (uint64_t k = a.lo + tid; k < vlo; k += stride) ar_reduce_group<T, false>(a, k);
  for (uint64_t k = (vhi > vlo ? vhi : vlo) + tid; k < a.hi; k += stride)
    if (k >= vlo) ar_reduce_group<T, false>(a, k);
  block_signal(a.signal);
}

template <typename T>
cudaError_t launch_ar_reduce(const ArReduceArgs<T>& a, uint32_t grid, cudaStream_t s) {
  DSGD_COUNTED(k_ar_reduce<T><<<grid, kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

// ------------------------------------------------ reference ring chunking
__device__ __forceinline__ uint32_t ring_chunk_of(uint64_t k, uint64_t base, uint64_t rem) {
  const uint64_t big = rem * (base + 1);  // chunks 0..rem-1 have base+1 elements
  if (k < big) return (uint32_t)(k / (base + 1));
  return (uint32_t)(rem + (k - big) / base);
}

// ------------------------------------------------ NVLS reduce + broadcast
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

__device__ __forceinline__ void nvls_group(const float* x, float* y, float inv_div) {
  float a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "l"(x)
               : "memory");
  a = __fdiv_rn(a, inv_div);
  b = __fdiv_rn(b, inv_div);
  c = __fdiv_rn(c, inv_div);
  d = __fdiv_rn(d, inv_div);
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(y), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}
// U switch reductions in flight per thread (U x 16 B), then U multicast stores
template <int U>
__device__ __forceinline__ void nvls_groupU(const float* x, float* y, uint64_t step, float div) {
  float r[4 * U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r[4 * u]), "=f"(r[4 * u + 1]), "=f"(r[4 * u + 2]), "=f"(r[4 * u + 3])
                 : "l"(x + u * step)
                 : "memory");
#pragma unroll
  for (int q = 0; q < 4 * U; ++q) r[q] = __fdiv_rn(r[q], div);
#pragma unroll
  for (int u = 0; u < U; ++u)
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(y + u * step),
                 "f"(r[4 * u]), "f"(r[4 * u + 1]), "f"(r[4 * u + 2]), "f"(r[4 * u + 3])
                 : "memory");
}
__device__ __forceinline__ void nvls_scalar(const float* x, float* y, float div) {
  float a;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(a) : "l"(x) : "memory");
  a = __fdiv_rn(a, div);
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(y), "f"(a) : "memory");
}
__device__ __forceinline__ void nvls_scalar(const double* x, double* y, double div) {
  double a;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(a) : "l"(x) : "memory");
  a = __ddiv_rn(a, div);
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(y), "d"(a) : "memory");
}

template <typename T, int U>
__global__ void __launch_bounds__(1024) k_ar_nvls(const __grid_constant__ ArNvlsArgs<T> a) {
  if (!block_wait(a.wait)) return;
  fence_proxy_alias();  // peers wrote x through their unicast mappings
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const T div = T(a.p);
  if constexpr (sizeof(T) == 4) {
    // lo is a multiple of 4 elements (16 B): vector body, scalar tail
    const uint64_t nv = (a.hi - a.lo) / 4;
    uint64_t v = tid;
    for (; v + (U - 1) * stride < nv; v += U * stride)  // U switch reductions in flight
      nvls_groupU<U>(a.x_mc + a.lo + 4 * v, a.avg_mc + a.lo + 4 * v, 4 * stride, div);
    for (; v < nv; v += stride)
      nvls_group(a.x_mc + a.lo + 4 * v, a.avg_mc + a.lo + 4 * v, div);
    for (uint64_t k = a.lo + 4 * nv + tid; k < a.hi; k += stride)
      nvls_scalar(a.x_mc + k, a.avg_mc + k, div);
  } else {
    for (uint64_t k = a.lo + tid; k < a.hi; k += stride) nvls_scalar(a.x_mc + k, a.avg_mc + k, div);
  }
  fence_proxy_alias();
  block_signal(a.signal);
}

template <typename T>
cudaError_t launch_ar_nvls(const ArNvlsArgs<T>& a, uint32_t grid, cudaStream_t s) {
  // DSGD_AR_COMM_SMEM=<KB>: reserve (unused) shared memory per CTA so that a
  // reduce CTA cannot share an SM with a (144 KB) delta CTA: SM-issued NVLink
  // traffic starves when co-resident with an HBM stream, not when the two
  // run on disjoint SMs (profiles/r1_nvlink_probe.txt, "split" rows)
  static const int pad = [] {
    const char* e = getenv("DSGD_AR_COMM_SMEM");
    const int kb = e ? atoi(e) : 120;  // measured best at p = 4 (r1_tune_allreduce_n4/split/)
    return kb < 0 ? 0 : (kb > 200 ? 200 : kb) * 1024;
  }();
  static const int unroll = [] {  // DSGD_NVLS_UNROLL: switch reductions in flight per thread
    const char* e = getenv("DSGD_NVLS_UNROLL");
    // 2 measured best at p = 4, 25M (263 vs 272 / 287 us per round for 4 / 8,
    // profiles/r2_nvls_knobs.md): more requests in flight congest the switch
    const int u = e ? atoi(e) : 2;
    return u >= 8 ? 8 : (u >= 4 ? 4 : (u >= 2 ? 2 : 1));
  }();
  if (pad) {
    smem_attr(k_ar_nvls<T, 1>, pad);
    smem_attr(k_ar_nvls<T, 2>, pad);
    smem_attr(k_ar_nvls<T, 4>, pad);
    smem_attr(k_ar_nvls<T, 8>, pad);
  }
  // one padded CTA per SM: 1024 threads keep enough switch reductions in flight
  const int threads = pad ? 1024 : kBlock;
  if (unroll == 8)
    DSGD_PDL_LAUNCH((k_ar_nvls<T, 8>), grid, threads, pad, s, a);
  else if (unroll == 1)
    DSGD_PDL_LAUNCH((k_ar_nvls<T, 1>), grid, threads, pad, s, a);
  else if (unroll == 2)
    DSGD_PDL_LAUNCH((k_ar_nvls<T, 2>), grid, threads, pad, s, a);
  else
    DSGD_PDL_LAUNCH((k_ar_nvls<T, 4>), grid, threads, pad, s, a);
  return cudaGetLastError();
}

// ------------------------------------------------ one-shot all-reduce round
// The ring-order average of lane l of every rank's previous exchange value.
template <typename T, bool VEC, int P>
__device__ __forceinline__ void ring_average(const Lanes<T, VEC> (&v)[P], uint64_t k,
                                             uint64_t base, uint64_t rem, Lanes<T, VEC>& avg) {
  constexpr int W = Lanes<T, VEC>::W;
#pragma unroll
  for (int l = 0; l < W; ++l) {
    const uint32_t c = ring_chunk_of(k + l, base, rem);
    T sum = T(0);
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const uint32_t node = c + r >= (uint32_t)P ? c + r - P : c + r;
      T val = v[0].v[l];
#pragma unroll
      for (int q = 1; q < P; ++q)
        if (q == (int)node) val = v[q].v[l];
      sum = r == 0 ? val : radd(sum, val);  // transport.cpp:224-226 fold
    }
    avg.v[l] = rdiv(sum, T(P));             // transport.cpp:229-235
  }
}

template <typename T, bool VEC, int P>
struct OneshotIn {
  Lanes<T, VEC> v[P], x, dp, gb, s, o, xi;
};

template <typename T, bool VEC, int P>
__device__ __forceinline__ void oneshot_load(const ArOneShotArgs<T>& a, uint64_t k,
                                             OneshotIn<T, VEC, P>& in) {
  const NodeIO<T>& n = a.node;
  if (a.pending) {
#pragma unroll
    for (int r = 0; r < P; ++r) ld(in.v[r], a.x_prev[r], k);  // P - 1 NVLink loads in flight
  }
  ld(in.x, n.theta_in, k);
  if (a.apply_only) return;
  if (!a.pending || !a.agg) ld(in.dp, n.delta, k);
  ld_grad_inputs(in.gb, in.s, in.o, in.xi, n, a.spec, a.opt, a.quad, k);
}

template <typename T, bool VEC, int P>
__device__ __forceinline__ void oneshot_store(const ArOneShotArgs<T>& a, uint64_t k,
                                              const OneshotIn<T, VEC, P>& in, bool norm,
                                              double& nacc) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  const NodeIO<T>& n = a.node;
  L avg, dp = in.dp, ot, od;
  if (a.apply_only) {
    ring_average<T, VEC, P>(in.v, k, a.ring_base, a.ring_rem, avg);
#pragma unroll
    for (int l = 0; l < W; ++l) ot.v[l] = radd(in.x.v[l], avg.v[l]);
    st(n.theta_out, k, ot);
    if (a.agg) st(n.delta, k, avg);
    return;
  }
  if (a.pending) {
    ring_average<T, VEC, P>(in.v, k, a.ring_base, a.ring_rem, avg);
    if (a.agg) dp = avg;  // aggregate scope: delta_prev is the average
  }
#pragma unroll
  for (int l = 0; l < W; ++l) {
    const T x1 = a.pending ? radd(in.x.v[l], avg.v[l]) : in.x.v[l];  // theta += avg (protocols.cpp:126)
    ot.v[l] = x1;
    od.v[l] = sgd_delta(x1, dp.v[l], in.gb.v[l], in.s.v[l], in.o.v[l], in.xi.v[l], n.alpha, a.mu,
                        a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
  }
  if (a.pending) st(n.theta_out, k, ot);
  st(a.x_out, k, od);
  if (!a.agg || !a.pending) st(n.delta, k, od);
}

template <typename T, bool VEC, int P>
__device__ __forceinline__ void oneshot_group(const ArOneShotArgs<T>& a, uint64_t k, bool norm,
                                              double& nacc) {
  OneshotIn<T, VEC, P> in;
  oneshot_load<T, VEC, P>(a, k, in);
  oneshot_store<T, VEC, P>(a, k, in, norm, nacc);
}

template <typename T, bool VEC, int P>
__global__ void __launch_bounds__(kBlock) k_ar_oneshot(const __grid_constant__ ArOneShotArgs<T> a) {
  if (!block_wait(a.wait)) return;
  constexpr int W = Lanes<T, VEC>::W;
  const bool norm = a.node.norm != nullptr;
  double nacc = 0.0;
  const uint64_t nv = a.d / W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t v = first;
  for (; v + stride < nv; v += 2 * stride) {  // two groups in flight per thread
    OneshotIn<T, VEC, P> i0, i1;
    oneshot_load<T, VEC, P>(a, v * W, i0);
    oneshot_load<T, VEC, P>(a, (v + stride) * W, i1);
    oneshot_store<T, VEC, P>(a, v * W, i0, norm, nacc);
    oneshot_store<T, VEC, P>(a, (v + stride) * W, i1, norm, nacc);
  }
  if (v < nv) oneshot_group<T, VEC, P>(a, v * W, norm, nacc);
  if constexpr (VEC) {
    for (uint64_t k = nv * W + first; k < a.d; k += stride)
      oneshot_group<T, false, P>(a, k, norm, nacc);
  }
  block_add_double(nacc, a.node.norm);
  block_signal(a.signal);
}

// One-shot round with the peer exchange buffers staged through shared memory
// by bulk async copies (TMA engine, mbarrier completion), kStages tiles
// ahead: the NVLink stream's bytes in flight no longer cost registers.
constexpr int kOsStages = 4;
constexpr int kOsVecPerThread = 2;

template <typename T>
__host__ __device__ constexpr uint64_t os_tile() {  // elements per tile
  return (uint64_t)kBlock * Vec<T>::N * kOsVecPerThread;
}

template <typename T, int P>
__device__ __forceinline__ void os_load_local(const ArOneShotArgs<T>& a, uint32_t me, uint64_t k,
                                              OneshotIn<T, true, P>& in) {
  const NodeIO<T>& n = a.node;
  (void)me;
  ld(in.x, n.theta_in, k);
  if (!a.agg) ld(in.dp, n.delta, k);
  ld_grad_inputs(in.gb, in.s, in.o, in.xi, n, a.spec, a.opt, a.quad, k);
}

// Every rank's tile (own included) sits in slot r of the stage, so the
// register array is indexed at compile time only.
template <typename T, int P>
__device__ __forceinline__ void os_load_stage(uint32_t me, const T* src0, OneshotIn<T, true, P>& in) {
  constexpr uint64_t TILE = os_tile<T>();
  (void)me;
#pragma unroll
  for (int r = 0; r < P; ++r) {
    Vec<T> t;
    t.u = *reinterpret_cast<const uint4*>(src0 + (uint64_t)r * TILE);
#pragma unroll
    for (int l = 0; l < Vec<T>::N; ++l) in.v[r].v[l] = t.t[l];
  }
}

// Thread 0: bulk-copy every remote rank's tile j (of this CTA) into stage s.
template <typename T, int P>
__device__ __forceinline__ void os_issue(const ArOneShotArgs<T>& a, uint32_t me, uint64_t nt,
                                         uint64_t j, int s, uint64_t* bars, T* stage) {
  constexpr uint64_t TILE = os_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  const uint64_t tile = blockIdx.x + j * gridDim.x;
  if (tile >= nt) return;
  (void)me;
  mbar_expect_tx(&bars[s], TB * P);
#pragma unroll
  for (int r = 0; r < P; ++r)  // P - 1 peers over NVLink + the own tile from local HBM
    bulk_g2s(stage + ((uint64_t)s * P + r) * TILE, a.x_prev[r] + tile * TILE, TB, &bars[s]);
}

template <typename T, int P>
__global__ void __launch_bounds__(kBlock) k_ar_oneshot_tma(const __grid_constant__ ArOneShotArgs<T> a,
                                                           uint32_t me) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = os_tile<T>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  if (!block_wait(a.wait)) return;
  const uint64_t nt = a.d / TILE;
  const bool norm = a.node.norm != nullptr;
  double nacc = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kOsStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < kOsStages; ++s) os_issue<T, P>(a, me, nt, s, s, bars, stage);
  using L = Lanes<T, true>;
  constexpr int W = L::W;
  for (uint64_t j = 0;; ++j) {
    const uint64_t tile = blockIdx.x + j * gridDim.x;
    if (tile >= nt) break;
    const int s = (int)(j % kOsStages);
    const uint32_t parity = (uint32_t)((j / kOsStages) & 1);
    OneshotIn<T, true, P> in0, in1;
    const uint64_t k0 = tile * TILE + (uint64_t)threadIdx.x * W;
    const uint64_t k1 = k0 + (uint64_t)kBlock * W;
    os_load_local<T, P>(a, me, k0, in0);  // local streams through registers (HBM latency)
    os_load_local<T, P>(a, me, k1, in1);
    mbar_wait(&bars[s], parity);
    const T* st0 = stage + (uint64_t)s * P * TILE + (uint64_t)threadIdx.x * W;
    os_load_stage<T, P>(me, st0, in0);
    os_load_stage<T, P>(me, st0 + (uint64_t)kBlock * W, in1);
    __syncthreads();  // every thread is done with stage s
    if (threadIdx.x == 0) os_issue<T, P>(a, me, nt, j + kOsStages, s, bars, stage);
    oneshot_store<T, true, P>(a, k0, in0, norm, nacc);
    oneshot_store<T, true, P>(a, k1, in1, norm, nacc);
  }
  // ragged tail [nt * TILE, d): plain global loads
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t kk = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < a.d;
       kk += stride)
    oneshot_group<T, false, P>(a, kk, norm, nacc);
  block_add_double(nacc, a.node.norm);
  block_signal(a.signal);
}

// One-shot round with EVERY stream staged through shared memory (every
// rank's exchange tile + this rank's theta, delta, gradient / s+opt, noise):
// S stages of up to P + 5 8-KB tiles per CTA, registers hold no loads.
// kOs2Stages stages (DSGD_OS_STAGES, default 2).
template <typename T, int P, int kOs2Stages>
__global__ void __launch_bounds__(kBlock) k_ar_oneshot_tma2(const __grid_constant__ ArOneShotArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = os_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  if (!block_wait(a.wait)) return;
  const NodeIO<T>& n = a.node;
  // slots: [0, P) exchange tiles, then theta, delta (per-node), g | s, opt, noise
  const T* src[kMaxFusedRanks + 5];
  int q = 0;
#pragma unroll
  for (int r = 0; r < P; ++r) src[q++] = a.x_prev[r];
  const int s_x = q;
  src[q++] = n.theta_in;
  const int s_dp = q;
  if (!a.agg) src[q++] = n.delta;
  const int s_g = q;
  if (a.quad) {
    src[q++] = a.spec;
    src[q++] = a.opt;
  } else {
    src[q++] = n.grad;
  }
  const int s_nz = q;
  if (n.noise) src[q++] = n.noise;
  const int nsl = q;
  const uint64_t nt = a.d / TILE;
  if (threadIdx.x == 0) {
    for (int sg = 0; sg < kOs2Stages; ++sg) mbar_init(&bars[sg], 1);
    fence_mbar_init();
    for (int sg = 0; sg < kOs2Stages; ++sg) {
      const uint64_t tile = blockIdx.x + (uint64_t)sg * gridDim.x;
      if (tile < nt) {
        mbar_expect_tx(&bars[sg], TB * nsl);
        for (int i = 0; i < nsl; ++i)
          bulk_g2s(stage + ((uint64_t)sg * nsl + i) * TILE, src[i] + tile * TILE, TB, &bars[sg]);
      }
    }
  }
  __syncthreads();
  const bool norm = n.norm != nullptr;
  double nacc = 0.0;
  for (uint64_t j = 0;; ++j) {
    const uint64_t tile = blockIdx.x + j * gridDim.x;
    if (tile >= nt) break;
    const int sg = (int)(j % kOs2Stages);
    mbar_wait(&bars[sg], (uint32_t)((j / kOs2Stages) & 1));
    const T* base = stage + (uint64_t)sg * nsl * TILE + (uint64_t)threadIdx.x * W;
    OneshotIn<T, true, P> in[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t off = (uint64_t)u * kBlock * W;
      auto rd = [&](int slot, Lanes<T, true>& dst) {
        Vec<T> v;
        v.u = *reinterpret_cast<const uint4*>(base + (uint64_t)slot * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) dst.v[l] = v.t[l];
      };
#pragma unroll
      for (int r = 0; r < P; ++r) rd(r, in[u].v[r]);
      rd(s_x, in[u].x);
      if (!a.agg) rd(s_dp, in[u].dp);
      if (a.quad) {
        rd(s_g, in[u].s);
        rd(s_g + 1, in[u].o);
      } else {
        rd(s_g, in[u].gb);
      }
      if (n.noise) {
        rd(s_nz, in[u].xi);
      } else if (n.nsigma != T(0)) {
        float z[W];
        dev_normals<W>(n.nkey, n.nctr, n.nbase + tile * TILE + (uint64_t)threadIdx.x * W + off, z);
#pragma unroll
        for (int l = 0; l < W; ++l) in[u].xi.v[l] = rmul(n.nsigma, (T)z[l]);
      } else {
#pragma unroll
        for (int l = 0; l < W; ++l) in[u].xi.v[l] = T(0);
      }
    }
    __syncthreads();  // stage consumed
    if (threadIdx.x == 0) {
      const uint64_t nxt = blockIdx.x + (j + kOs2Stages) * gridDim.x;
      if (nxt < nt) {
        mbar_expect_tx(&bars[sg], TB * nsl);
        for (int i = 0; i < nsl; ++i)
          bulk_g2s(stage + ((uint64_t)sg * nsl + i) * TILE, src[i] + nxt * TILE, TB, &bars[sg]);
      }
    }
    const uint64_t k0 = tile * TILE + (uint64_t)threadIdx.x * W;
    oneshot_store<T, true, P>(a, k0, in[0], norm, nacc);
    oneshot_store<T, true, P>(a, k0 + (uint64_t)kBlock * W, in[1], norm, nacc);
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t kk = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < a.d;
       kk += stride)
    oneshot_group<T, false, P>(a, kk, norm, nacc);
  block_add_double(nacc, a.node.norm);
  block_signal(a.signal);
}

template <typename T, int P, int S>
cudaError_t launch_os2(const ArOneShotArgs<T>& a, int max_ctas, cudaStream_t s) {
  const int nsl = P + 1 + (a.agg ? 0 : 1) + (a.quad ? 2 : 1) + (a.node.noise ? 1 : 0);
  const size_t smem = 128 + (size_t)S * nsl * os_tile<T>() * sizeof(T);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  smem_attr(k_ar_oneshot_tma2<T, P, S>, smem);
  int resident = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_ar_oneshot_tma2<T, P, S>, kBlock, smem);
  if (resident < 1) resident = 1;
  if (max_ctas > 0 && resident > max_ctas) resident = max_ctas;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = a.d / os_tile<T>();
  uint32_t g = (uint32_t)sms * (uint32_t)resident;
  if (tiles < g) g = (uint32_t)(tiles ? tiles : 1);
  DSGD_PDL_LAUNCH((k_ar_oneshot_tma2<T, P, S>), g, kBlock, smem, s, a);
  return cudaGetLastError();
}

template <typename T, int P>
cudaError_t launch_ar_oneshot_p(const ArOneShotArgs<T>& a, int vec, uint32_t grid, cudaStream_t s) {
  static const bool all_staged = [] {  // DSGD_OS_STAGE_ALL=0: stage only the exchange tiles
    const char* e = getenv("DSGD_OS_STAGE_ALL");
    return !(e && e[0] == '0');
  }();
  if (vec && a.pending && !a.apply_only && a.tma_rank >= 0 && all_staged) {
    static const int stages = [] {
      // 2 stages at 3 CTAs/SM measured best at p = 2, d = 25M (182.5 vs
      // 192-203 us/round for 3 stages at 2 CTAs/SM, profiles/r1_os_stages_n2.md)
      const char* e = getenv("DSGD_OS_STAGES");
      const int v = e ? atoi(e) : 2;
      return v < 2 ? 2 : (v > 6 ? 6 : v);
    }();
    static const int max_ctas = [] {  // DSGD_OS_CTAS: cap on CTAs per SM (0: occupancy)
      const char* e = getenv("DSGD_OS_CTAS");
      return e ? atoi(e) : 0;
    }();
    switch (stages) {
      case 2: return launch_os2<T, P, 2>(a, max_ctas, s);
      case 4: return launch_os2<T, P, 4>(a, max_ctas, s);
      case 5: return launch_os2<T, P, 5>(a, max_ctas, s);
      case 6: return launch_os2<T, P, 6>(a, max_ctas, s);
      default: return launch_os2<T, P, 3>(a, max_ctas, s);
    }
  }
  if (vec && a.pending && !a.apply_only && a.tma_rank >= 0) {
    const size_t smem = 128 + (size_t)kOsStages * P * os_tile<T>() * sizeof(T);
    smem_attr(k_ar_oneshot_tma<T, P>, smem);
    static int resident = 0;  // CTAs per SM at this smem size (persistent grid)
    if (!resident) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_ar_oneshot_tma<T, P>, kBlock,
                                                    smem);
      if (resident < 1) resident = 1;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t tiles = a.d / os_tile<T>();
    uint32_t g = (uint32_t)sms * (uint32_t)resident;
    if (tiles < g) g = (uint32_t)(tiles ? tiles : 1);
    (void)grid;
    DSGD_COUNTED(k_ar_oneshot_tma<T, P><<<g, kBlock, smem, s>>>(a, (uint32_t)a.tma_rank));
  } else if (vec) {
    DSGD_COUNTED(k_ar_oneshot<T, true, P><<<grid, kBlock, 0, s>>>(a));
  } else {
    DSGD_COUNTED(k_ar_oneshot<T, false, P><<<grid, kBlock, 0, s>>>(a));
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_ar_oneshot(const ArOneShotArgs<T>& a, int vec, uint32_t grid, cudaStream_t s) {
  switch (a.p) {
    case 2: return launch_ar_oneshot_p<T, 2>(a, vec, grid, s);
    case 3: return launch_ar_oneshot_p<T, 3>(a, vec, grid, s);
    case 4: return launch_ar_oneshot_p<T, 4>(a, vec, grid, s);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------- single-context all-reduce round
// allreduce_round protocols.cpp:110-131 for p nodes on one GPU, one pass:
// every node's delta, the pivot-form mean of param_vec.cpp:26-38
//   dev = 0; dev += (d_i - d_0) for i = 1..p-1; avg = d_0 + dev * (1/p)
// and the apply theta_i += avg, delta_prev_i = aggregate ? avg : d_i.
template <typename T, bool VEC, bool NORM>
__global__ void __launch_bounds__(kBlock) k_allreduce_local(const __grid_constant__ AllreduceArgs<T> a) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  double nacc[NORM ? kMaxLocal : 1];
  if constexpr (NORM)
    for (uint32_t i = 0; i < a.p; ++i) nacc[i] = 0.0;
  const uint64_t nv = a.d / W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const uint64_t k = v * W;
    L d0, dev, avg;
    zero(dev);
    for (uint32_t i = 0; i < a.p; ++i) {
      const NodeIO<T>& n = a.node[i];
      L x, dp, gb, s, o, xi, di;
      ld(x, n.theta_in, k);
      ld(dp, n.delta, k);
      ld_grad_inputs(gb, s, o, xi, n, a.spec, a.opt, a.quad, k);
      double dummy = 0.0;
#pragma unroll
      for (int l = 0; l < W; ++l) {
        di.v[l] = sgd_delta(x.v[l], dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu,
                            a.wd, a.mu_nz, a.wd_pos, a.quad, NORM, NORM ? nacc[i] : dummy);
        if (i == 0)
          d0.v[l] = di.v[l];
        else
          dev.v[l] = radd(dev.v[l], rsub(di.v[l], d0.v[l]));
      }
      if (a.per_node) st(n.delta, k, di);
    }
#pragma unroll
    for (int l = 0; l < W; ++l) avg.v[l] = radd(d0.v[l], rmul(dev.v[l], a.inv_p));
    for (uint32_t i = 0; i < a.p; ++i) {
      const NodeIO<T>& n = a.node[i];
      L x, out;
      ld(x, n.theta_in, k);
#pragma unroll
      for (int l = 0; l < W; ++l) out.v[l] = radd(x.v[l], avg.v[l]);
      st(n.theta_out, k, out);
      if (!a.per_node) st(n.delta, k, avg);
    }
  }
  if constexpr (NORM)
    for (uint32_t i = 0; i < a.p; ++i) block_add_double(nacc[i], a.node[i].norm);
}

// p = 1 round with every input stream (theta, delta, gradient or s/opt,
// noise) staged through shared memory by cp.async.bulk, kLtStages tiles
// ahead: the HBM read stream's bytes in flight cost no registers.
constexpr int kLtStages = 3;
template <typename T>
__host__ __device__ constexpr uint64_t lt_tile() {
  return (uint64_t)kBlock * Vec<T>::N * 2;
}

template <typename T, bool NORM>
__global__ void __launch_bounds__(kBlock) k_local_tma(const __grid_constant__ AllreduceArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = lt_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  const NodeIO<T>& n = a.node[0];
  const T* src[5];
  int ns = 0;
  src[ns++] = n.theta_in;
  src[ns++] = n.delta;
  if (a.quad) {
    src[ns++] = a.spec;
    src[ns++] = a.opt;
  } else {
    src[ns++] = n.grad;
  }
  if (n.noise) src[ns++] = n.noise;
  const uint64_t nt = a.d / TILE;
  // programmatic dependent launch: let the next round's grid be scheduled
  // now.  Then either wait until the previous round's grid has finished and
  // its writes are visible (theta / delta are read-after-write across
  // rounds), or -- chained rounds -- only until the previous round's CTA
  // with this index, the sole writer of this CTA's tiles (and sole reader of
  // the snapshot this CTA overwrites), has published them: no grid-wide
  // drain between rounds.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int chain_ok;
  if (a.cta_chain) {
    if (threadIdx.x == 0) {
      chain_ok = wait_flag_gpu(&a.cta_flags[blockIdx.x], a.cta_seq - 1, a.timeout_ns, a.error);
      // generic-proxy stores of the previous round -> this round's bulk reads
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
    if (!chain_ok) return;
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLtStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    for (int s = 0; s < kLtStages; ++s) {
      const uint64_t tile = blockIdx.x + (uint64_t)s * gridDim.x;
      if (tile < nt) {
        mbar_expect_tx(&bars[s], TB * ns);
        for (int q = 0; q < ns; ++q)
          bulk_g2s(stage + ((uint64_t)s * 5 + q) * TILE, src[q] + tile * TILE, TB, &bars[s]);
      }
    }
  }
  __syncthreads();
  constexpr bool norm = NORM;  // grad_norm_out: sum of g^2 (fp64)
  double nacc = 0.0;
  for (uint64_t j = 0;; ++j) {
    const uint64_t tile = blockIdx.x + j * gridDim.x;
    if (tile >= nt) break;
    const int s = (int)(j % kLtStages);
    mbar_wait(&bars[s], (uint32_t)((j / kLtStages) & 1));
    Lanes<T, true> x[2], dp[2], gb[2], sp[2], o[2], xi[2];
    const T* base = stage + (uint64_t)s * 5 * TILE + (uint64_t)threadIdx.x * W;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t off = (uint64_t)u * kBlock * W;
      Vec<T> v;
      v.u = *reinterpret_cast<const uint4*>(base + off);
#pragma unroll
      for (int l = 0; l < W; ++l) x[u].v[l] = v.t[l];
      v.u = *reinterpret_cast<const uint4*>(base + TILE + off);
#pragma unroll
      for (int l = 0; l < W; ++l) dp[u].v[l] = v.t[l];
      int q = 2;
      if (a.quad) {
        v.u = *reinterpret_cast<const uint4*>(base + q * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) sp[u].v[l] = v.t[l];
        v.u = *reinterpret_cast<const uint4*>(base + (q + 1) * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) o[u].v[l] = v.t[l];
        q += 2;
      } else {
        v.u = *reinterpret_cast<const uint4*>(base + q * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) gb[u].v[l] = v.t[l];
        q += 1;
      }
      if (n.noise) {
        v.u = *reinterpret_cast<const uint4*>(base + q * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) xi[u].v[l] = v.t[l];
      } else if (n.nsigma != T(0)) {
        float z[W];
        dev_normals<W>(n.nkey, n.nctr, n.nbase + tile * TILE + (uint64_t)threadIdx.x * W + off, z);
#pragma unroll
        for (int l = 0; l < W; ++l) xi[u].v[l] = rmul(n.nsigma, (T)z[l]);
      } else {
#pragma unroll
        for (int l = 0; l < W; ++l) xi[u].v[l] = T(0);
      }
    }
    __syncthreads();  // stage s consumed
    if (threadIdx.x == 0) {
      const uint64_t nxt = blockIdx.x + (j + kLtStages) * gridDim.x;
      if (nxt < nt) {
        mbar_expect_tx(&bars[s], TB * ns);
        for (int q = 0; q < ns; ++q)
          bulk_g2s(stage + ((uint64_t)s * 5 + q) * TILE, src[q] + nxt * TILE, TB, &bars[s]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t k = tile * TILE + (uint64_t)threadIdx.x * W + (uint64_t)u * kBlock * W;
      Lanes<T, true> ot, od;
#pragma unroll
      for (int l = 0; l < W; ++l) {
        const T d0 = sgd_delta(x[u].v[l], dp[u].v[l], gb[u].v[l], sp[u].v[l], o[u].v[l],
                               xi[u].v[l], n.alpha, a.mu, a.wd, a.mu_nz, a.wd_pos, a.quad, norm,
                               nacc);
        const T avg = radd(d0, rmul(T(0), a.inv_p));  // spatial_mean of one node (param_vec.cpp:37)
        ot.v[l] = radd(x[u].v[l], avg);
        od.v[l] = a.per_node ? d0 : avg;
      }
      st(n.theta_out, k, ot);
      st(n.delta, k, od);
    }
  }
  // ragged tail: the plain kernel's scalar path
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.d;
       k += stride) {
    Lanes<T, false> x, dp, gb, sp, o, xi;
    ld(x, n.theta_in, k);
    ld(dp, n.delta, k);
    ld_grad_inputs(gb, sp, o, xi, n, a.spec, a.opt, a.quad, k);
    const T d0 = sgd_delta(x.v[0], dp.v[0], gb.v[0], sp.v[0], o.v[0], xi.v[0], n.alpha, a.mu,
                           a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
    const T avg = radd(d0, rmul(T(0), a.inv_p));
    n.theta_out[k] = radd(x.v[0], avg);
    n.delta[k] = a.per_node ? d0 : avg;
  }
  if constexpr (NORM) block_add_double(nacc, n.norm);
  if (a.cta_flags) {
    __syncthreads();  // every thread's theta / delta stores before the release
    if (threadIdx.x == 0) st_release_gpu(&a.cta_flags[blockIdx.x], a.cta_seq);
  }
}

template <typename T>
cudaError_t launch_local_tma(const AllreduceArgs<T>& a, cudaStream_t s) {
  const size_t smem = 128 + (size_t)kLtStages * 5 * lt_tile<T>() * sizeof(T);
  smem_attr(k_local_tma<T, false>, smem);
  smem_attr(k_local_tma<T, true>, smem);
  static int resident = 0;
  if (!resident) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_local_tma<T, false>, kBlock, smem);
    if (resident < 1) resident = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = a.d / lt_tile<T>();
  uint32_t g = (uint32_t)sms * (uint32_t)resident;
  if (tiles < g) g = (uint32_t)(tiles ? tiles : 1);
  ++g_launches;
  if (a.node[0].norm) return launch_pdl(k_local_tma<T, true>, g, kBlock, smem, s, a);
  return launch_pdl(k_local_tma<T, false>, g, kBlock, smem, s, a);
}

// Two-shot all-reduce delta kernel (kModeArDelta / kModeApplyDelta) of one
// node with its input streams staged through shared memory by cp.async.bulk
// (kLtStages tiles ahead).  Saturates HBM from a fraction of the SMs, so the
// NVLink-bound reduce of the other pipeline can run on the rest.
template <typename T, int MODE>
__global__ void __launch_bounds__(kBlock) k_ard_tma(const __grid_constant__ StepArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = lt_tile<T>();
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  constexpr bool PEND = MODE == kModeApplyDelta;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  if (!block_wait(a.wait)) return;
  const NodeIO<T>& n = a.node[0];
  const bool need_dp = !(PEND && a.agg);
  const T* src[6];
  int ns = 0;
  src[ns++] = n.theta_in;                              // slot 0
  if (PEND) src[ns++] = n.partner;                     // slot 1: avg of round t-1
  const int s_dp = ns;
  if (need_dp) src[ns++] = n.delta;
  const int s_g = ns;
  if (a.quad) {
    src[ns++] = a.spec;
    src[ns++] = a.opt;
  } else {
    src[ns++] = n.grad;
  }
  const int s_nz = ns;
  if (n.noise) src[ns++] = n.noise;
  const uint64_t nt = a.d / TILE;
  if (threadIdx.x == 0) {
    for (int sg = 0; sg < kLtStages; ++sg) mbar_init(&bars[sg], 1);
    fence_mbar_init();
    for (int sg = 0; sg < kLtStages; ++sg) {
      const uint64_t tile = blockIdx.x + (uint64_t)sg * gridDim.x;
      if (tile < nt) {
        mbar_expect_tx(&bars[sg], TB * ns);
        for (int q = 0; q < ns; ++q)
          bulk_g2s(stage + ((uint64_t)sg * 6 + q) * TILE, src[q] + tile * TILE, TB, &bars[sg]);
      }
    }
  }
  __syncthreads();
  const bool norm = n.norm != nullptr;
  double nacc = 0.0;
  for (uint64_t j = 0;; ++j) {
    const uint64_t tile = blockIdx.x + j * gridDim.x;
    if (tile >= nt) break;
    const int sg = (int)(j % kLtStages);
    mbar_wait(&bars[sg], (uint32_t)((j / kLtStages) & 1));
    const T* base = stage + (uint64_t)sg * 6 * TILE + (uint64_t)threadIdx.x * W;
    Lanes<T, true> x[2], ax[2], dp[2], gb[2], sp[2], o[2], xi[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t off = (uint64_t)u * kBlock * W;
      auto rd = [&](int slot, Lanes<T, true>& dst) {
        Vec<T> v;
        v.u = *reinterpret_cast<const uint4*>(base + (uint64_t)slot * TILE + off);
#pragma unroll
        for (int l = 0; l < W; ++l) dst.v[l] = v.t[l];
      };
      rd(0, x[u]);
      if (PEND) rd(1, ax[u]);
      if (need_dp) rd(s_dp, dp[u]);
      if (PEND && a.agg) dp[u] = ax[u];
      if (a.quad) {
        rd(s_g, sp[u]);
        rd(s_g + 1, o[u]);
      } else {
        rd(s_g, gb[u]);
      }
      if (n.noise) {
        rd(s_nz, xi[u]);
      } else if (n.nsigma != T(0)) {
        float z[W];
        dev_normals<W>(n.nkey, n.nctr, n.nbase + tile * TILE + (uint64_t)threadIdx.x * W + off, z);
#pragma unroll
        for (int l = 0; l < W; ++l) xi[u].v[l] = rmul(n.nsigma, (T)z[l]);
      } else {
#pragma unroll
        for (int l = 0; l < W; ++l) xi[u].v[l] = T(0);
      }
    }
    __syncthreads();  // stage consumed
    if (threadIdx.x == 0) {
      const uint64_t nxt = blockIdx.x + (j + kLtStages) * gridDim.x;
      if (nxt < nt) {
        mbar_expect_tx(&bars[sg], TB * ns);
        for (int q = 0; q < ns; ++q)
          bulk_g2s(stage + ((uint64_t)sg * 6 + q) * TILE, src[q] + nxt * TILE, TB, &bars[sg]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t k = tile * TILE + (uint64_t)threadIdx.x * W + (uint64_t)u * kBlock * W;
      Lanes<T, true> ot, od;
#pragma unroll
      for (int l = 0; l < W; ++l) {
        const T x1 = PEND ? radd(x[u].v[l], ax[u].v[l]) : x[u].v[l];  // theta += avg
        ot.v[l] = x1;
        od.v[l] = sgd_delta(x1, dp[u].v[l], gb[u].v[l], sp[u].v[l], o[u].v[l], xi[u].v[l],
                            n.alpha, a.mu, a.wd, a.mu_nz, a.wd_pos, a.quad, norm, nacc);
      }
      if (PEND) st(n.theta_out, k, ot);
      st(n.aux, k, od);
      if (!(PEND && a.agg) && n.aux != n.delta) st(n.delta, k, od);
    }
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = nt * TILE + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.d;
       k += stride)
    step_group<T, MODE, false>(a, n, k, norm, nacc);
  block_add_double(nacc, n.norm);
  block_signal(a.signal);
}

template <typename T>
cudaError_t launch_ard_tma(int mode, const StepArgs<T>& a, uint32_t grid, cudaStream_t s) {
  const size_t smem = 128 + (size_t)kLtStages * 6 * lt_tile<T>() * sizeof(T);
  smem_attr(k_ard_tma<T, kModeArDelta>, smem);
  smem_attr(k_ard_tma<T, kModeApplyDelta>, smem);
  const uint64_t tiles = a.d / lt_tile<T>();
  if (tiles < grid) grid = (uint32_t)(tiles ? tiles : 1);
  if (mode == kModeApplyDelta)
    DSGD_PDL_LAUNCH((k_ard_tma<T, kModeApplyDelta>), grid, kBlock, smem, s, a);
  else
    DSGD_PDL_LAUNCH((k_ard_tma<T, kModeArDelta>), grid, kBlock, smem, s, a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_allreduce_local(const AllreduceArgs<T>& a, int vec, int norm, uint32_t grid,
                                   cudaStream_t s) {
  if (local_tma_enabled() && a.p == 1 && vec) return launch_local_tma<T>(a, s);  // norm fused too
  // the vector kernel covers d - d % W; a scalar launch finishes the tail
  if (vec) {
    if (norm)
      DSGD_COUNTED(k_allreduce_local<T, true, true><<<grid, kBlock, 0, s>>>(a));
    else
      DSGD_COUNTED(k_allreduce_local<T, true, false><<<grid, kBlock, 0, s>>>(a));
    const uint64_t W = Vec<T>::N, head = (a.d / W) * W;
    if (head != a.d) {
      AllreduceArgs<T> t = a;
      for (uint32_t i = 0; i < a.p; ++i) {
        NodeIO<T>& n = t.node[i];
        n.theta_in += head;
        n.theta_out += head;
        n.delta += head;
        if (n.grad) n.grad += head;
        if (n.noise) n.noise += head;
        n.nbase += head;
      }
      if (t.spec) t.spec += head;
      if (t.opt) t.opt += head;
      t.d = a.d - head;
      if (norm)
        DSGD_COUNTED(k_allreduce_local<T, false, true><<<1, kBlock, 0, s>>>(t));
      else
        DSGD_COUNTED(k_allreduce_local<T, false, false><<<1, kBlock, 0, s>>>(t));
    }
  } else {
    if (norm)
      DSGD_COUNTED(k_allreduce_local<T, false, true><<<grid, kBlock, 0, s>>>(a));
    else
      DSGD_COUNTED(k_allreduce_local<T, false, false><<<grid, kBlock, 0, s>>>(a));
  }
  return cudaGetLastError();
}

// -------------------------------------------------- single-context EASGD
// Synchronous sweep simulator.cpp:335-346 fused over the p clients: per
// coordinate the center is one register carried through the clients in node
// order -- u = beta*(theta_i - c); theta_i -= u; SGD step; c += u
// (protocols.cpp:148-151, 156) -- so the serial server order costs nothing.
// MIX: the client/server half only (theta_i -= u, c += u, no SGD step): the
// logistic gradient source evaluates its minibatch gradient at the moved
// theta before the step (a global dot product per row).
template <typename T, bool VEC, bool NORM, bool MIX = false>
__global__ void __launch_bounds__(kBlock) k_ea_local(const __grid_constant__ EaArgs<T> a) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  double nacc[NORM ? kMaxLocal : 1];
  if constexpr (NORM)
    for (uint32_t i = 0; i < a.p; ++i) nacc[i] = 0.0;
  const uint64_t nv = a.d / W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const uint64_t k = v * W;
    L c;
    ld(c, a.center, k);
    for (uint32_t i = 0; i < a.p; ++i) {
      const NodeIO<T>& n = a.node[i];
      L x, dp, gb, s, o, xi, ot, od, uo;
      ld(x, n.theta_in, k);
      if constexpr (MIX) {
#pragma unroll
        for (int l = 0; l < W; ++l) {
          const T u = rmul(a.beta, rsub(x.v[l], c.v[l]));
          ot.v[l] = rsub(x.v[l], u);
          uo.v[l] = u;
          c.v[l] = radd(c.v[l], u);
        }
        st(n.theta_out, k, ot);
        if (n.aux) st(n.aux, k, uo);
        continue;
      }
      ld(dp, n.delta, k);
      ld_grad_inputs(gb, s, o, xi, n, a.spec, a.opt, a.quad, k);
      double dummy = 0.0;
#pragma unroll
      for (int l = 0; l < W; ++l) {
        T xv = x.v[l];
        T u = T(0);
        if (a.gated) {
          u = rmul(a.beta, rsub(xv, c.v[l]));
          xv = rsub(xv, u);
        }
        const T dl = sgd_delta(xv, dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu, a.wd,
                               a.mu_nz, a.wd_pos, a.quad, NORM, NORM ? nacc[i] : dummy);
        od.v[l] = dl;
        ot.v[l] = radd(xv, dl);
        uo.v[l] = u;
        if (a.gated) c.v[l] = radd(c.v[l], u);
      }
      st(n.theta_out, k, ot);
      st(n.delta, k, od);
      if (n.aux) st(n.aux, k, uo);  // the client's update (ea_client_step's second result)
    }
    if (a.gated) st(a.center, k, c);
  }
  if constexpr (NORM)
    for (uint32_t i = 0; i < a.p; ++i) block_add_double(nacc[i], a.node[i].norm);
}

template <typename T>
cudaError_t launch_ea_local(const EaArgs<T>& a, int vec, int norm, uint32_t grid, cudaStream_t s,
                            bool mix_only) {
  if (mix_only) {  // gated client/server half only (the gradient comes later)
    DSGD_COUNTED(k_ea_local<T, false, false, true><<<grid, kBlock, 0, s>>>(a));
    return cudaGetLastError();
  }
  if (vec) {
    if (norm)
      DSGD_COUNTED(k_ea_local<T, true, true><<<grid, kBlock, 0, s>>>(a));
    else
      DSGD_COUNTED(k_ea_local<T, true, false><<<grid, kBlock, 0, s>>>(a));
    const uint64_t W = Vec<T>::N, head = (a.d / W) * W;
    if (head != a.d) {
      EaArgs<T> t = a;
      for (uint32_t i = 0; i < a.p; ++i) {
        NodeIO<T>& n = t.node[i];
        n.theta_in += head;
        n.theta_out += head;
        n.delta += head;
        if (n.grad) n.grad += head;
        if (n.noise) n.noise += head;
        if (n.aux) n.aux += head;
        n.nbase += head;
      }
      if (t.spec) t.spec += head;
      if (t.opt) t.opt += head;
      t.center += head;
      t.d = a.d - head;
      if (norm)
        DSGD_COUNTED(k_ea_local<T, false, true><<<1, kBlock, 0, s>>>(t));
      else
        DSGD_COUNTED(k_ea_local<T, false, false><<<1, kBlock, 0, s>>>(t));
    }
  } else {
    if (norm)
      DSGD_COUNTED(k_ea_local<T, false, true><<<grid, kBlock, 0, s>>>(a));
    else
      DSGD_COUNTED(k_ea_local<T, false, false><<<grid, kBlock, 0, s>>>(a));
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------- push gossip
// push_mix protocols.cpp:207-225 then the step: acc = 0; acc += x_k - x_i
// over senders k ascending; mixed = x_i + acc * (1/count).
template <typename T, bool VEC>
__device__ __forceinline__ void push_group(const PushArgs<T>& a, uint32_t node, uint64_t k,
                                           bool norm, double& nacc) {
  using L = Lanes<T, VEC>;
  constexpr int W = L::W;
  const NodeIO<T>& n = a.node[node];
  L x, acc, m;
  ld(x, n.theta_in, k);
  zero(acc);
  const uint32_t ns = a.n_senders[node];
  for (uint32_t j = 0; j < ns; ++j) {
    L xs;
    ld(xs, a.senders[node][j], k);
#pragma unroll
    for (int l = 0; l < W; ++l) acc.v[l] = radd(acc.v[l], rsub(xs.v[l], x.v[l]));
  }
  const T inv = a.inv[node];
#pragma unroll
  for (int l = 0; l < W; ++l) m.v[l] = radd(x.v[l], rmul(acc.v[l], inv));
  if (!a.step) {
    st(n.theta_out, k, m);
    return;
  }
  L dp, gb, s, o, xi, ot, od;
  ld(dp, n.delta, k);
  ld_grad_inputs(gb, s, o, xi, n, a.spec, a.opt, a.quad, k);
#pragma unroll
  for (int l = 0; l < W; ++l) {
    const T dl = sgd_delta(m.v[l], dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu, a.wd,
                           a.mu_nz, a.wd_pos, a.quad, norm, nacc);
    od.v[l] = dl;
    ot.v[l] = radd(m.v[l], dl);
  }
  st(n.theta_out, k, ot);
  st(n.delta, k, od);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kBlock) k_push(const __grid_constant__ PushArgs<T> a) {
  if (!block_wait(a.wait)) return;
  const uint32_t node = blockIdx.x / a.blocks_per_node;
  const uint32_t bid = blockIdx.x - node * a.blocks_per_node;
  const bool norm = a.node[node].norm != nullptr;
  double nacc = 0.0;
  constexpr int W = Lanes<T, VEC>::W;
  const uint64_t nv = a.d / W;
  const uint64_t stride = (uint64_t)a.blocks_per_node * blockDim.x;
  const uint64_t first = (uint64_t)bid * blockDim.x + threadIdx.x;
  for (uint64_t v = first; v < nv; v += stride) push_group<T, VEC>(a, node, v * W, norm, nacc);
  if constexpr (VEC) {
    for (uint64_t k = nv * W + first; k < a.d; k += stride)
      push_group<T, false>(a, node, k, norm, nacc);
  }
  block_add_double(nacc, a.node[node].norm);
  block_signal(a.signal);
}

template <typename T>
cudaError_t launch_push(const PushArgs<T>& a, int vec, uint32_t grid, cudaStream_t s) {
  if (vec)
    DSGD_COUNTED(k_push<T, true><<<grid, kBlock, 0, s>>>(a));
  else
    DSGD_COUNTED(k_push<T, false><<<grid, kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

// ------------------------------------------------------ multi-GPU EASGD chain
// Rank r of the chain, chunk by chunk: wait until the previous rank (rank 0:
// the last rank of the previous gated round) has published the running
// center of this chunk into our c_in, run the client update + step, forward
// the center to the next rank over NVLink and publish the chunk flag.  The
// per-coordinate operation order is the single-context sweep's exactly.
template <typename T, bool VEC, bool MIX = false>
__global__ void __launch_bounds__(kBlock) k_ea_chain(const __grid_constant__ EaChainArgs<T> a) {
  __shared__ int ok;
  const NodeIO<T>& n = a.node;
  const bool norm = n.norm != nullptr;
  double nacc = 0.0;
  for (uint64_t c = blockIdx.x; c < a.n_chunks; c += gridDim.x) {
    if (threadIdx.x == 0) ok = wait_flag(&a.flag_in[c], a.need, a.timeout_ns, a.error) ? 1 : 0;
    __syncthreads();
    if (!ok) return;
    for (uint64_t part = 0; part < a.chunk; part += kEaChunk) {
    const uint64_t base = c * a.chunk + part + (uint64_t)threadIdx.x * 4;
    constexpr int W = Lanes<T, VEC>::W;
    for (int sub = 0; sub < 4; sub += W) {
      const uint64_t k = base + sub;
      if (VEC ? (k + W > a.d) : (k >= a.d)) {
        if (VEC) {  // ragged tail of the last chunk: scalar
          for (uint64_t kk = k; kk < base + 4 && kk < a.d; ++kk) {
            const T cv0 = a.c_in[kk];
            T xv = n.theta_in[kk];
            const T u = rmul(a.beta, rsub(xv, cv0));
            xv = rsub(xv, u);
            if constexpr (MIX) {
              n.theta_out[kk] = xv;
              a.c_out[kk] = radd(cv0, u);
              continue;
            }
            const T gb = a.quad ? T(0) : n.grad[kk];
            const T sv = a.quad ? a.spec[kk] : T(0), ov = a.quad ? a.opt[kk] : T(0);
            const T xiv = noise_at(n, kk);
            const T dl = sgd_delta(xv, n.delta[kk], gb, sv, ov, xiv, n.alpha, a.mu, a.wd, a.mu_nz,
                                   a.wd_pos, a.quad, norm, nacc);
            n.delta[kk] = dl;
            n.theta_out[kk] = radd(xv, dl);
            a.c_out[kk] = radd(cv0, u);
          }
        }
        break;
      }
      using L = Lanes<T, VEC>;
      L cv, x, dp, gb, s, o, xi, ot, od;
      ld(cv, a.c_in, k);
      ld(x, n.theta_in, k);
      if constexpr (MIX) {
#pragma unroll
        for (int l = 0; l < W; ++l) {
          const T u = rmul(a.beta, rsub(x.v[l], cv.v[l]));
          ot.v[l] = rsub(x.v[l], u);
          cv.v[l] = radd(cv.v[l], u);
        }
        st(n.theta_out, k, ot);
        st(a.c_out, k, cv);
        continue;
      }
      ld(dp, n.delta, k);
      ld_grad_inputs(gb, s, o, xi, n, a.spec, a.opt, a.quad, k);
#pragma unroll
      for (int l = 0; l < W; ++l) {
        const T u = rmul(a.beta, rsub(x.v[l], cv.v[l]));
        const T xv = rsub(x.v[l], u);
        const T dl = sgd_delta(xv, dp.v[l], gb.v[l], s.v[l], o.v[l], xi.v[l], n.alpha, a.mu, a.wd,
                               a.mu_nz, a.wd_pos, a.quad, norm, nacc);
        od.v[l] = dl;
        ot.v[l] = radd(xv, dl);
        cv.v[l] = radd(cv.v[l], u);
      }
      st(n.theta_out, k, ot);
      st(n.delta, k, od);
      st(a.c_out, k, cv);
    }
    }
    // the barrier orders every thread's center stores before thread 0's
    // release (cumulative at system scope): no separate fence.sc
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys(&a.flag_out[c], a.seq);
  }
  block_add_double(nacc, n.norm);
  block_signal(a.signal);
}

// Staged chain (the B200 path, chunk = one st_tile): a persistent grid, CTA
// b owning chunks b, b + G, ...  Warp 8 (producer) bulk-copies each chunk's
// theta / delta / gradient (or s, opt) / host-noise tiles into a 4-stage
// shared-memory ring as soon as a stage frees -- they do not depend on the
// chain -- and the center tile once the previous rank has published it
// (flag acquire, then proxy fence).  Warps 0-7 run the client update + SGD
// step out of shared memory, store the new center straight into the next
// rank's c_in with 16-B SM stores (NVLink) and write theta' / delta' back
// into the stage; they arrive on the stage's named barrier.  Warp 9
// (signal) waits there, bulk-stores theta' / delta' to local HBM, recycles
// the stage and hands the chunk index to warp 10 (publisher), which issues
// one system fence for every chunk handed over before it and then the
// chunks' flags with relaxed system-scope stores.  Neither the NVLink write
// acknowledgement (the fence) nor the flag wait ever sits on the path that
// recycles stages (profiles/r2_ea_chain.md).  Per-coordinate operation
// order is k_ea_chain's (the single-context sweep's) exactly.
constexpr int kEcStages = 4;
constexpr int kEcThreads = kBlock + 96;  // + producer, signal, publisher warps

template <typename T>
__device__ __forceinline__ void ec_slot_rd(const T* p, T (&v)[Vec<T>::N]) {
  Vec<T> t;
  t.u = *reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int l = 0; l < Vec<T>::N; ++l) v[l] = t.t[l];
}
template <typename T>
__device__ __forceinline__ void ec_slot_wr(T* p, const T (&v)[Vec<T>::N]) {
  Vec<T> t;
#pragma unroll
  for (int l = 0; l < Vec<T>::N; ++l) t.t[l] = v[l];
  *reinterpret_cast<uint4*>(p) = t.u;
}

// U: 16-B vectors per update thread per chunk (chunk = kBlock * 16 B * U)
template <typename T, int U>
__global__ void __launch_bounds__(kEcThreads, U == 1 ? 2 : 1)
    k_ea_chain_tma(const __grid_constant__ EaChainArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint64_t TILE = (uint64_t)kBlock * Vec<T>::N * U;
  constexpr uint32_t TB = (uint32_t)(TILE * sizeof(T));
  constexpr int W = Vec<T>::N;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + kEcStages;
  uint64_t* ready = empty + kEcStages;  // chunks handed to the publisher warp
  T* stage = reinterpret_cast<T*>(smem_raw + 128);
  const NodeIO<T>& n = a.node;
  const bool hnoise = n.noise != nullptr;
  constexpr int s_c = 0, s_x = 1, s_dp = 2, s_g = 3;  // center, theta, delta, g | s, opt
  const int s_nz = a.quad ? 5 : 4;                      // host noise
  const int nsl = s_nz + (hnoise ? 1 : 0);
  const uint64_t nfull = a.d / TILE;
  const uint64_t G = gridDim.x;
  const uint64_t mine = nfull > blockIdx.x ? (nfull - 1 - blockIdx.x) / G + 1 : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL (see block_wait)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int sg = 0; sg < kEcStages; ++sg) {
      mbar_init(&full[sg], 1);
      mbar_init(&empty[sg], 1);
    }
    *ready = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kBlock / 32) {
    if (lane == 0) {  // producer
      auto issue_local = [&](uint64_t j, int sg) {
        const uint64_t off = (blockIdx.x + j * G) * TILE;
        T* dst = stage + (uint64_t)sg * nsl * TILE;
        mbar_expect_tx(&full[sg], TB * (uint32_t)nsl);  // + the center tile, issued later
        bulk_g2s(dst + s_x * TILE, n.theta_in + off, TB, &full[sg]);
        bulk_g2s(dst + s_dp * TILE, n.delta + off, TB, &full[sg]);
        if (a.quad) {
          bulk_g2s(dst + s_g * TILE, a.spec + off, TB, &full[sg]);
          bulk_g2s(dst + (s_g + 1) * TILE, a.opt + off, TB, &full[sg]);
        } else {
          bulk_g2s(dst + s_g * TILE, n.grad + off, TB, &full[sg]);
        }
        if (hnoise) bulk_g2s(dst + (uint64_t)s_nz * TILE, n.noise + off, TB, &full[sg]);
      };
      for (uint64_t j = 0; j < mine && j < (uint64_t)kEcStages; ++j) issue_local(j, (int)j);
      bool live = true;
      for (uint64_t j = 0; j < mine; ++j) {
        const int sg = (int)(j % kEcStages);
        if (j >= (uint64_t)kEcStages) {
          mbar_wait(&empty[sg], (uint32_t)((j / kEcStages - 1) & 1));
          issue_local(j, sg);
        }
        const uint64_t c = blockIdx.x + j * G;
        // after a timeout (error raised) the remaining chunks run on stale
        // centers so that every role still terminates
        if (live) live = wait_flag(&a.flag_in[c], a.need, a.timeout_ns, a.error);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // peer wrote c_in
        bulk_g2s(stage + (uint64_t)sg * nsl * TILE + s_c * TILE, a.c_in + c * TILE, TB, &full[sg]);
      }
    }
  } else if (warp == kBlock / 32 + 1) {  // signal warp
    for (uint64_t j = 0; j < mine; ++j) {
      const int sg = (int)(j % kEcStages);
      // the update warps' center stores (NVLink) and shared-memory results
      // of chunk j are performed relative to this warp past the barrier
      asm volatile("bar.sync %0, %1;" ::"r"(1 + sg), "r"(kBlock + 32) : "memory");
      if (lane == 0) {
        const uint64_t off = (blockIdx.x + j * G) * TILE;
        T* src = stage + (uint64_t)sg * nsl * TILE;
        bulk_s2g(n.theta_out + off, src + s_x * TILE, TB);
        bulk_s2g(n.delta + off, src + s_dp * TILE, TB);
        bulk_commit();
        // chunk j's center is out: hand it to the publisher warp
        asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(smem_u32(ready)),
                     "l"((unsigned long long)(j + 1))
                     : "memory");
        bulk_wait_read<0>();
        mbar_arrive(&empty[sg]);
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();  // theta' / delta' landed before the round counter
  } else if (warp == kBlock / 32 + 2) {  // publisher warp
    if (lane == 0) {
      // one system fence publishes every chunk handed over before it: the
      // fence waits for the SM's outstanding NVLink writes, so it must not
      // sit on the stage-recycling path (that is the signal warp's)
      uint64_t pub = 0;
      while (pub < mine) {
        unsigned long long got;
        asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(got) : "r"(smem_u32(ready))
                     : "memory");
        if (got == pub) {
          __nanosleep(32);
          continue;
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (; pub < got; ++pub) st_relaxed_sys(&a.flag_out[blockIdx.x + pub * G], a.seq);
      }
    }
  } else {  // warps 0-7: the update
    const bool norm = n.norm != nullptr;
    double nacc = 0.0;
    for (uint64_t j = 0; j < mine; ++j) {
      const int sg = (int)(j % kEcStages);
      const uint64_t c = blockIdx.x + j * G;
      mbar_wait(&full[sg], (uint32_t)((j / kEcStages) & 1));
      T* base = stage + (uint64_t)sg * nsl * TILE + (uint64_t)threadIdx.x * W;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t o = (uint64_t)u * kBlock * W;
        T cv[W], x[W], dp[W], gb[W], sv[W], ov[W], xi[W];
        ec_slot_rd(base + s_c * TILE + o, cv);
        ec_slot_rd(base + s_x * TILE + o, x);
        ec_slot_rd(base + s_dp * TILE + o, dp);
        if (a.quad) {
          ec_slot_rd(base + s_g * TILE + o, sv);
          ec_slot_rd(base + (s_g + 1) * TILE + o, ov);
#pragma unroll
          for (int l = 0; l < W; ++l) gb[l] = T(0);
        } else {
          ec_slot_rd(base + s_g * TILE + o, gb);
#pragma unroll
          for (int l = 0; l < W; ++l) sv[l] = ov[l] = T(0);
        }
        if (hnoise) {
          ec_slot_rd(base + (uint64_t)s_nz * TILE + o, xi);
        } else if (n.nsigma != T(0)) {
          float z[W];
          dev_normals<W>(n.nkey, n.nctr, n.nbase + c * TILE + (uint64_t)threadIdx.x * W + o, z);
#pragma unroll
          for (int l = 0; l < W; ++l) xi[l] = rmul(n.nsigma, (T)z[l]);
        } else {
#pragma unroll
          for (int l = 0; l < W; ++l) xi[l] = T(0);
        }
#pragma unroll
        for (int l = 0; l < W; ++l) {
          const T uu = rmul(a.beta, rsub(x[l], cv[l]));
          const T xv = rsub(x[l], uu);
          const T dl = sgd_delta(xv, dp[l], gb[l], sv[l], ov[l], xi[l], n.alpha, a.mu, a.wd,
                                 a.mu_nz, a.wd_pos, a.quad, norm, nacc);
          dp[l] = dl;
          x[l] = radd(xv, dl);
          cv[l] = radd(cv[l], uu);
        }
        // the running center straight into the next rank's c_in (NVLink
        // stores from the SM: the TMA engine stays free for the HBM stages)
        ec_slot_wr(a.c_out + c * TILE + (uint64_t)threadIdx.x * W + o, cv);
        ec_slot_wr(base + s_x * TILE + o, x);
        ec_slot_wr(base + s_dp * TILE + o, dp);
      }
      fence_async_smem();  // theta' / delta' are read next by the signal warp's bulk stores
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + sg), "r"(kBlock + 32) : "memory");
    }
    if (norm) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
      if (lane == 0) atomicAdd(n.norm, nacc);
    }
  }
  __syncthreads();
  // the ragged last chunk [nfull * TILE, d): its owner, with plain loads
  if (nfull * TILE < a.d && blockIdx.x == nfull % G) {
    __shared__ int ok;
    if (threadIdx.x == 0) ok = wait_flag(&a.flag_in[nfull], a.need, a.timeout_ns, a.error) ? 1 : 0;
    __syncthreads();
    if (!ok) return;
    const bool norm = n.norm != nullptr;
    double nacc = 0.0;
    for (uint64_t kk = nfull * TILE + threadIdx.x; kk < a.d; kk += blockDim.x) {
      const T cv0 = a.c_in[kk];
      T xv = n.theta_in[kk];
      const T u = rmul(a.beta, rsub(xv, cv0));
      xv = rsub(xv, u);
      const T gb = a.quad ? T(0) : n.grad[kk];
      const T sv = a.quad ? a.spec[kk] : T(0), ov = a.quad ? a.opt[kk] : T(0);
      const T dl = sgd_delta(xv, n.delta[kk], gb, sv, ov, noise_at(n, kk), n.alpha, a.mu, a.wd,
                             a.mu_nz, a.wd_pos, a.quad, norm, nacc);
      n.delta[kk] = dl;
      n.theta_out[kk] = radd(xv, dl);
      a.c_out[kk] = radd(cv0, u);
    }
    if (norm) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
      if (lane == 0) atomicAdd(n.norm, nacc);
    }
    __syncthreads();  // every thread's center stores before the (cumulative) release
    if (threadIdx.x == 0) st_release_sys(&a.flag_out[nfull], a.seq);
  }
  block_signal(a.signal);
}

// vectors per update thread per chunk: DSGD_EA_TILE_U = 1 (fp32 only: 1024
// elements per chunk, two CTAs per SM) or 2 (default: 2048 fp32 / 1024 fp64)
template <typename T>
int ea_chain_u() {
  static const int u = [] {
    const char* e = getenv("DSGD_EA_TILE_U");
    return (e && atoi(e) == 1 && sizeof(T) == 4) ? 1 : 2;
  }();
  return u;
}

template <typename T>
uint64_t ea_chain_tile() {
  return (uint64_t)kBlock * Vec<T>::N * ea_chain_u<T>();
}

template <typename T, int U>
cudaError_t launch_ea_chain_tma(const EaChainArgs<T>& a, cudaStream_t s) {
  constexpr uint64_t TILE = (uint64_t)kBlock * Vec<T>::N * U;
  const bool hnoise = a.node.noise != nullptr;
  const int nsl = (a.quad ? 5 : 4) + (hnoise ? 1 : 0);
  const size_t smem = 128 + (size_t)kEcStages * nsl * TILE * sizeof(T);
  smem_attr(k_ea_chain_tma<T, U>, smem);
  int dev = 0, sms = 148, resident = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_ea_chain_tma<T, U>, kEcThreads, smem);
  if (resident < 1) resident = 1;
  const uint64_t nfull = a.d / TILE;
  const uint32_t g = (uint32_t)std::min<uint64_t>(nfull, (uint64_t)sms * resident);
  DSGD_PDL_LAUNCH((k_ea_chain_tma<T, U>), g, kEcThreads, smem, s, a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_ea_chain(const EaChainArgs<T>& a, int vec, uint32_t grid, cudaStream_t s,
                            bool mix_only) {
  if (mix_only) {
    if (vec)
      DSGD_COUNTED(k_ea_chain<T, true, true><<<grid, kBlock, 0, s>>>(a));
    else
      DSGD_COUNTED(k_ea_chain<T, false, true><<<grid, kBlock, 0, s>>>(a));
    return cudaGetLastError();
  }
  if (vec && a.chunk == ea_chain_tile<T>() && a.d >= a.chunk && ea_chain_staged())
    return ea_chain_u<T>() == 1 ? launch_ea_chain_tma<T, 1>(a, s) : launch_ea_chain_tma<T, 2>(a, s);
  if (vec)
    DSGD_COUNTED(k_ea_chain<T, true><<<grid, kBlock, 0, s>>>(a));
  else
    DSGD_COUNTED(k_ea_chain<T, false><<<grid, kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

// ------------------------------------------------- logistic gradient source
// LogisticObjective::stochastic_gradient objectives.cpp:147-162 in three
// launches.  (1) per (node, row) and per slice of d: partial dot products
// z = sum_k x_k * la_k in fp64 (products of two context-dtype values are
// exact in fp64); (2) per (node, row): the slices summed in a fixed order
// (deterministic run to run; the reference sums k sequentially, so fp64 z
// agrees to rounding, not bitwise), coeff = sigmoid(z) - y (34-38, 131);
// (3) elementwise in the reference order: g = 0; g += coeff_b * x_b over b
// (132-133, 155); g *= 1/batch (158); g += l2 * la (159).
template <typename T>
__device__ __forceinline__ T logistic_point(const LogisticArgs<T>& a, uint32_t n, uint64_t k) {
  const T x = a.theta[n][k];
  return a.lookahead ? radd(x, rmul(a.mu, a.delta[n][k])) : x;
}

__device__ __forceinline__ double block_sum_fixed(double v) {
  __shared__ double red[kBlock / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;  // valid in thread 0
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_logit_partial(const __grid_constant__ LogisticArgs<T> a) {
  const uint32_t nr = a.n_nodes * a.batch;
  const uint64_t span = (a.d + a.nblk - 1) / a.nblk;
  const uint64_t lo = (uint64_t)blockIdx.x * span;
  const uint64_t hi = lo + span < a.d ? lo + span : a.d;
  for (uint32_t r = blockIdx.y; r < nr; r += gridDim.y) {  // r = node * batch + b
    const uint32_t n = r / a.batch;
    const T* x = a.X + a.rows[r] * a.d;
    double acc = 0.0;
    for (uint64_t k = lo + threadIdx.x; k < hi; k += blockDim.x)
      acc += (double)x[k] * (double)logistic_point(a, n, k);
    const double s = block_sum_fixed(acc);
    if (threadIdx.x == 0) a.partial[(uint64_t)r * a.nblk + blockIdx.x] = s;
    __syncthreads();  // block_sum_fixed's smem is reused by the next row
  }
}

__device__ __forceinline__ double sigmoid_ref(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

template <typename T>
__global__ void __launch_bounds__(32) k_logit_coeff(const __grid_constant__ LogisticArgs<T> a) {
  const uint32_t r = blockIdx.x;
  double v = 0.0;
  for (uint32_t b = threadIdx.x; b < a.nblk; b += 32) v += a.partial[(uint64_t)r * a.nblk + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) {
    const double y = (double)a.y[a.rows[r]];
    if (a.value_mode)  // log1pexp objectives.cpp:29-32, value 116-125
      a.coeff[r] = (v > 0.0 ? v + log1p(exp(-v)) : log1p(exp(v))) - y * v;
    else
      a.coeff[r] = sigmoid_ref(v) - y;
  }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_logistic_grad(const __grid_constant__ LogisticArgs<T> a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.d; k += stride) {
    for (uint32_t n = 0; n < a.n_nodes; ++n) {
      T g = T(0);
      for (uint32_t b = 0; b < a.batch; ++b) {
        const uint32_t r = n * a.batch + b;
        g = radd(g, rmul((T)a.coeff[r], a.X[a.rows[r] * a.d + k]));
      }
      g = rmul(g, a.inv_batch);
      a.out[n][k] = radd(g, rmul(a.l2, logistic_point(a, n, k)));
    }
  }
}

template <typename T>
cudaError_t launch_logistic(const LogisticArgs<T>& a, uint32_t grid, cudaStream_t s) {
  const uint32_t nr = a.n_nodes * a.batch;
  DSGD_COUNTED(k_logit_partial<T><<<dim3(a.nblk, nr < 65535u ? nr : 65535u), kBlock, 0, s>>>(a));
  DSGD_COUNTED(k_logit_coeff<T><<<nr, 32, 0, s>>>(a));
  if (!a.value_mode) DSGD_COUNTED(k_logistic_grad<T><<<grid, kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

// ------------------------------------------------------------ trace metrics
// make_trace_record simulator.cpp:92-123 over p node vectors (local or NVLink
// peer pointers): pivot-form mean (param_vec.cpp:26-38), consensus error,
// objective value and optimum error, accumulated in fp64.
template <typename T>
__global__ void __launch_bounds__(kBlock) k_trace(const __grid_constant__ TraceArgs<T> a) {
  if (!block_wait(a.wait)) return;
  double cons = 0.0, loss = 0.0, err = 0.0, bad = 0.0;
  const double inv_p = 1.0 / (double)a.p;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.d;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const double x0 = (double)a.x[0][k];
    double dev = 0.0;
    for (uint32_t i = 1; i < a.p; ++i) dev += (double)a.x[i][k] - x0;
    const double mean = x0 + dev * inv_p;
    const double o = a.opt ? (double)a.opt[k] : 0.0;
    const double sp = a.spec ? (double)a.spec[k] : 0.0;
    for (uint32_t i = 0; i < a.p; ++i) {
      const double xi = (double)a.x[i][k];
      if (!isfinite(xi)) bad += 1.0;
      const double c = xi - mean;
      cons += c * c;
      const double b = xi - o;
      err += b * b;
      loss += sp * b * b;
    }
  }
  block_add_double(cons, a.out + 0);
  block_add_double(loss, a.out + 1);
  block_add_double(err, a.out + 2);
  block_add_double(bad, a.out + 3);
}

template <typename T>
cudaError_t launch_trace(const TraceArgs<T>& a, uint32_t grid, cudaStream_t s) {
  DSGD_COUNTED(k_trace<T><<<grid, kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

// ------------------------------------------------------------ spatial mean
// param_vec.cpp:19-40 over p device vectors (EASGD center init).
template <typename T>
struct MeanArgs {
  const T* x[kMaxLocal];
  uint32_t p;
  uint64_t d;
  T inv_p;
  T* out;
};

template <typename T>
__global__ void __launch_bounds__(kBlock) k_spatial_mean(const __grid_constant__ MeanArgs<T> a) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.d;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const T x0 = a.x[0][k];
    T dev = T(0);
    for (uint32_t i = 1; i < a.p; ++i) dev = radd(dev, rsub(a.x[i][k], x0));
    a.out[k] = radd(x0, rmul(dev, a.inv_p));
  }
}

template <typename T>
cudaError_t launch_spatial_mean(const T* const* x, uint32_t p, uint64_t d, T* out, cudaStream_t s) {
  if (p == 0 || p > (uint32_t)kMaxLocal) return cudaErrorInvalidValue;
  MeanArgs<T> a{};
  for (uint32_t i = 0; i < p; ++i) a.x[i] = x[i];
  a.p = p;
  a.d = d;
  a.inv_p = T(1) / T(p);
  a.out = out;
  const uint64_t blocks = (d + kBlock - 1) / kBlock;
  DSGD_COUNTED(k_spatial_mean<T><<<(unsigned)(blocks < 4096 ? (blocks ? blocks : 1) : 4096), kBlock, 0, s>>>(a));
  return cudaGetLastError();
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_fill_normal(T* out, uint64_t n, double sigma,
                                                        uint64_t seed, uint64_t offset) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ctr = q + offset;
    const uint4 r = philox(make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), 0x6a09e667u, 0xbb67ae85u), key);
    const float u0 = ((r.x >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u1 = ((r.y >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = ((r.z >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u3 = ((r.w >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float r0 = sqrtf(-2.0f * __logf(u0)), r1 = sqrtf(-2.0f * __logf(u2));
    float s0, c0, s1, c1;
    __sincosf(6.2831853071795864f * u1, &s0, &c0);
    __sincosf(6.2831853071795864f * u3, &s1, &c1);
    const float z[4] = {r0 * c0, r0 * s0, r1 * c1, r1 * s1};
#pragma unroll
    for (int l = 0; l < 4; ++l)
      if (q * 4 + l < n) out[q * 4 + l] = (T)(sigma * (double)z[l]);
  }
}

template <typename T>
cudaError_t launch_fill_normal(T* out, uint64_t n, double sigma, uint64_t seed, uint64_t offset,
                               cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t need = (n / 4 + kBlock) / kBlock;
  const uint64_t grid = need < (uint64_t)sms * 8 ? (need ? need : 1) : (uint64_t)sms * 8;
  DSGD_COUNTED(k_fill_normal<T><<<(unsigned)grid, kBlock, 0, s>>>(out, n, sigma, seed, offset));
  return cudaGetLastError();
}

#if !defined(DSGD_KERNEL_DTYPE) || DSGD_KERNEL_DTYPE == 32
__global__ void __launch_bounds__(kBlock) k_norm_fold(double* acc, uint64_t n, double* max) {
  double m = 0.0;
  for (uint64_t k = threadIdx.x; k < n; k += blockDim.x) {
    m = fmax(m, sqrt(acc[k]));  // ParamVec::norm = sqrt(squared_norm)
    acc[k] = 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double part[kBlock / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, part[w]);
    *max = fmax(*max, m);
  }
}

__global__ void k_wait_chunks(const unsigned long long* flags, uint64_t n, unsigned long long need,
                              unsigned long long timeout_ns, unsigned int* error) {
  for (uint64_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (!wait_flag(&flags[c], need, timeout_ns, error)) return;
}

cudaError_t launch_wait_chunks(const unsigned long long* flags, uint64_t n, unsigned long long need,
                               unsigned long long timeout_ns, unsigned int* error, cudaStream_t s) {
  const uint32_t g = (uint32_t)std::min<uint64_t>((n + kBlock - 1) / kBlock, 1024);
  DSGD_COUNTED(k_wait_chunks<<<g ? g : 1, kBlock, 0, s>>>(flags, n, need, timeout_ns, error));
  return cudaGetLastError();
}

bool ea_chain_staged() {
  static const bool on = [] {  // DSGD_EA_STAGED=0: the one-CTA-per-chunk LDG chain
    const char* e = getenv("DSGD_EA_STAGED");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool local_tma_enabled() {
  static const bool tma = [] {  // DSGD_LOCAL_TMA=0 selects the LDG kernel
    const char* e = getenv("DSGD_LOCAL_TMA");
    return !(e && e[0] == '0');
  }();
  return tma;
}

cudaError_t launch_norm_fold(double* acc, uint64_t n, double* max, cudaStream_t s) {
  DSGD_COUNTED(k_norm_fold<<<1, kBlock, 0, s>>>(acc, n, max));
  return cudaGetLastError();
}
#endif

#define DSGD_INSTANTIATE(T)                                                                        \
  template cudaError_t launch_step<T>(int, const StepArgs<T>&, int, uint32_t, cudaStream_t);       \
  template cudaError_t launch_allreduce_local<T>(const AllreduceArgs<T>&, int, int, uint32_t,      \
                                                 cudaStream_t);                                    \
  template cudaError_t launch_ea_local<T>(const EaArgs<T>&, int, int, uint32_t, cudaStream_t,      \
                                          bool);                                                   \
  template cudaError_t launch_logistic<T>(const LogisticArgs<T>&, uint32_t, cudaStream_t);         \
  template cudaError_t launch_push<T>(const PushArgs<T>&, int, uint32_t, cudaStream_t);            \
  template uint64_t ea_chain_tile<T>();                                                           \
  template cudaError_t launch_ea_chain<T>(const EaChainArgs<T>&, int, uint32_t, cudaStream_t,      \
                                          bool);                                                   \
  template cudaError_t launch_ar_reduce<T>(const ArReduceArgs<T>&, uint32_t, cudaStream_t);        \
  template cudaError_t launch_trace<T>(const TraceArgs<T>&, uint32_t, cudaStream_t);               \
  template cudaError_t launch_ar_oneshot<T>(const ArOneShotArgs<T>&, int, uint32_t, cudaStream_t); \
  template cudaError_t launch_ar_nvls<T>(const ArNvlsArgs<T>&, uint32_t, cudaStream_t);            \
  template cudaError_t launch_ard_tma<T>(int, const StepArgs<T>&, uint32_t, cudaStream_t);         \
  template cudaError_t launch_spatial_mean<T>(const T* const*, uint32_t, uint64_t, T*,             \
                                              cudaStream_t);                                       \
  template cudaError_t launch_fill_normal<T>(T*, uint64_t, double, uint64_t, uint64_t, cudaStream_t);

#if !defined(DSGD_KERNEL_DTYPE) || DSGD_KERNEL_DTYPE == 32
DSGD_INSTANTIATE(float)
#endif
#if !defined(DSGD_KERNEL_DTYPE) || DSGD_KERNEL_DTYPE == 64
DSGD_INSTANTIATE(double)
#endif

}  // namespace dsgd
