// dsgd_kernels.cuh -- launch-parameter structs shared by the runtime
// (dsgd_runtime.cu) and the kernels (dsgd_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dsgd_device.cuh"

namespace dsgd {

// One node's device buffers for one launch.
template <typename T>
struct NodeIO {
  const T* theta_in;   // theta at the start of the round (snapshot buffer)
  T* theta_out;        // theta after the round (the other ping-pong buffer)
  T* delta;            // delta_prev, read then overwritten in place
  const T* grad;       // minibatch gradient at the lookahead (GRAD_BUFFER)
  const T* noise;      // additive noise draw, or null (zero noise: adds +0)
  const T* partner;    // partner's snapshot theta (local or NVLink peer)
  T* aux;              // all-reduce exchange buffer
  double* norm;        // sum of g^2 accumulator (grad_norm_out), or null
  T alpha;             // step_size_at(h, t_i)
  T nsigma;            // device Philox noise sigma (used when noise == null), 0: none
  uint64_t nkey;       // device noise key (seed, node)
  uint64_t nctr;       // device noise counter (the node's t)
  uint64_t nbase;      // element offset of this launch's k = 0 (tail launches)
};

// Trace metrics over all p nodes (make_trace_record simulator.cpp:92-123).
template <typename T>
struct TraceArgs {
  const T* x[kMaxLocal];
  const T* spec;  // null: no loss / optimum error
  const T* opt;
  uint32_t p;
  uint64_t d;
  double* out;    // [0] sq_err_consensus, [1] sum_i 2 f(theta_i), [2] sq_err_opt, [3] non-finite count
  WaitSpec wait;  // one node per GPU: every peer finished its last round
};

// Kernel modes of the fused gossip-family kernel k_step.
enum StepMode : int {
  kModeStep = 0,     // local_sgd_step                      protocols.cpp:102-108
  kModePull = 1,     // mix_toward(x_i, x_j, 1/2) then step  protocols.cpp:161-185
  kModeStale = 2,    // delta at x_i; mix(x_i,x_j,b) + delta protocols.cpp:252-263
  kModeMix = 3,      // mix only (pull_mix / gossip_fresh_mix)
  kModeArDelta = 4,  // compute_local_delta -> aux            protocols.cpp:85-100
  kModeApply = 5,    // theta += aux (averaged delta)        protocols.cpp:125-129
  kModeAsync = 6,    // async_pull_event                      protocols.cpp:278-297
  kModeApplyDelta = 7,  // previous round's theta += avg fused with this round's delta
  kModeLookahead = 8    // out = theta + mu * delta_prev (compute_local_delta's evaluation point)
};

template <typename T>
struct StepArgs {
  NodeIO<T> node[kMaxLocal];
  const T* spec;  // quadratic spectrum (GRAD_QUADRATIC)
  const T* opt;   // quadratic optimum
  uint64_t d;
  T mu, wd, beta;
  int mu_nz;   // h.mu != 0  (lookahead taken)       protocols.cpp:90
  int wd_pos;  // h.weight_decay > 0                 protocols.cpp:31
  int quad;    // gradient = spec * (la - opt)
  uint32_t n_local;
  uint32_t blocks_per_node;
  int agg;  // kModeApplyDelta: aggregate momentum scope (delta_prev = the average)
  int tma_partner;  // stage the (peer-GPU) partner snapshot via bulk async copies
  WaitSpec wait;
  SignalSpec signal;
};

// Multi-GPU all-reduce over NVLink peer memory (replaces ring_allreduce,
// transport.cpp:183-248): this rank owns reference ring chunk `slice`
// [lo, hi); it reads every rank's exchange buffer x[k] for that range, folds
// the sum left in ring order starting at node `slice` ("received + own",
// transport.cpp:224-226), divides by p (229-235) and writes the average into
// every rank's avg buffer (the all-gather, 238-246).
template <typename T>
struct ArReduceArgs {
  const T* x[kMaxWait];
  T* avg[kMaxWait];
  uint32_t p;
  uint32_t slice;
  uint64_t lo, hi;
  WaitSpec wait;
  SignalSpec signal;
};

constexpr int kMaxFusedRanks = 8;  // peer-memory all-reduce kernels: p <= 8

// NVLS reduce + broadcast of this rank's slice [lo, hi) (the second kernel of
// the two-shot all-reduce round): multimem.ld_reduce on the multicast
// address of the exchange buffers returns the sum over every GPU, reduced in
// the NVSwitch; the average is written to every GPU's avg buffer with one
// multimem.st.  (Summation order is the switch's: tolerance parity, like
// NCCL.)
template <typename T>
struct ArNvlsArgs {
  const T* x_mc;
  T* avg_mc;
  uint64_t lo, hi;
  uint32_t p;
  WaitSpec wait;
  SignalSpec signal;
};

// One-shot multi-GPU all-reduce round (small p): every rank reads every
// peer's exchange buffer of the previous round directly over NVLink, folds
// the average in the reference ring order and applies it fused with this
// round's delta; exchange buffers are double-buffered by round parity.
template <typename T>
struct ArOneShotArgs {
  NodeIO<T> node;                      // theta/delta/grad/noise of this rank
  const T* x_prev[kMaxFusedRanks];     // every rank's x[(t-1) % 2]
  T* x_out;                            // own x[t % 2]
  const T* spec;
  const T* opt;
  uint64_t d;
  uint32_t p;
  uint64_t ring_base, ring_rem;
  T mu, wd;
  int mu_nz, wd_pos, quad, agg, pending, apply_only;
  int tma_rank;                        // >= 0: stage peers through smem (this rank's id)
  WaitSpec wait;
  SignalSpec signal;
};

// Single-context all-reduce round (p nodes on one GPU), fused:
// deltas -> pivot-form spatial mean -> apply.
template <typename T>
struct AllreduceArgs {
  NodeIO<T> node[kMaxLocal];
  const T* spec;
  const T* opt;
  uint64_t d;
  T mu, wd, inv_p;
  int mu_nz, wd_pos, quad;
  int per_node;
  uint32_t p;
  // k_local_tma round-to-round chaining (dsgd_run_rounds, p = 1): CTA b
  // publishes cta_flags[b] = cta_seq when its tiles are written; with
  // cta_chain set, CTA b of the next round waits for exactly that flag
  // (its tiles are the same) instead of the whole previous grid
  unsigned long long* cta_flags;
  unsigned long long cta_seq;
  int cta_chain;
  unsigned int* error;
  unsigned long long timeout_ns;
};

// Single-context EASGD sweep over p nodes in node order.
template <typename T>
struct EaArgs {
  NodeIO<T> node[kMaxLocal];
  const T* spec;
  const T* opt;
  T* center;
  uint64_t d;
  T mu, wd, beta;
  int mu_nz, wd_pos, quad;
  int gated;
  uint32_t p;
};

// Push mix + step: node i averages its own snapshot with every sender's.
template <typename T>
struct PushArgs {
  NodeIO<T> node[kMaxLocal];
  const T* senders[kMaxLocal][kMaxLocal];  // ascending sender order (protocols.cpp:212)
  uint32_t n_senders[kMaxLocal];
  T inv[kMaxLocal];  // 1 / (1 + n_senders)
  const T* spec;
  const T* opt;
  uint64_t d;
  T mu, wd;
  int mu_nz, wd_pos, quad;
  int step;  // 0: push_mix only
  uint32_t n_local;
  uint32_t blocks_per_node;
  WaitSpec wait;
  SignalSpec signal;
};

// Multi-GPU EASGD chain: this rank consumes the running center chunk by
// chunk from its c_in (written by the previous rank over NVLink), applies
// its client update + SGD step, and forwards the center to the next rank.
constexpr uint64_t kEaChunk = 1024;  // elements per chunk (kBlock * 4)

// LogisticObjective::stochastic_gradient (objectives.cpp:147-162) for a set
// of local nodes: node n's minibatch rows are rows[n * batch + b]; its
// evaluation point is theta[n] (+ mu * delta[n] when lookahead).
template <typename T>
struct LogisticArgs {
  const T* X;                 // n_samples x d, row-major
  const int32_t* y;           // labels 0/1
  const T* theta[kMaxLocal];
  const T* delta[kMaxLocal];
  T* out[kMaxLocal];          // the node's gradient buffer
  const uint64_t* rows;       // device, n_nodes * batch
  double* partial;            // n_nodes * batch * nblk partial dot products
  double* coeff;              // n_nodes * batch: sigmoid(z) - y
  uint64_t d;
  uint32_t n_nodes, batch, nblk;
  T mu, l2, inv_batch;
  int lookahead;
  int value_mode;             // coeff[r] = log1pexp(z) - y z (LogisticObjective::value terms)
};

template <typename T>
struct EaChainArgs {
  NodeIO<T> node;
  const T* spec;
  const T* opt;
  const T* c_in;                         // own memory
  T* c_out;                              // next rank's c_in (peer) -- rank p-1: rank 0's
  const unsigned long long* flag_in;     // own chunk flags
  unsigned long long* flag_out;          // next rank's chunk flags (peer)
  unsigned long long need;               // wait flag_in[c] >= need
  unsigned long long seq;                // value published to flag_out[c]
  uint64_t d;
  uint64_t n_chunks;
  uint64_t chunk;  // elements per flag (multiple of kEaChunk)
  T mu, wd, beta;
  int mu_nz, wd_pos, quad;
  unsigned long long timeout_ns;
  unsigned int* error;
  SignalSpec signal;  // publishes this rank's round counter when every chunk is done
};

// Kernels launched by the calling thread so far (every launch, tails included).
uint64_t launches_issued();

// Host-side launchers (explicitly instantiated for float and double).
template <typename T>
cudaError_t launch_step(int mode, const StepArgs<T>& a, int vec, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_allreduce_local(const AllreduceArgs<T>& a, int vec, int norm, uint32_t grid,
                                   cudaStream_t s);
template <typename T>
cudaError_t launch_ea_local(const EaArgs<T>& a, int vec, int norm, uint32_t grid, cudaStream_t s,
                            bool mix_only = false);
template <typename T>
cudaError_t launch_logistic(const LogisticArgs<T>& a, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_push(const PushArgs<T>& a, int vec, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_ea_chain(const EaChainArgs<T>& a, int vec, uint32_t grid, cudaStream_t s,
                            bool mix_only = false);
template <typename T>
cudaError_t launch_ar_reduce(const ArReduceArgs<T>& a, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_ar_nvls(const ArNvlsArgs<T>& a, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_ard_tma(int mode, const StepArgs<T>& a, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_ar_oneshot(const ArOneShotArgs<T>& a, int vec, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_trace(const TraceArgs<T>& a, uint32_t grid, cudaStream_t s);
template <typename T>
cudaError_t launch_spatial_mean(const T* const* x, uint32_t p, uint64_t d, T* out, cudaStream_t s);
// max over `n` per-round sums of g^2 of sqrt(sum) into *max, zeroing the sums
// true when the p = 1 fused round runs the staged k_local_tma (DSGD_LOCAL_TMA)
bool local_tma_enabled();
// true unless DSGD_EA_STAGED=0: the multi-GPU EASGD chain runs k_ea_chain_tma
// with one flag per ea_chain_tile<T>() elements (every rank the same)
bool ea_chain_staged();
// waits (bounded; error flag on timeout) until flags[0..n) >= need
cudaError_t launch_wait_chunks(const unsigned long long* flags, uint64_t n, unsigned long long need,
                               unsigned long long timeout_ns, unsigned int* error, cudaStream_t s);
template <typename T>
uint64_t ea_chain_tile();
cudaError_t launch_norm_fold(double* acc, uint64_t n, double* max, cudaStream_t s);
template <typename T>
cudaError_t launch_fill_normal(T* out, uint64_t n, double sigma, uint64_t seed, uint64_t offset,
                               cudaStream_t s);

}  // namespace dsgd
