// dsgd_runtime.cu -- the C ABI (include/dsgd_b200.h): device contexts, node
// state, the protocol rounds, multi-GPU wiring (CUDA IPC peer memory over
// NVLink + NCCL) and the per-step worker loop.
//
// Layout in HBM (per context, SoA, dtype T, d elements per vector):
//   arena (one cudaMalloc, exported through CUDA IPC):
//     theta[i][0], theta[i][1]   ping-pong parameters of each local node
//     c_in                       EASGD running center (node 0's = the server center)
//     chunk_flags[d / 1024]      EASGD per-chunk "center arrived" counters
//     round[i]                   per-node completed-round counters (u64)
//   private allocations: delta[i], grad[i], noise[i], aux[i] (all-reduce
//   exchange buffer, per-node scope only), spec/opt (quadratic objective),
//   norm accumulators, arrival counter, error flag.
// Every round reads theta[cur] and writes theta[cur ^ 1]; a remote partner
// therefore always reads a snapshot nobody is writing (the reference's
// pull/push/stale snapshot semantics, protocols.cpp:164-166).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "dsgd_b200.h"
#include "dsgd_internal.h"
#include "dsgd_kernels.cuh"
#include "dsgd_multicast.h"

#include <unistd.h>

namespace dsgd {

thread_local std::string g_error;

dsgd_status set_error(dsgd_status st, const std::string& msg) {
  g_error = msg;
  return st;
}

}  // namespace dsgd

using dsgd::kMaxLocal;
using dsgd::kMaxWait;
using dsgd::set_error;

#define DSGD_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_error(DSGD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define DSGD_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return set_error(DSGD_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));   \
  } while (0)

#define DSGD_TRY(call)                    \
  do {                                    \
    dsgd_status s_ = (call);              \
    if (s_ != DSGD_OK) return s_;         \
  } while (0)

namespace {

constexpr uint32_t kMagic = 0xD56DB200u;
constexpr uint64_t kBlockU = dsgd::kBlock;

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// What a peer needs to address this context's shared arena.
struct HandleBlob {
  uint32_t magic;
  uint32_t abi;
  uint32_t first_node;
  uint32_t n_local;
  uint32_t dtype;
  uint32_t flags;
  uint64_t d;
  int32_t device;
  int32_t pad;
  cudaIpcMemHandle_t handle;
  uint64_t arena_bytes;
  uint64_t off_theta[2];
  uint64_t off_c_in;
  uint64_t off_flags;
  uint64_t off_round;
  uint64_t off_x;    // all-reduce exchange buffer (0: none)
  uint64_t off_a;    // all-reduce average buffer
  uint64_t off_ar;   // all-reduce counters: [0] exchange written, [1] average written
  uint64_t off_arf;  // reserved
  uint64_t off_x2;   // second exchange buffer (one-shot all-reduce, round parity)
  uint64_t off_hb;   // host-barrier slots (rank 0's are the ones used)
  // NVLS: rank 0's multicast object, shared as a POSIX fd fetched with
  // pidfd_getfd(pid, fd) (mc_kind 0: none, everybody uses the peer-memory
  // two-shot)
  uint32_t mc_kind;
  int32_t mc_pid;
  int32_t mc_fd;
  int32_t pad2;
  uint64_t mc_size;
};
static_assert(sizeof(HandleBlob) <= DSGD_HANDLE_BYTES, "handle blob too large");

struct PeerNode {  // device-addressable view of one node (local or IPC-mapped)
  char* theta[2] = {nullptr, nullptr};
  char* c_in = nullptr;
  unsigned long long* flags = nullptr;
  unsigned long long* round = nullptr;
  char* x = nullptr;                  // all-reduce exchange buffer
  char* x2 = nullptr;                 // second exchange buffer (one-shot, odd rounds)
  char* avg = nullptr;                // all-reduce average buffer
  unsigned long long* ar = nullptr;   // [0] exchange written, [1] average written (rounds)
  unsigned long long* hb = nullptr;   // host-barrier slots (connect-time agreement)
};

struct Prof {
  int id;
  cudaEvent_t a, b;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// One-node contexts of one process wired to each other by raw device
// pointers (dsgd_group_create_inproc): the ranks' launches are issued in host
// order (rank 0..p-1 per round, two-shot reduces after every rank's
// exchange), so every cross-rank wait is already satisfied when a kernel
// starts.  Ranks on one GPU share one stream, which makes the multi-GPU
// kernels executable -- and checkable -- on a single GPU.
struct InprocGroup {
  std::vector<dsgd_ctx*> ctx;                         // node order
  std::vector<std::pair<int, cudaStream_t>> streams;  // one per device, owned
  ~InprocGroup() {
    for (auto& s : streams) {
      DeviceGuard g(s.first);
      cudaStreamSynchronize(s.second);
      cudaStreamDestroy(s.second);
    }
  }
};

}  // namespace

struct dsgd_ctx {
  int device = 0;
  uint64_t d = 0;
  dsgd_dtype dtype = DSGD_F32;
  size_t es = 4;
  uint32_t p = 1, first = 0, n_local = 1, flags = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 148;
  int blocks_per_sm = 4;

  char* arena = nullptr;
  size_t arena_bytes = 0;
  size_t off_theta[kMaxLocal][2] = {};
  size_t off_c_in = 0, off_flags = 0, off_round = 0, off_x = 0, off_a = 0, off_ar = 0;
  bool p2p_allreduce = true;       // multi-GPU all-reduce over NVLink peer memory (else NCCL)
  bool ar_oneshot = false;         // ... one-shot: read every peer's exchange buffer (p <= 4)
  bool ar_tma = true;              // ... staging the peer reads through smem (bulk async copies)
  bool ar_nvls = false;            // ... two-shot with the reduce/broadcast in the NVSwitch
  uint32_t ar_pipes = 2;           // two-shot: independent pipelines (streams) over d
  bool ar_pipes_env = false;       // DSGD_AR_PIPES given (no size-based choice)
  double ar_delta_frac = 2.0;      // delta-kernel CTAs per SM, split over the pipelines
  double ar_comm_frac = 2.0;       // reduce-kernel CTAs per SM, split over the pipelines
  cudaStream_t pipe_stream[4] = {};
  cudaEvent_t pipe_event[9] = {};  // [0..3] join, [4] fork, [5..8] delta kernels done
  bool pipes_forked = false;
  // DSGD_TRACE: per launch {kind, round, %globaltimer entry / after wait / done}
  unsigned long long* trace_dev = nullptr;
  uint32_t trace_cap = 0, trace_n = 0;
  std::vector<uint32_t> trace_kind;
  std::vector<uint64_t> trace_round;
  uint32_t ar_pipes_used = 1;      // pipelines of the pending rounds (counters in use)
  char* nvls_x_mc = nullptr;
  char* nvls_avg_mc = nullptr;
  size_t off_x2 = 0;
  size_t off_hb = 0;
  std::string ar_mode;             // requested backend (DSGD_ALLREDUCE or the default)
  dsgd::McState mc;                // NVLS multicast buffers owned by the library
  std::string nvls_note;           // why NVLS is not in use (empty when it is)

  uint64_t ar_rounds = 0;          // peer-memory all-reduce rounds run
  uint64_t n_chunks = 0;
  uint64_t ea_chunk = 4 * dsgd::kEaChunk;  // elements per EASGD chain flag (DSGD_EA_CHUNK)

  char* delta[kMaxLocal] = {};
  char* grad[kMaxLocal] = {};
  char* noise[kMaxLocal] = {};
  char* aux[kMaxLocal] = {};
  char* spec = nullptr;
  char* opt = nullptr;
  // grad_norm_out (protocols.cpp:34-36) on the device: each round (or
  // event) accumulates every local node's sum of g^2 into its own slot of a
  // ring; a fold kernel turns the used slots into max ||g|| (norm_max) every
  // kNormSlots rounds and whenever the host reads, so no round syncs.
  double* norm = nullptr;        // kNormSlots * n_local sums of g^2 (zeroed after each fold)
  double* norm_max = nullptr;    // running max of ||g|| since the last host read
  double* norm_host = nullptr;   // pinned
  uint32_t norm_slot = 0;        // next free slot
  double* norm_out = nullptr;    // host grad_norm_out raised at the next read
  double* scratch = nullptr;     // trace metrics (4 doubles)
  unsigned int* arrive = nullptr;
  unsigned int* error = nullptr;
  // k_local_tma per-CTA round flags: inside dsgd_run_rounds, consecutive
  // p = 1 rounds chain CTA to CTA instead of draining the whole grid
  unsigned long long* lt_flags = nullptr;
  uint64_t lt_seq = 0;           // k_local_tma launches (the flag value of the last one)
  bool lt_run = false;           // inside dsgd_run_rounds
  bool lt_prev = false;          // ... and the previous round was a k_local_tma launch
  char* staging = nullptr;       // pinned host staging (d * 8 bytes)

  int cur = 0;                   // theta buffer holding the current state
  std::vector<uint64_t> t;       // NodeState::t per local node
  uint64_t rounds_done = 0;      // rounds this context has run (lock-step)
  uint64_t seq = 0;              // round counters published so far (multi-GPU)
  uint64_t ea_seq = 0;           // gated EASGD rounds run (multi-GPU chain)
  uint64_t ea_chunk_used = 1024; // elements per chain flag of the last chain round
  void* ea_update_out[kMaxLocal] = {};   // optional ea_client_step update outputs
  std::vector<uint32_t> prev_readers;  // nodes that read this context's snapshot last round
  bool ar_pending = false;             // multi-GPU all-reduce: theta += avg not yet applied
  dsgd_momentum_scope ar_pending_scope = DSGD_SCOPE_AGGREGATE;
  unsigned long long timeout_ns = 30ull * 1000 * 1000 * 1000;

  // multi-GPU
  std::shared_ptr<InprocGroup> grp;  // in-process group (null: one process per GPU)
  unsigned long long reduce_t = 0;   // in-process two-shot: round of the deferred reduces
  std::vector<uint32_t> fresh_map;   // in-process gossip-fresh: the deferred mix's partners
  double fresh_beta = 0.0;
  bool connected = false;
  std::vector<PeerNode> peers;   // all p nodes
  std::vector<void*> ipc_opened;
  ncclComm_t comm = nullptr;

  // LogisticObjective dataset (dsgd_set_logistic), replicated per context
  char* lg_X = nullptr;                       // n x d, context dtype
  int32_t* lg_y = nullptr;
  uint64_t lg_n = 0;
  double lg_l2 = 0.0;
  std::vector<uint64_t> lg_begin, lg_end;     // per local node sample range
  uint64_t* lg_rows = nullptr;                // device minibatch rows
  double* lg_scratch = nullptr;               // partial dots + coefficients
  size_t lg_rows_cap = 0, lg_scratch_cap = 0;
  std::vector<uint64_t> lg_rows_host;
  uint64_t* lg_pin[4] = {};                   // pinned staging ring for the rows (async H2D)
  cudaEvent_t lg_ev[4] = {};
  size_t lg_pin_cap = 0;
  uint32_t lg_slot = 0;

  // worker-loop streams
  std::vector<dsgd_stream*> partner_streams;  // all p (every context draws the full map)
  std::vector<dsgd_stream*> noise_streams;    // local nodes
  std::vector<dsgd_stream*> sample_streams;   // local nodes (logistic minibatch rows)
  dsgd_stream* clock_stream = nullptr;        // run-level Poisson clock (async drivers)
  double* noise_host = nullptr;               // d doubles

  // measurement
  bool profile = false;
  std::vector<Prof> prof_pending;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[DSGD_K_COUNT] = {};
  uint64_t prof_launches[DSGD_K_COUNT] = {};
  uint64_t kernels = 0, nccl_calls = 0;

  char* theta_ptr(uint32_t i, int buf) const { return arena + off_theta[i][buf]; }
  unsigned long long* round_ptr(uint32_t i) const {
    return reinterpret_cast<unsigned long long*>(arena + off_round) + i;
  }
  bool distributed() const { return n_local < p; }
};

namespace {

dsgd_status check_ctx(dsgd_ctx* ctx) {
  if (!ctx) return set_error(DSGD_EINVAL, "null context");
  return DSGD_OK;
}

cudaEvent_t take_event(dsgd_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launch with events when profiling.
struct LaunchScope {
  dsgd_ctx* c;
  int id;
  cudaStream_t st;
  bool nccl;  // an NCCL call (counted apart from this library's kernels)
  cudaEvent_t a = nullptr;
  uint64_t issued0;  // dsgd::launches_issued() at entry: every kernel, tails included
  LaunchScope(dsgd_ctx* ctx, int kid, cudaStream_t on = nullptr, bool is_nccl = false)
      : c(ctx), id(kid), st(on ? on : ctx->stream), nccl(is_nccl),
        issued0(dsgd::launches_issued()) {
    if (c->profile) {
      a = take_event(c);
      cudaEventRecord(a, st);
    }
  }
  ~LaunchScope() {
    if (nccl)
      c->nccl_calls++;
    c->kernels += dsgd::launches_issued() - issued0;
    if (c->profile) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, st);
      c->prof_pending.push_back({id, a, b});
    }
  }
};

dsgd_status collect_profile(dsgd_ctx* c) {
  if (c->prof_pending.empty()) return DSGD_OK;
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  for (const Prof& p : c->prof_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->prof_ms[p.id] += ms;
    c->prof_launches[p.id] += 1;
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->prof_pending.clear();
  return DSGD_OK;
}

uint32_t blocks_for(const dsgd_ctx* c, uint64_t elems_per_node, uint32_t nodes) {
  const uint64_t want = std::max<uint64_t>(1, (elems_per_node + dsgd::kBlock - 1) / dsgd::kBlock);
  const uint64_t cap = std::max<uint64_t>(1, (uint64_t)c->sm_count * c->blocks_per_sm / nodes);
  return (uint32_t)std::min(want, cap);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
T* as(char* p) {
  return reinterpret_cast<T*>(p);
}

// Resolved gradient source for one launch.
struct GradSel {
  int quad = 0;
  bool logistic = false;          // produce the gradient into c->grad first
  const uint64_t* rows = nullptr; // caller-drawn logistic rows (host), or null
  const void* grad[kMaxLocal] = {};
  bool noise = false;
  bool norm = false;
  bool dev_noise = false;  // Philox noise inside the kernel
  double sigma = 0.0;
  uint64_t seed = 0;
};

dsgd_status resolve_grad(dsgd_ctx* c, const dsgd_grad_spec* g, GradSel* out) {
  GradSel s;
  if (!g) return set_error(DSGD_EINVAL, "null gradient spec");
  if (g->source == DSGD_GRAD_QUADRATIC) {
    if (!c->spec) return set_error(DSGD_ESTATE, "no quadratic objective (DSGD_CTX_QUADRATIC)");
    s.quad = 1;
  } else if (g->source == DSGD_GRAD_BUFFER) {
    for (uint32_t i = 0; i < c->n_local; ++i) {
      s.grad[i] = g->grad ? g->grad[i] : c->grad[i];
      if (!s.grad[i]) return set_error(DSGD_EINVAL, "missing gradient buffer");
    }
  } else if (g->source == DSGD_GRAD_LOGISTIC) {
    if (!c->lg_X) return set_error(DSGD_ESTATE, "no logistic dataset (dsgd_set_logistic)");
    s.logistic = true;
    s.rows = g->rows;
    for (uint32_t i = 0; i < c->n_local; ++i) s.grad[i] = c->grad[i];
  } else {
    return set_error(DSGD_EINVAL, "unknown gradient source");
  }
  if (g->use_noise == 1) {
    if (!c->noise[0]) return set_error(DSGD_ESTATE, "no noise buffers (DSGD_CTX_NOISE)");
    s.noise = true;
  } else if (g->use_noise == 2) {
    if (!(g->noise_sigma >= 0.0)) return set_error(DSGD_EINVAL, "noise sigma must be >= 0");
    s.dev_noise = g->noise_sigma > 0.0;
    s.sigma = g->noise_sigma;
    s.seed = g->noise_seed;
  } else if (g->use_noise != 0) {
    return set_error(DSGD_EINVAL, "use_noise must be 0, 1 or 2");
  }
  s.norm = g->grad_norm_out != nullptr;
  *out = s;
  return DSGD_OK;
}

template <typename T>
void fill_node(dsgd_ctx* c, uint32_t i, const GradSel& gs, const dsgd_hyperparams* h,
               dsgd::NodeIO<T>* n, bool negate_alpha = false) {
  n->theta_in = as<T>(c->theta_ptr(i, c->cur));
  n->theta_out = as<T>(c->theta_ptr(i, c->cur ^ 1));
  n->delta = as<T>(c->delta[i]);
  n->grad = gs.quad ? nullptr : static_cast<const T*>(gs.grad[i]);
  n->noise = gs.noise ? as<T>(c->noise[i]) : nullptr;
  n->partner = nullptr;
  n->aux = nullptr;
  n->norm = gs.norm ? c->norm + (size_t)c->norm_slot * c->n_local + i : nullptr;
  const double alpha = h ? dsgd_step_size_at(h, c->t[i]) : 0.0;
  n->alpha = (T)(negate_alpha ? -alpha : alpha);
  n->nsigma = gs.dev_noise ? (T)gs.sigma : T(0);
  n->nkey = gs.seed * 0x9E3779B97F4A7C15ull ^ (uint64_t(c->first + i) + 1) * 0xD1B54A32D192ED03ull;
  n->nctr = c->t[i];
  n->nbase = 0;
}

template <typename A>
void fill_common(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs, A* a) {
  using T = std::remove_pointer_t<decltype(a->spec)>;
  using TT = std::remove_const_t<T>;
  a->spec = gs.quad ? as<TT>(c->spec) : nullptr;
  a->opt = gs.quad ? as<TT>(c->opt) : nullptr;
  a->d = c->d;
  a->mu = (TT)h->mu;
  a->wd = (TT)h->weight_decay;
  a->mu_nz = h->mu != 0.0;
  a->wd_pos = h->weight_decay > 0.0;
  a->quad = gs.quad;
}

bool all_aligned(dsgd_ctx* c, const GradSel& gs) {
  for (uint32_t i = 0; i < c->n_local; ++i)
    if (!gs.quad && !aligned16(gs.grad[i])) return false;
  return true;
}

dsgd_status join_pipes(dsgd_ctx* c);

// Folds the used norm slots into norm_max on the device (no host wait).
dsgd_status norm_fold(dsgd_ctx* c) {
  if (c->norm_slot == 0) return DSGD_OK;
  DSGD_TRY(join_pipes(c));
  {
    LaunchScope ls(c, DSGD_K_OTHER);
    DSGD_CUDA(dsgd::launch_norm_fold(c->norm, (uint64_t)c->norm_slot * c->n_local, c->norm_max,
                                     c->stream));
  }
  c->norm_slot = 0;
  return DSGD_OK;
}

// Raises the registered host grad_norm_out to the device running max and
// restarts the max (the only place the norm path waits for the device).
dsgd_status norm_read(dsgd_ctx* c) {
  if (!c->norm_out) return DSGD_OK;
  DSGD_TRY(norm_fold(c));
  DSGD_TRY(join_pipes(c));
  DSGD_CUDA(cudaMemcpyAsync(c->norm_host, c->norm_max, sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
  DSGD_CUDA(cudaMemsetAsync(c->norm_max, 0, sizeof(double), c->stream));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  *c->norm_out = std::max(*c->norm_out, c->norm_host[0]);
  c->norm_out = nullptr;
  return DSGD_OK;
}

// A round that reports its gradient norm writes slot norm_slot; a different
// host pointer than the registered one first settles the registered one.
dsgd_status norm_begin(dsgd_ctx* c, const GradSel& gs, const dsgd_grad_spec* g) {
  if (!gs.norm) return DSGD_OK;
  if (c->norm_out && c->norm_out != g->grad_norm_out) DSGD_TRY(norm_read(c));
  c->norm_out = g->grad_norm_out;
  if (c->norm_slot >= dsgd::kNormSlots) DSGD_TRY(norm_fold(c));
  return DSGD_OK;
}

dsgd_status norm_end(dsgd_ctx* c, const GradSel& gs, const dsgd_grad_spec* g) {
  (void)g;
  if (gs.norm) c->norm_slot += 1;
  return DSGD_OK;
}

void finish_round(dsgd_ctx* c, bool flip, bool advance_t = true) {
  if (flip) c->cur ^= 1;
  if (advance_t)
    for (auto& t : c->t) t += 1;
  c->rounds_done += 1;
}

dsgd_status check_common_round(dsgd_ctx* c) {
  for (uint64_t t : c->t)
    if (t != c->t[0])
      return set_error(DSGD_EINVAL, "synchronous round requires equal node clocks");
  return DSGD_OK;
}

dsgd_status check_map(dsgd_ctx* c, const uint32_t* m) {
  if (!m) return set_error(DSGD_EINVAL, "null partner map");
  for (uint32_t i = 0; i < c->p; ++i)
    if (m[i] >= c->p) return set_error(DSGD_EINVAL, "partner index out of range");
  return DSGD_OK;
}

// DSGD_TRACE: give this launch a trace slot (kind = dsgd_kernel_id).
void trace_slot(dsgd_ctx* c, int kind, dsgd::WaitSpec* w, dsgd::SignalSpec* s) {
  if (!c->trace_dev || c->trace_n >= c->trace_cap) return;
  unsigned long long* slot = c->trace_dev + 3ull * c->trace_n;
  c->trace_kind.push_back((uint32_t)kind);
  c->trace_round.push_back(c->rounds_done);
  c->trace_n++;
  if (w) w->trace = slot;
  if (s) s->trace = slot;
}

// Wait list of a multi-GPU round that reads `reads` (the partner, or none)
// and overwrites the snapshot the previous round's pullers read.
dsgd_status build_waits(dsgd_ctx* c, const std::vector<uint32_t>& reads, dsgd::WaitSpec* w) {
  w->n = 0;
  w->timeout_ns = c->timeout_ns;
  w->error = c->error;
  if (!c->distributed()) return DSGD_OK;
  const uint32_t me = c->first;
  bool full = false;
  auto add = [&](uint32_t node) {
    if (node == me) return;
    for (int k = 0; k < w->n; ++k)
      if (w->ptr[k] == c->peers[node].round) return;
    if (w->n == kMaxWait) {
      full = true;
      return;
    }
    w->ptr[w->n] = c->peers[node].round;
    w->val[w->n] = c->seq;
    w->n++;
  };
  for (uint32_t j : reads) add(j);            // RAW: partner finished round r-1
  for (uint32_t k : c->prev_readers) add(k);  // WAR: last round's readers of my snapshot
  if (full)  // never drop a wait: that would be a silent race
    return set_error(DSGD_EINVAL, "more than 16 peers to wait for in one round");
  return DSGD_OK;
}

// Waits until every peer has published round counter `value` (all of them
// finished the same lock-step launch sequence).
dsgd_status all_peer_waits(dsgd_ctx* c, unsigned long long value, dsgd::WaitSpec* w) {
  w->n = 0;
  w->timeout_ns = c->timeout_ns;
  w->error = c->error;
  if (!c->distributed()) return DSGD_OK;
  for (uint32_t k = 0; k < c->p; ++k) {
    if (k == c->first) continue;
    if (w->n == kMaxWait) return set_error(DSGD_EINVAL, "more than 16 peers to wait for");
    w->ptr[w->n] = c->peers[k].round;
    w->val[w->n] = value;
    w->n++;
  }
  return DSGD_OK;
}

// local_writes: the kernel stores only into this GPU's memory (see
// SignalSpec::local_only)
bool signal_gpu_scope() {
  static const bool on = [] {  // DSGD_SIGNAL_GPU=0: a system fence in every CTA
    const char* e = std::getenv("DSGD_SIGNAL_GPU");
    return !(e && e[0] == '0');
  }();
  return on;
}

void build_signal(dsgd_ctx* c, dsgd::SignalSpec* s, bool local_writes = true) {
  if (!c->distributed()) {
    s->counter = nullptr;
    return;
  }
  s->counter = c->round_ptr(0);
  s->value = c->seq + 1;
  s->arrive = c->arrive;
  s->local_only = local_writes && signal_gpu_scope() ? 1 : 0;
}

template <typename T>
dsgd_status run_step_mode(dsgd_ctx* c, int mode, int kid, const dsgd_hyperparams* h,
                          const GradSel& gs, const uint32_t* partner_of, T beta,
                          bool negate_alpha, const std::vector<uint32_t>& reads) {
  dsgd::StepArgs<T> a{};
  for (uint32_t i = 0; i < c->n_local; ++i) {
    fill_node<T>(c, i, gs, h, &a.node[i], negate_alpha);
    if (partner_of) {
      const uint32_t j = partner_of[c->first + i];
      a.node[i].partner = as<T>(c->peers[j].theta[c->cur]);
    }
  }
  if (h) {
    fill_common(c, h, gs, &a);
  } else {
    a.d = c->d;
  }
  a.beta = beta;
  a.n_local = c->n_local;
  bool vec = all_aligned(c, gs);
  if (partner_of)
    for (uint32_t i = 0; i < c->n_local; ++i) vec = vec && aligned16(a.node[i].partner);
  // a remote partner (one node per GPU): stage its snapshot through smem
  a.tma_partner = partner_of && c->distributed() && c->ar_tma &&
                  partner_of[c->first] != c->first;
  const uint64_t W = vec ? 16 / sizeof(T) : 1;
  a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, c->n_local);
  DSGD_TRY(build_waits(c, reads, &a.wait));
  build_signal(c, &a.signal);
  trace_slot(c, kid, &a.wait, &a.signal);
  const uint32_t grid = a.blocks_per_node * c->n_local;
  LaunchScope ls(c, kid);
  DSGD_CUDA(dsgd::launch_step<T>(mode, a, vec ? 1 : 0, grid, c->stream));
  if (c->distributed()) c->seq += 1;
  return DSGD_OK;
}

// Copies lg_rows_host[0, nr) to the device rows buffer through a ring of
// pinned slots (an async copy; a slot is reused once its copy completed), so
// the host does not wait for the stream every round.
dsgd_status stage_rows(dsgd_ctx* c, size_t nr) {
  if (c->lg_pin_cap < nr) {
    for (int k = 0; k < 4; ++k) {
      if (c->lg_ev[k]) DSGD_CUDA(cudaEventSynchronize(c->lg_ev[k]));
      cudaFreeHost(c->lg_pin[k]);
      c->lg_pin[k] = nullptr;
    }
    for (int k = 0; k < 4; ++k) {
      DSGD_CUDA(cudaMallocHost(&c->lg_pin[k], nr * sizeof(uint64_t)));
      if (!c->lg_ev[k]) DSGD_CUDA(cudaEventCreateWithFlags(&c->lg_ev[k], cudaEventDisableTiming));
    }
    c->lg_pin_cap = nr;
  }
  const uint32_t k = c->lg_slot++ % 4;
  DSGD_CUDA(cudaEventSynchronize(c->lg_ev[k]));
  std::memcpy(c->lg_pin[k], c->lg_rows_host.data(), nr * sizeof(uint64_t));
  DSGD_CUDA(cudaMemcpyAsync(c->lg_rows, c->lg_pin[k], nr * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, c->stream));
  DSGD_CUDA(cudaEventRecord(c->lg_ev[k], c->stream));
  return DSGD_OK;
}

// LogisticObjective::stochastic_gradient (objectives.cpp:147-162) of the
// local nodes `nodes` at theta[cur] (+ mu * delta_prev when lookahead, the
// compute_local_delta evaluation point protocols.cpp:90-93), written into
// their gradient buffers.  Rows come from the caller (gs.rows) or from each
// node's sample stream, in batch order (objectives.cpp:154-157).
template <typename T>
dsgd_status produce_logistic(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs,
                             const std::vector<uint32_t>& nodes, bool lookahead) {
  if (!gs.logistic || nodes.empty()) return DSGD_OK;
  const uint32_t B = h->batch;
  if (B == 0) return set_error(DSGD_EINVAL, "batch must be >= 1");
  const uint32_t nn = (uint32_t)nodes.size();
  c->lg_rows_host.resize((size_t)nn * B);
  for (uint32_t q = 0; q < nn; ++q) {
    const uint32_t i = nodes[q];
    for (uint32_t b = 0; b < B; ++b) {
      uint64_t row;
      if (gs.rows) {
        row = gs.rows[(size_t)i * B + b];
        if (row >= c->lg_n) return set_error(DSGD_EINVAL, "logistic row out of range");
      } else {
        if (c->sample_streams.size() != c->n_local)
          return set_error(DSGD_ESTATE, "dsgd_ctx_seed_streams first");
        uint32_t j = 0;
        DSGD_TRY(dsgd_stream_uniform_index(c->sample_streams[i],
                                           (uint32_t)(c->lg_end[i] - c->lg_begin[i]), &j));
        row = c->lg_begin[i] + j;
      }
      c->lg_rows_host[(size_t)q * B + b] = row;
    }
  }
  const uint32_t nblk = (uint32_t)std::min<uint64_t>(
      64, std::max<uint64_t>(1, (c->d + 8 * kBlockU - 1) / (8 * kBlockU)));
  const size_t nr = (size_t)nn * B;
  if (c->lg_rows_cap < nr) {
    cudaFree(c->lg_rows);
    c->lg_rows = nullptr;
    DSGD_CUDA(cudaMalloc(&c->lg_rows, nr * sizeof(uint64_t)));
    c->lg_rows_cap = nr;
  }
  if (c->lg_scratch_cap < nr * (nblk + 1)) {
    cudaFree(c->lg_scratch);
    c->lg_scratch = nullptr;
    DSGD_CUDA(cudaMalloc(&c->lg_scratch, nr * (nblk + 1) * sizeof(double)));
    c->lg_scratch_cap = nr * (nblk + 1);
  }
  DSGD_TRY(stage_rows(c, nr));
  dsgd::LogisticArgs<T> a{};
  a.X = as<T>(c->lg_X);
  a.y = c->lg_y;
  for (uint32_t q = 0; q < nn; ++q) {
    const uint32_t i = nodes[q];
    a.theta[q] = as<T>(c->theta_ptr(i, c->cur));
    a.delta[q] = as<T>(c->delta[i]);
    a.out[q] = as<T>(c->grad[i]);
  }
  a.rows = c->lg_rows;
  a.partial = c->lg_scratch;
  a.coeff = c->lg_scratch + nr * nblk;
  a.d = c->d;
  a.n_nodes = nn;
  a.batch = B;
  a.nblk = nblk;
  a.mu = (T)h->mu;
  a.l2 = (T)c->lg_l2;
  a.inv_batch = (T)(1.0 / (double)B);
  a.lookahead = lookahead && h->mu != 0.0;
  LaunchScope ls(c, DSGD_K_OTHER);
  DSGD_CUDA(dsgd::launch_logistic<T>(a, blocks_for(c, c->d, 1), c->stream));
  return DSGD_OK;
}

// sum over all p nodes of the data term of LogisticObjective::value
// (objectives.cpp:116-125), each node's rows summed in row order on the host.
template <typename T>
dsgd_status logistic_values(dsgd_ctx* c, double* data) {
  const uint32_t p = c->p;
  const uint64_t n = c->lg_n;
  const size_t nr = (size_t)p * n;
  if (nr > 0xffffffffull) return set_error(DSGD_EINVAL, "trace: logistic dataset too large");
  const uint32_t nblk = (uint32_t)std::min<uint64_t>(
      64, std::max<uint64_t>(1, (c->d + 8 * kBlockU - 1) / (8 * kBlockU)));
  if (c->lg_rows_cap < nr) {
    cudaFree(c->lg_rows);
    c->lg_rows = nullptr;
    DSGD_CUDA(cudaMalloc(&c->lg_rows, nr * sizeof(uint64_t)));
    c->lg_rows_cap = nr;
  }
  if (c->lg_scratch_cap < nr * (nblk + 1)) {
    cudaFree(c->lg_scratch);
    c->lg_scratch = nullptr;
    DSGD_CUDA(cudaMalloc(&c->lg_scratch, nr * (nblk + 1) * sizeof(double)));
    c->lg_scratch_cap = nr * (nblk + 1);
  }
  c->lg_rows_host.resize(nr);
  for (size_t r = 0; r < nr; ++r) c->lg_rows_host[r] = r % n;
  DSGD_TRY(stage_rows(c, nr));
  dsgd::LogisticArgs<T> a{};
  a.X = as<T>(c->lg_X);
  a.y = c->lg_y;
  for (uint32_t k = 0; k < p; ++k) a.theta[k] = as<T>(c->peers[k].theta[c->cur]);
  a.rows = c->lg_rows;
  a.partial = c->lg_scratch;
  a.coeff = c->lg_scratch + nr * nblk;
  a.d = c->d;
  a.n_nodes = p;
  a.batch = (uint32_t)n;
  a.nblk = nblk;
  a.value_mode = 1;
  {
    LaunchScope ls(c, DSGD_K_OTHER);
    DSGD_CUDA(dsgd::launch_logistic<T>(a, 1, c->stream));
  }
  std::vector<double> terms(nr);
  DSGD_CUDA(cudaMemcpyAsync(terms.data(), a.coeff, nr * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  double total = 0.0;
  for (uint32_t k = 0; k < p; ++k) {
    double s = 0.0;
    for (uint64_t r = 0; r < n; ++r) s += terms[(size_t)k * n + r];
    total += s / (double)n;
  }
  *data = total;
  return DSGD_OK;
}

std::vector<uint32_t> all_local(const dsgd_ctx* c) {
  std::vector<uint32_t> v(c->n_local);
  for (uint32_t i = 0; i < c->n_local; ++i) v[i] = i;
  return v;
}

template <typename T>
dsgd_status do_local_step(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs) {
  DSGD_TRY(run_step_mode<T>(c, dsgd::kModeStep, DSGD_K_STEP, h, gs, nullptr, T(0), false, {}));
  c->prev_readers.clear();
  return DSGD_OK;
}

template <typename T>
dsgd_status do_pull(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs,
                    const uint32_t* partner_of, int mode, T beta) {
  std::vector<uint32_t> reads;
  for (uint32_t i = 0; i < c->n_local; ++i) reads.push_back(partner_of[c->first + i]);
  DSGD_TRY(run_step_mode<T>(c, mode, DSGD_K_STEP, h, gs, partner_of, beta, false, reads));
  c->prev_readers.clear();
  for (uint32_t k = 0; k < c->p; ++k)
    if (partner_of[k] == c->first && c->distributed()) c->prev_readers.push_back(k);
  return DSGD_OK;
}

// Waits of a peer-memory all-reduce kernel: every rank's counter `which`
// (0: exchange written, 1: average written) has reached `need`.
void ar_waits(dsgd_ctx* c, int which, unsigned long long need, dsgd::WaitSpec* w) {
  w->n = 0;
  w->timeout_ns = c->timeout_ns;
  w->error = c->error;
  for (uint32_t k = 0; k < c->p && w->n < kMaxWait; ++k) {
    w->ptr[w->n] = c->peers[k].ar + which;
    w->val[w->n] = need;
    w->n++;
  }
}

// Joins the two-shot pipeline streams back into the context stream.
dsgd_status join_pipes(dsgd_ctx* c) {
  if (!c->pipes_forked) return DSGD_OK;
  for (uint32_t h = 0; h < 4; ++h) {  // every pipeline stream (the size table may pick 4)
    DSGD_CUDA(cudaEventRecord(c->pipe_event[h], c->pipe_stream[h]));
    DSGD_CUDA(cudaStreamWaitEvent(c->stream, c->pipe_event[h], 0));
  }
  c->pipes_forked = false;
  return DSGD_OK;
}

// Orders this round's pipeline work after everything on the context stream
// (e.g. the caller's gradient upload).  Recorded every round.
dsgd_status fork_pipes(dsgd_ctx* c) {
  DSGD_CUDA(cudaEventRecord(c->pipe_event[4], c->stream));
  for (uint32_t h = 0; h < 4; ++h)
    DSGD_CUDA(cudaStreamWaitEvent(c->pipe_stream[h], c->pipe_event[4], 0));
  c->pipes_forked = true;
  return DSGD_OK;
}

char* x_of(dsgd_ctx* c, uint32_t k, uint64_t round) {
  return (round & 1) ? c->peers[k].x2 : c->peers[k].x;
}

template <typename T>
dsgd::ArOneShotArgs<T> oneshot_args(dsgd_ctx* c, dsgd_momentum_scope scope) {
  dsgd::ArOneShotArgs<T> a{};
  const uint64_t t = c->ar_rounds;
  for (uint32_t k = 0; k < c->p; ++k) a.x_prev[k] = t ? as<T>(x_of(c, k, t - 1)) : nullptr;
  a.x_out = as<T>(x_of(c, c->first, t));
  a.d = c->d;
  a.p = c->p;
  a.ring_base = c->d / c->p;
  a.ring_rem = c->d % c->p;
  a.agg = scope == DSGD_SCOPE_AGGREGATE;
  a.pending = c->ar_pending;
  a.tma_rank = c->ar_tma ? (int)c->first : -1;
  return a;
}

// Materialises a deferred multi-GPU all-reduce apply: theta += avg.
template <typename T>
dsgd_status flush_pending_t(dsgd_ctx* c) {
  if (!c->ar_pending) return DSGD_OK;
  if (c->p2p_allreduce && c->ar_oneshot) {
    dsgd::ArOneShotArgs<T> a = oneshot_args<T>(c, c->ar_pending_scope);
    a.node.theta_in = as<T>(c->theta_ptr(0, c->cur));
    a.node.theta_out = as<T>(c->theta_ptr(0, c->cur ^ 1));
    a.node.delta = as<T>(c->delta[0]);
    a.apply_only = 1;
    ar_waits(c, 0, c->ar_rounds, &a.wait);  // every rank's last exchange is written
    build_signal(c, &a.signal);
    {
      LaunchScope ls(c, DSGD_K_AR_APPLY);
      DSGD_CUDA(dsgd::launch_ar_oneshot<T>(a, 1, blocks_for(c, (c->d / (16 / sizeof(T)) + 1), 1),
                                           c->stream));
    }
    c->seq += 1;
    c->cur ^= 1;
    c->ar_pending = false;
    return DSGD_OK;
  }
  DSGD_TRY(join_pipes(c));
  const bool p2p = c->p2p_allreduce;
  char* xbuf = p2p ? c->peers[c->first].avg
                   : (c->ar_pending_scope == DSGD_SCOPE_PER_NODE ? c->aux[0] : c->delta[0]);
  dsgd::StepArgs<T> a{};
  if (p2p) {  // every owner wrote its average slice, in every pipeline
    a.wait.n = 0;
    a.wait.timeout_ns = c->timeout_ns;
    a.wait.error = c->error;
    for (uint32_t h = 0; h < c->ar_pipes_used; ++h)
      for (uint32_t k = 0; k < c->p && a.wait.n < kMaxWait; ++k) {
        a.wait.ptr[a.wait.n] = c->peers[k].ar + 2 * h + 1;
        a.wait.val[a.wait.n] = c->ar_rounds;
        a.wait.n++;
      }
  }
  a.node[0].theta_in = as<T>(c->theta_ptr(0, c->cur));
  a.node[0].theta_out = as<T>(c->theta_ptr(0, c->cur ^ 1));
  a.node[0].aux = as<T>(xbuf);
  a.d = c->d;
  a.n_local = 1;
  const uint64_t W = 16 / sizeof(T);
  a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
  build_signal(c, &a.signal);
  {
    LaunchScope ls(c, DSGD_K_AR_APPLY);
    DSGD_CUDA(dsgd::launch_step<T>(dsgd::kModeApply, a, 1, a.blocks_per_node, c->stream));
  }
  c->seq += 1;
  c->cur ^= 1;
  c->ar_pending = false;
  if (p2p && c->ar_pending_scope == DSGD_SCOPE_AGGREGATE)  // delta_prev = the average
    DSGD_CUDA(cudaMemcpyAsync(c->delta[0], xbuf, c->d * c->es, cudaMemcpyDeviceToDevice,
                              c->stream));
  return DSGD_OK;
}

dsgd_status flush_pending(dsgd_ctx* c) {
  if (!c->ar_pending) return DSGD_OK;
  DeviceGuard g(c->device);
  return c->dtype == DSGD_F32 ? flush_pending_t<float>(c) : flush_pending_t<double>(c);
}

// Second kernel of pipeline `pi` of a two-shot round t: reduce this rank's
// slice of every rank's exchange buffer and write the average to every rank
// (NVLS multimem, or peer memory in the reference ring order).
template <typename T>
dsgd_status launch_reduce_pipe(dsgd_ctx* c, uint32_t pi, uint32_t K, unsigned long long t) {
  const uint32_t me = c->first;
  cudaStream_t st = K > 1 ? c->pipe_stream[pi] : c->stream;
  const uint64_t b0 = (c->d * pi / K) / 64 * 64;
  const uint64_t b1 = pi + 1 == K ? c->d : (c->d * (pi + 1) / K) / 64 * 64;
  const uint64_t len = b1 - b0;
  unsigned int* arrive = c->arrive + 40 + pi;
  dsgd::WaitSpec wx{};
  wx.timeout_ns = c->timeout_ns;
  wx.error = c->error;
  for (uint32_t k = 0; k < c->p; ++k) {  // every rank's exchange of this pipeline is written
    wx.ptr[wx.n] = c->peers[k].ar + 2 * pi;
    wx.val[wx.n] = t + 1;
    wx.n++;
  }
  dsgd::SignalSpec sx{c->peers[me].ar + 2 * pi + 1, t + 1, arrive, nullptr};
  trace_slot(c, DSGD_K_NCCL + 16 * pi, &wx, &sx);
  if (c->ar_nvls) {
    dsgd::ArNvlsArgs<T> a{};
    a.x_mc = as<T>(c->nvls_x_mc);
    a.avg_mc = as<T>(c->nvls_avg_mc);
    const uint64_t per = ((len + c->p - 1) / c->p + 3) / 4 * 4;
    a.lo = std::min<uint64_t>(b1, b0 + (uint64_t)me * per);
    a.hi = std::min<uint64_t>(b1, a.lo + per);
    a.p = c->p;
    a.wait = wx;
    a.signal = sx;
    const uint32_t cap = std::max<uint32_t>(1, (uint32_t)(c->sm_count * c->ar_comm_frac / K));
    const uint32_t grid = std::min<uint32_t>(cap, std::max<uint32_t>(1, (uint32_t)((a.hi - a.lo) / 4 / kBlockU + 1)));
    LaunchScope ls(c, DSGD_K_NCCL, st);
    DSGD_CUDA(dsgd::launch_ar_nvls<T>(a, grid, st));
  } else {
    dsgd::ArReduceArgs<T> a{};
    for (uint32_t k = 0; k < c->p; ++k) {
      a.x[k] = as<T>(c->peers[k].x);
      a.avg[k] = as<T>(c->peers[k].avg);
    }
    a.p = c->p;
    a.slice = me;
    const uint64_t base = c->d / c->p, rem = c->d % c->p;  // transport.cpp:193-198
    const uint64_t clo = (uint64_t)me * base + std::min<uint64_t>(me, rem);
    const uint64_t chi = clo + base + (me < rem ? 1 : 0);
    a.lo = std::max(clo, b0);  // my ring chunk within this pipeline's range
    a.hi = std::max(a.lo, std::min(chi, b1));
    a.wait = wx;
    a.signal = sx;
    const uint32_t grid =
        std::max<uint32_t>(1, blocks_for(c, (a.hi - a.lo) / (16 / sizeof(T)) + 1, 1) / K);
    LaunchScope ls(c, DSGD_K_NCCL, st);
    DSGD_CUDA(dsgd::launch_ar_reduce<T>(a, grid, st));
  }
  return DSGD_OK;
}

// Multi-GPU all-reduce round over NVLink peer memory, two kernels:
//  1. fused (previous apply +) delta kernel -> own exchange buffer x
//     [waits: every rank's averages of the previous round are written]
//  2. reduce + all-gather of this rank's reference ring chunk: sum of every
//     rank's x in ring order / p -> every rank's avg buffer
//     [waits: every rank's exchange buffer is written]
// Bit-exact with the reference's ring_allreduce (transport.cpp:183-248).
template <typename T>
dsgd_status do_allreduce_p2p(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs,
                             dsgd_momentum_scope scope) {
  if (!c->peers[c->first].x) return set_error(DSGD_ESTATE, "no all-reduce buffers");
  if (c->ar_pending && c->ar_pending_scope != scope) DSGD_TRY(flush_pending_t<T>(c));
  const uint32_t me = c->first;
  const bool fused = c->ar_pending;
  const unsigned long long t = c->ar_rounds;
  if (c->ar_oneshot) {
    dsgd::ArOneShotArgs<T> a = oneshot_args<T>(c, scope);
    fill_node<T>(c, 0, gs, h, &a.node);
    if (fused) a.node.theta_out = as<T>(c->theta_ptr(0, c->cur ^ 1));
    a.spec = gs.quad ? as<T>(c->spec) : nullptr;
    a.opt = gs.quad ? as<T>(c->opt) : nullptr;
    a.mu = (T)h->mu;
    a.wd = (T)h->weight_decay;
    a.mu_nz = h->mu != 0.0;
    a.wd_pos = h->weight_decay > 0.0;
    a.quad = gs.quad;
    // RAW on every rank's x[t-1], WAR on my x[t % 2] (read by peers in round t-1)
    ar_waits(c, 0, t, &a.wait);
    a.signal.counter = c->peers[me].ar + 0;
    a.signal.value = t + 1;
    a.signal.arrive = c->arrive;
    a.signal.local_only = signal_gpu_scope() ? 1 : 0;  // x', theta', delta: own memory
    trace_slot(c, DSGD_K_NCCL, &a.wait, &a.signal);
    const bool vec = all_aligned(c, gs);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    {
      LaunchScope ls(c, DSGD_K_NCCL);
      DSGD_CUDA(dsgd::launch_ar_oneshot<T>(a, vec, blocks_for(c, c->d / W, 1), c->stream));
    }
    if (fused) c->cur ^= 1;
    c->ar_rounds = t + 1;
    c->ar_pending = true;
    c->ar_pending_scope = scope;
    c->prev_readers.clear();
    return DSGD_OK;
  }
  // K independent pipelines over d, one stream each: pipeline h's NVLink-bound
  // reduce overlaps pipeline h'`s HBM-bound delta kernel.
  if (t == 0) {  // the split is fixed for the context's lifetime (counters per pipeline)
    uint32_t k0 = c->ar_pipes;
    // NVLS at >= ~700M per worker: 4 pipelines (10.37 vs 11.37 ms per round
    // at 1B, p = 4, profiles/r2_split_n4.md) unless DSGD_AR_PIPES is set
    if (!c->ar_pipes_env && c->ar_nvls && c->d >= (700ull << 20)) k0 = 4;
    // small d is latency-bound: one pipeline (fewer launches / cross-GPU waits)
    if (c->d < (8u << 20)) k0 = 1;
    while (k0 > 1 && k0 * c->p > (uint32_t)kMaxWait) k0 /= 2;  // wait slots per kernel
    c->ar_pipes_used = k0;
  }
  const uint32_t K = c->ar_pipes_used;
  if (K > 1) DSGD_TRY(fork_pipes(c));
  const bool vec = all_aligned(c, gs);
  const uint64_t W = vec ? 16 / sizeof(T) : 1;
  for (uint32_t pi = 0; pi < K; ++pi) {
    cudaStream_t st = K > 1 ? c->pipe_stream[pi] : c->stream;
    const uint64_t b0 = (c->d * pi / K) / 64 * 64;
    const uint64_t b1 = pi + 1 == K ? c->d : (c->d * (pi + 1) / K) / 64 * 64;
    const uint64_t len = b1 - b0;
    unsigned int* arrive = c->arrive + 40 + pi;  // per pipeline: kernels run concurrently
    {
      dsgd::StepArgs<T> a{};
      fill_node<T>(c, 0, gs, h, &a.node[0]);
      dsgd::NodeIO<T>& n = a.node[0];
      n.theta_in += b0;
      n.theta_out += b0;
      n.delta += b0;
      if (n.grad) n.grad += b0;
      if (n.noise) n.noise += b0;
      n.nbase = b0;
      n.aux = as<T>(c->peers[me].x) + b0;
      n.partner = fused ? as<T>(c->peers[me].avg) + b0 : nullptr;
      fill_common(c, h, gs, &a);
      if (a.spec) a.spec += b0;
      if (a.opt) a.opt += b0;
      a.d = len;
      a.agg = scope == DSGD_SCOPE_AGGREGATE;
      a.n_local = 1;
      a.blocks_per_node = std::max<uint32_t>(1, blocks_for(c, (len / W + 1) / 2, 1) / K);
      a.wait.n = 0;
      a.wait.timeout_ns = c->timeout_ns;
      a.wait.error = c->error;
      for (uint32_t k = 0; k < c->p; ++k) {  // every rank averaged this pipeline's round t-1
        a.wait.ptr[a.wait.n] = c->peers[k].ar + 2 * pi + 1;
        a.wait.val[a.wait.n] = t;
        a.wait.n++;
      }
      a.signal.counter = c->peers[me].ar + 2 * pi;
      a.signal.value = t + 1;
      a.signal.arrive = arrive;
      // per-CTA system fences here: the reduce of every rank starts on this
      // counter, and one GPU-wide fence in the last CTA publishes it later
      // than the CTAs' own fences do (N=4: 272 vs 289-310 us per round,
      // profiles/r2_small_d.md)
      a.signal.local_only = 0;
      trace_slot(c, DSGD_K_AR_DELTA + 16 * pi, &a.wait, &a.signal);
      LaunchScope ls(c, DSGD_K_AR_DELTA, st);
      const int mode = fused ? dsgd::kModeApplyDelta : dsgd::kModeArDelta;
      if (vec && c->ar_tma) {
        // smem-staged streams: a fraction of the SMs saturates HBM and leaves
        // the rest to the other pipeline's NVLink reduce
        const uint32_t g = std::max<uint32_t>(1, (uint32_t)(c->sm_count * c->ar_delta_frac / K));
        DSGD_CUDA(dsgd::launch_ard_tma<T>(mode, a, g, st));
      } else {
        DSGD_CUDA(dsgd::launch_step<T>(mode, a, vec, a.blocks_per_node, st));
      }
    }
    if (K > 1) {
      // the delta kernel is this round's only reader of the caller's buffers
      // (gradient, noise): order the context stream after it, so the next
      // upload into them cannot overwrite what it still reads
      DSGD_CUDA(cudaEventRecord(c->pipe_event[5 + pi], st));
      DSGD_CUDA(cudaStreamWaitEvent(c->stream, c->pipe_event[5 + pi], 0));
    }
    if (!c->grp) DSGD_TRY(launch_reduce_pipe<T>(c, pi, K, t));
  }
  if (c->grp) {
    // in-process group: every rank's exchange kernels are issued before any
    // reduce (host order satisfies every cross-rank wait: the ranks of one
    // GPU share a stream); the last rank issues the reduces of all ranks
    c->reduce_t = t;
    if (c->first + 1 == c->p)
      for (dsgd_ctx* r : c->grp->ctx) {
        DeviceGuard dg(r->device);
        for (uint32_t q = 0; q < K; ++q) DSGD_TRY(launch_reduce_pipe<T>(r, q, K, r->reduce_t));
      }
  }
  if (fused) c->cur ^= 1;
  c->ar_rounds = t + 1;
  c->ar_pending = true;
  c->ar_pending_scope = scope;
  c->prev_readers.clear();
  return DSGD_OK;
}

template <typename T>
dsgd_status do_allreduce(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs,
                         dsgd_momentum_scope scope) {
  if (!c->distributed()) {
    dsgd::AllreduceArgs<T> a{};
    for (uint32_t i = 0; i < c->n_local; ++i) fill_node<T>(c, i, gs, h, &a.node[i]);
    fill_common(c, h, gs, &a);
    a.inv_p = T(1) / T(c->p);
    a.per_node = scope == DSGD_SCOPE_PER_NODE;
    a.p = c->p;
    const bool vec = all_aligned(c, gs);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    const uint32_t grid = blocks_for(c, c->d / W, 1);
    static const bool chain_on = [] {  // DSGD_LT_CHAIN=0: grid-wide waits only
      const char* e = getenv("DSGD_LT_CHAIN");
      return !(e && e[0] == '0');
    }();
    const bool lt = chain_on && c->lt_run && dsgd::local_tma_enabled() && c->n_local == 1 && vec;
    if (lt) {
      // inside dsgd_run_rounds: publish per-CTA flags, and chain behind this
      // run's own previous k_local_tma (every op in between is stream-ordered:
      // host-noise copies, norm folds); the logistic producer kernels write
      // the gradient, so they keep the grid-wide wait
      a.cta_flags = c->lt_flags;
      a.cta_seq = ++c->lt_seq;
      a.cta_chain = c->lt_prev && !gs.logistic ? 1 : 0;
      a.error = c->error;
      a.timeout_ns = c->timeout_ns;
    }
    LaunchScope ls(c, DSGD_K_ALLREDUCE);
    DSGD_CUDA(dsgd::launch_allreduce_local<T>(a, vec, gs.norm, grid, c->stream));
    c->lt_prev = lt;
    c->prev_readers.clear();
    return DSGD_OK;
  }
  if (c->p2p_allreduce) return do_allreduce_p2p<T>(c, h, gs, scope);
  if (!c->comm) return set_error(DSGD_ESTATE, "multi-GPU all-reduce needs dsgd_ctx_init_nccl");
  // delta kernel -> ncclAllReduce(avg) in place on the exchange buffer.
  // Aggregate scope exchanges delta_prev itself, so the averaged delta lands
  // where the next round's momentum reads it.  The apply theta += avg
  // (protocols.cpp:126) is deferred and fused into the next round's delta
  // kernel (kModeApplyDelta: 20 instead of 16 + 12 B/param); any other call
  // first materialises it (flush_pending).
  const bool per_node = scope == DSGD_SCOPE_PER_NODE;
  if (c->ar_pending && c->ar_pending_scope != scope) DSGD_TRY(flush_pending_t<T>(c));
  if (per_node && !c->aux[0]) DSGD_CUDA(cudaMalloc(&c->aux[0], c->d * c->es));
  char* xbuf = per_node ? c->aux[0] : c->delta[0];
  const bool fused = c->ar_pending;
  {
    dsgd::StepArgs<T> a{};
    fill_node<T>(c, 0, gs, h, &a.node[0]);
    a.node[0].aux = as<T>(xbuf);
    fill_common(c, h, gs, &a);
    a.agg = scope == DSGD_SCOPE_AGGREGATE;
    a.n_local = 1;
    const bool vec = all_aligned(c, gs);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
    LaunchScope ls(c, DSGD_K_AR_DELTA);
    DSGD_CUDA(dsgd::launch_step<T>(fused ? dsgd::kModeApplyDelta : dsgd::kModeArDelta, a, vec,
                                   a.blocks_per_node, c->stream));
  }
  if (fused) c->cur ^= 1;  // theta_{t} + avg_{t-1} now materialised in the other buffer
  {
    LaunchScope ls(c, DSGD_K_NCCL, nullptr, true);
    DSGD_NCCL(ncclAllReduce(xbuf, xbuf, c->d, sizeof(T) == 4 ? ncclFloat : ncclDouble, ncclAvg,
                            c->comm, c->stream));
  }
  c->ar_pending = true;
  c->ar_pending_scope = scope;
  c->prev_readers.clear();
  return DSGD_OK;
}

template <typename T>
dsgd_status do_ea(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel& gs, int gated,
                  bool mix_only = false) {
  if (!c->distributed()) {
    if (!(c->flags & DSGD_CTX_CENTER)) return set_error(DSGD_ESTATE, "no center (DSGD_CTX_CENTER)");
    dsgd::EaArgs<T> a{};
    for (uint32_t i = 0; i < c->n_local; ++i) {
      fill_node<T>(c, i, gs, h, &a.node[i]);
      a.node[i].aux = static_cast<T*>(c->ea_update_out[i]);
    }
    fill_common(c, h, gs, &a);
    a.center = as<T>(c->arena + c->off_c_in);
    a.beta = (T)h->beta_ea;
    a.gated = gated;
    a.p = c->p;
    const bool vec = all_aligned(c, gs);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    const uint32_t grid = blocks_for(c, c->d / W, 1);
    LaunchScope ls(c, DSGD_K_EA);
    DSGD_CUDA(dsgd::launch_ea_local<T>(a, vec, gs.norm, grid, c->stream, mix_only));
    c->prev_readers.clear();
    return DSGD_OK;
  }
  if (!gated) return do_local_step<T>(c, h, gs);
  if (!(c->flags & DSGD_CTX_CENTER) || !c->connected)
    return set_error(DSGD_ESTATE, "multi-GPU EASGD needs DSGD_CTX_CENTER on every rank and peers");
  const uint32_t r = c->first;
  const uint32_t next = (r + 1) % c->p;
  c->ea_seq += 1;
  dsgd::EaChainArgs<T> a{};
  fill_node<T>(c, 0, gs, h, &a.node);
  a.spec = gs.quad ? as<T>(c->spec) : nullptr;
  a.opt = gs.quad ? as<T>(c->opt) : nullptr;
  a.c_in = as<T>(c->arena + c->off_c_in);
  a.c_out = as<T>(c->peers[next].c_in);
  a.flag_in = reinterpret_cast<const unsigned long long*>(c->arena + c->off_flags);
  a.flag_out = c->peers[next].flags;
  a.need = r == 0 ? c->ea_seq - 1 : c->ea_seq;
  a.seq = c->ea_seq;
  a.d = c->d;
  // staged chain: one flag per staged tile (the same on every rank)
  a.chunk = dsgd::ea_chain_staged() ? dsgd::ea_chain_tile<T>() : c->ea_chunk;
  a.n_chunks = (c->d + a.chunk - 1) / a.chunk;
  c->ea_chunk_used = a.chunk;
  a.mu = (T)h->mu;
  a.wd = (T)h->weight_decay;
  a.beta = (T)h->beta_ea;
  a.mu_nz = h->mu != 0.0;
  a.wd_pos = h->weight_decay > 0.0;
  a.quad = gs.quad;
  a.timeout_ns = c->timeout_ns;
  a.error = c->error;
  // the center goes into the next rank's memory, but every chunk of it is
  // published with its own system-scope release (flag) before the CTA
  // arrives, so the round counter needs only the gpu-scope arrival chain
  build_signal(c, &a.signal, true);
  const bool vec = all_aligned(c, gs);
  // one CTA per chunk: a CTA blocked on its flag or in its release fence
  // leaves the SM to the other resident chunks (dispatch is in chunk order,
  // the order the previous rank produces them)
  const uint32_t grid = (uint32_t)std::min<uint64_t>(a.n_chunks, 0x7fffffffu);
  LaunchScope ls(c, DSGD_K_EA);
  DSGD_CUDA(dsgd::launch_ea_chain<T>(a, vec, grid, c->stream, mix_only));
  c->seq += 1;
  c->prev_readers.clear();
  return DSGD_OK;
}

template <typename T>
dsgd_status do_push(dsgd_ctx* c, const dsgd_hyperparams* h, const GradSel* gs,
                    const uint32_t* target_of) {
  dsgd::PushArgs<T> a{};
  std::vector<uint32_t> reads;
  for (uint32_t i = 0; i < c->n_local; ++i) {
    const uint32_t me = c->first + i;
    if (gs) fill_node<T>(c, i, *gs, h, &a.node[i]);
    else {
      a.node[i].theta_in = as<T>(c->theta_ptr(i, c->cur));
      a.node[i].theta_out = as<T>(c->theta_ptr(i, c->cur ^ 1));
    }
    uint32_t n = 0;
    for (uint32_t k = 0; k < c->p; ++k) {
      if (target_of[k] == me) {
        a.senders[i][n++] = as<T>(c->peers[k].theta[c->cur]);
        reads.push_back(k);
      }
    }
    a.n_senders[i] = n;
    a.inv[i] = T(1) / T(n + 1);
  }
  if (gs) {
    fill_common(c, h, *gs, &a);
  } else {
    a.d = c->d;
  }
  a.step = gs ? 1 : 0;
  a.n_local = c->n_local;
  bool vec = gs ? all_aligned(c, *gs) : true;
  const uint64_t W = vec ? 16 / sizeof(T) : 1;
  a.blocks_per_node = blocks_for(c, c->d / W, c->n_local);
  DSGD_TRY(build_waits(c, reads, &a.wait));
  build_signal(c, &a.signal);
  LaunchScope ls(c, DSGD_K_PUSH);
  DSGD_CUDA(dsgd::launch_push<T>(a, vec, a.blocks_per_node * c->n_local, c->stream));
  if (c->distributed()) c->seq += 1;
  // WAR for the next round: my snapshot was read by my push target.
  c->prev_readers.clear();
  if (c->distributed()) c->prev_readers.push_back(target_of[c->first]);
  return DSGD_OK;
}

template <typename F>
dsgd_status dispatch(dsgd_ctx* c, F&& f) {
  DeviceGuard g(c->device);
  if (c->dtype == DSGD_F32) return f(float{});
  return f(double{});
}

dsgd_status ensure_staging(dsgd_ctx* c) {
  if (!c->staging) DSGD_CUDA(cudaMallocHost(&c->staging, c->d * 4));
  return DSGD_OK;
}

dsgd_status upload_vec(dsgd_ctx* c, char* dst, const double* host) {
  if (c->dtype == DSGD_F64) {
    DSGD_CUDA(cudaMemcpyAsync(dst, host, c->d * 8, cudaMemcpyHostToDevice, c->stream));
    DSGD_CUDA(cudaStreamSynchronize(c->stream));
    return DSGD_OK;
  }
  DSGD_TRY(ensure_staging(c));
  float* st = reinterpret_cast<float*>(c->staging);
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  for (uint64_t k = 0; k < c->d; ++k) st[k] = (float)host[k];
  DSGD_CUDA(cudaMemcpyAsync(dst, st, c->d * 4, cudaMemcpyHostToDevice, c->stream));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  return DSGD_OK;
}

dsgd_status download_vec(dsgd_ctx* c, const char* src, double* host) {
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  if (c->dtype == DSGD_F64) {
    DSGD_CUDA(cudaMemcpy(host, src, c->d * 8, cudaMemcpyDeviceToHost));
    return DSGD_OK;
  }
  DSGD_TRY(ensure_staging(c));
  float* st = reinterpret_cast<float*>(c->staging);
  DSGD_CUDA(cudaMemcpy(st, src, c->d * 4, cudaMemcpyDeviceToHost));
  for (uint64_t k = 0; k < c->d; ++k) host[k] = (double)st[k];
  return DSGD_OK;
}

char* buffer_of(dsgd_ctx* c, uint32_t local, dsgd_buffer which) {
  switch (which) {
    case DSGD_BUF_THETA: return c->theta_ptr(local, c->cur);
    case DSGD_BUF_DELTA: return c->delta[local];
    case DSGD_BUF_GRAD: return c->grad[local];
    case DSGD_BUF_NOISE: return c->noise[local];
    case DSGD_BUF_SPECTRUM: return c->spec;
    case DSGD_BUF_OPT: return c->opt;
    case DSGD_BUF_CENTER: return (c->flags & DSGD_CTX_CENTER) ? c->arena + c->off_c_in : nullptr;
  }
  return nullptr;
}

// One local node, in place, against an arbitrary device vector: the
// reference's single-node gossip rules (protocols.hpp:124-139).
template <typename T>
dsgd_status node_step(dsgd_ctx* c, int mode, const dsgd_hyperparams* h, const GradSel* gs,
                      uint32_t i, const void* partner, T beta) {
  dsgd::StepArgs<T> a{};
  GradSel none;
  none.quad = 1;
  const GradSel& g = gs ? *gs : none;
  fill_node<T>(c, i, g, h, &a.node[0]);
  a.node[0].theta_out = as<T>(c->theta_ptr(i, c->cur));  // each element read, then written
  a.node[0].partner = static_cast<const T*>(partner);
  if (gs) {
    if (!gs->quad) a.node[0].grad = static_cast<const T*>(gs->grad[i]);
    if (gs->noise) a.node[0].noise = as<T>(c->noise[i]);
    a.node[0].norm = gs->norm ? c->norm + (size_t)c->norm_slot * c->n_local : nullptr;
    fill_common(c, h, *gs, &a);
  } else {
    a.d = c->d;
  }
  a.beta = beta;
  a.n_local = 1;
  const bool vec = aligned16(partner) && (g.quad || aligned16(g.grad[i]));
  const uint64_t W = vec ? 16 / sizeof(T) : 1;
  a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
  LaunchScope ls(c, DSGD_K_STEP);
  DSGD_CUDA(dsgd::launch_step<T>(mode, a, vec, a.blocks_per_node, c->stream));
  return DSGD_OK;
}

// ------------------------------------------------ NVLS set-up (library-owned)
// The two-shot all-reduce runs its reduce in the NVSwitch when the requested
// backend is "nvls" (the default for p > 2 outside the one-shot's small-d
// range) and every GPU of the group joins one multicast object.
bool wants_nvls(const dsgd_ctx* c) {
  return c->distributed() && c->p2p_allreduce && !c->ar_oneshot && c->ar_mode == "nvls";
}

size_t nvls_half(const dsgd_ctx* c) { return align_up(c->d * c->es, size_t(1) << 21); }
size_t nvls_bytes(const dsgd_ctx* c) { return 2 * nvls_half(c); }

void attach_nvls(dsgd_ctx* c, char* x, char* x_mc, char* avg, char* avg_mc) {
  c->peers[c->first].x = x;      // kernel 1 writes here (unicast)
  c->peers[c->first].avg = avg;  // next round / flush read here
  c->nvls_x_mc = x_mc;
  c->nvls_avg_mc = avg_mc;
  c->p2p_allreduce = true;
  c->ar_oneshot = false;
  c->ar_nvls = true;
  c->nvls_note.clear();
  // reduce CTAs on SMs of their own (1024 threads, padded smem) and a wider
  // delta grid: 271.5 vs 328.7 us/round at p = 4, d = 25M
  // (profiles/r1_tune_allreduce_n4.md).  Per-worker size table measured at
  // p = 4 (profiles/r2_split_n4.md): 1.5 / 0.5 CTAs per SM up to ~200M, 1.25
  // / 0.75 from there to ~700M, 1.5 / 0.5 with 4 pipelines above (see
  // ar_pipes_for).  p = 8 runs the same table (no 8-GPU box measured it).
  // The environment still overrides.
  const bool mid = c->d >= (200ull << 20) && c->d < (700ull << 20);
  if (!std::getenv("DSGD_AR_DELTA_FRAC")) c->ar_delta_frac = mid ? 1.25 : 1.5;
  if (!std::getenv("DSGD_AR_COMM_FRAC")) c->ar_comm_frac = mid ? 0.75 : 0.5;
}

void attach_mc_state(dsgd_ctx* c) {
  char* uc = reinterpret_cast<char*>(c->mc.uc);
  char* mc = reinterpret_cast<char*>(c->mc.mcva);
  const size_t half = nvls_half(c);
  attach_nvls(c, uc, mc, uc + half, mc + half);
}

// Connect-time agreement of one-process-per-GPU ranks over the already
// mapped peer memory: every rank posts (phase, ok) into rank 0's slots and
// waits until all posted phase `phase`; *all_ok tells whether every rank
// succeeded.  (A rank that posted a later phase passed this one.)
dsgd_status host_barrier(dsgd_ctx* c, uint32_t phase, bool ok, bool* all_ok) {
  unsigned long long* slots = c->peers[0].hb;
  if (!slots) return set_error(DSGD_ESTATE, "no barrier slots");
  const unsigned long long v = ((unsigned long long)phase << 8) | (ok ? 1u : 2u);
  DSGD_CUDA(cudaMemcpy(slots + c->first, &v, sizeof(v), cudaMemcpyDefault));
  std::vector<unsigned long long> got(c->p);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    DSGD_CUDA(cudaMemcpy(got.data(), slots, sizeof(v) * c->p, cudaMemcpyDefault));
    bool done = true, good = true;
    for (unsigned long long g : got) {
      const unsigned long long ph = g >> 8;
      if (ph < phase) done = false;
      else if (ph == phase && (g & 0xff) != 1) good = false;
    }
    if (done) {
      *all_ok = good;
      return DSGD_OK;
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
      return set_error(DSGD_ETIMEOUT, "a peer never reached the NVLS set-up barrier");
    usleep(100);
  }
}

// Every rank joins rank 0's multicast object: import (pidfd_getfd) ->
// barrier -> add this GPU -> barrier -> back it, bind and map -> barrier.
// Any failure anywhere leaves every rank on the peer-memory two-shot.
dsgd_status join_nvls(dsgd_ctx* c, const HandleBlob& b0) {
  bool ok = true, all = false;
  if (c->first != 0) {
    ok = dsgd::mc_import_fd(&c->mc, b0.mc_pid, b0.mc_fd, b0.mc_size) == DSGD_OK;
    if (!ok) c->nvls_note = dsgd::g_error;
  }
  DSGD_TRY(host_barrier(c, 1, ok, &all));
  if (c->mc.export_fd >= 0) {  // rank 0: everybody holds its own handle now
    close(c->mc.export_fd);
    c->mc.export_fd = -1;
  }
  if (all) {
    ok = dsgd::mc_add_device(&c->mc, c->device) == DSGD_OK;
    if (!ok) c->nvls_note = dsgd::g_error;
    DSGD_TRY(host_barrier(c, 2, ok, &all));
  }
  if (all) {
    ok = dsgd::mc_bind_map(&c->mc, c->device, true) == DSGD_OK;
    if (!ok) c->nvls_note = dsgd::g_error;
    DSGD_TRY(host_barrier(c, 3, ok, &all));
  }
  if (!all) {
    if (c->nvls_note.empty()) c->nvls_note = "a peer could not join the multicast object";
    dsgd::mc_release(&c->mc, c->device);
    return DSGD_OK;
  }
  attach_mc_state(c);
  return DSGD_OK;
}

// In-process group on distinct GPUs: one object, every GPU added by this
// thread before any backing is bound.
dsgd_status inproc_nvls(InprocGroup* g) {
  dsgd_ctx* c0 = g->ctx[0];
  for (dsgd_ctx* c : g->ctx) {
    if (!wants_nvls(c)) return DSGD_OK;
    for (dsgd_ctx* o : g->ctx)
      if (o != c && o->device == c->device) return DSGD_OK;  // ranks sharing a GPU
    if (!dsgd::mc_supported(c->device)) {
      for (dsgd_ctx* o : g->ctx) o->nvls_note = "a GPU reports no multicast (NVLS) support";
      return DSGD_OK;
    }
  }
  dsgd_status st;
  {
    DeviceGuard dg(c0->device);
    st = dsgd::mc_create(&c0->mc, c0->device, c0->p, nvls_bytes(c0), false);
  }
  for (dsgd_ctx* c : g->ctx) {
    if (st != DSGD_OK) break;
    if (c != c0) dsgd::mc_share(&c->mc, &c0->mc);
    DeviceGuard dg(c->device);
    st = dsgd::mc_add_device(&c->mc, c->device);
  }
  for (dsgd_ctx* c : g->ctx) {
    if (st != DSGD_OK) break;
    DeviceGuard dg(c->device);
    st = dsgd::mc_bind_map(&c->mc, c->device, false);
  }
  if (st != DSGD_OK) {
    const std::string why = dsgd::g_error;
    for (auto it = g->ctx.rbegin(); it != g->ctx.rend(); ++it) {  // owner last
      DeviceGuard dg((*it)->device);
      dsgd::mc_release(&(*it)->mc, (*it)->device);
      (*it)->nvls_note = why;
    }
    return DSGD_OK;
  }
  for (dsgd_ctx* c : g->ctx) attach_mc_state(c);
  return DSGD_OK;
}

}  // namespace

extern "C" {

const char* dsgd_last_error(void) { return dsgd::g_error.c_str(); }
int dsgd_abi_version(void) { return DSGD_B200_ABI_VERSION; }

dsgd_status dsgd_ctx_create(const dsgd_ctx_desc* desc, dsgd_ctx** out) {
  if (!desc || !out) return set_error(DSGD_EINVAL, "null argument");
  if (desc->dim == 0) return set_error(DSGD_EINVAL, "dim must be >= 1");
  if (desc->p == 0 || desc->n_local == 0 || desc->n_local > (uint32_t)kMaxLocal ||
      desc->first_node + desc->n_local > desc->p)
    return set_error(DSGD_EINVAL, "bad node layout (p, first_node, n_local)");
  if (desc->n_local != desc->p && desc->n_local != 1)
    return set_error(DSGD_EINVAL, "a context hosts all p nodes or exactly one");
  if (desc->n_local < desc->p && desc->p > (uint32_t)kMaxWait)
    return set_error(DSGD_EINVAL, "one node per context supports p <= 16");
  if (desc->dtype != DSGD_F32 && desc->dtype != DSGD_F64) return set_error(DSGD_EINVAL, "dtype");
  auto c = std::make_unique<dsgd_ctx>();
  c->device = desc->device;
  c->d = desc->dim;
  c->dtype = desc->dtype;
  c->es = desc->dtype == DSGD_F32 ? 4 : 8;
  c->p = desc->p;
  c->first = desc->first_node;
  c->n_local = desc->n_local;
  c->flags = desc->flags;
  c->t.assign(c->n_local, 0);
  DeviceGuard g(c->device);
  DSGD_CUDA(cudaSetDevice(c->device));
  DSGD_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
  if (const char* e = std::getenv("DSGD_BLOCKS_PER_SM")) c->blocks_per_sm = std::max(1, atoi(e));
  if (const char* e = std::getenv("DSGD_EA_CHUNK"))
    c->ea_chunk = std::max<uint64_t>(1, strtoull(e, nullptr, 10) / dsgd::kEaChunk) * dsgd::kEaChunk;
  if (desc->stream) {
    c->stream = static_cast<cudaStream_t>(desc->stream);
  } else {
    DSGD_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  const size_t vb = align_up(c->d * c->es);
  size_t off = 0;
  for (uint32_t i = 0; i < c->n_local; ++i)
    for (int b = 0; b < 2; ++b) {
      c->off_theta[i][b] = off;
      off += vb;
    }
  c->n_chunks = (c->d + dsgd::kEaChunk - 1) / dsgd::kEaChunk;
  c->off_c_in = off;
  if (c->flags & DSGD_CTX_CENTER) off += vb;
  c->off_flags = off;
  if (c->flags & DSGD_CTX_CENTER) off += align_up(c->n_chunks * 8);
  c->off_round = off;
  off += align_up(8 * c->n_local);
  if (c->n_local < c->p) {  // one node per context: peer-memory all-reduce buffers
    c->off_x = off;
    off += vb;
    c->off_a = off;
    off += vb;
    c->off_ar = off;
    off += 256;
    c->off_x2 = off;
    off += vb;
    c->off_hb = off;
    off += 256;
  }
  c->arena_bytes = off;
  // multi-GPU all-reduce backend: oneshot (default p <= 2), p2p (two-shot,
  // default p > 2), nccl
  {
    // one kernel per round wins at p <= 2, and at p <= 4 while d is latency-bound
    // (nvls falls back to the peer-memory two-shot "p2p" when the GPUs
    // cannot join a multicast object)
    std::string mode = (c->p <= 2 || (c->p <= 4 && c->d < (4u << 20))) ? "oneshot" : "nvls";
    if (const char* e = std::getenv("DSGD_ALLREDUCE")) mode = e;
    if (mode == "p2p2k") mode = "p2p";
    c->ar_mode = mode;
    c->p2p_allreduce = mode != "nccl";
    c->ar_oneshot = mode == "oneshot" && c->p <= 4;
  }
  if (const char* e = std::getenv("DSGD_AR_TMA")) c->ar_tma = atoi(e) != 0;
  if (const char* e = std::getenv("DSGD_TRACE")) {
    c->trace_cap = (uint32_t)std::max(1, atoi(e));
    if (c->trace_cap < 64) c->trace_cap = 65536;
  }
  if (const char* e = std::getenv("DSGD_AR_PIPES")) {
    c->ar_pipes = (uint32_t)std::min(4, std::max(1, atoi(e)));
    c->ar_pipes_env = true;
  }
  if (const char* e = std::getenv("DSGD_AR_DELTA_FRAC")) c->ar_delta_frac = std::max(0.05, atof(e));
  if (const char* e = std::getenv("DSGD_AR_COMM_FRAC")) c->ar_comm_frac = std::max(0.05, atof(e));

  DSGD_CUDA(cudaMalloc(&c->arena, c->arena_bytes));
  DSGD_CUDA(cudaMemset(c->arena, 0, c->arena_bytes));
  for (uint32_t i = 0; i < c->n_local; ++i) {
    DSGD_CUDA(cudaMalloc(&c->delta[i], vb));
    DSGD_CUDA(cudaMemset(c->delta[i], 0, vb));
    if (c->flags & DSGD_CTX_GRAD) {
      DSGD_CUDA(cudaMalloc(&c->grad[i], vb));
      DSGD_CUDA(cudaMemset(c->grad[i], 0, vb));
    }
    if (c->flags & DSGD_CTX_NOISE) {
      DSGD_CUDA(cudaMalloc(&c->noise[i], vb));
      DSGD_CUDA(cudaMemset(c->noise[i], 0, vb));
    }
  }
  if (c->flags & DSGD_CTX_QUADRATIC) {
    DSGD_CUDA(cudaMalloc(&c->spec, vb));
    DSGD_CUDA(cudaMalloc(&c->opt, vb));
    DSGD_CUDA(cudaMemset(c->spec, 0, vb));
    DSGD_CUDA(cudaMemset(c->opt, 0, vb));
  }
  {
    const size_t nb = sizeof(double) * dsgd::kNormSlots * c->n_local;
    DSGD_CUDA(cudaMalloc(&c->norm, nb));
    DSGD_CUDA(cudaMemset(c->norm, 0, nb));
    DSGD_CUDA(cudaMalloc(&c->norm_max, sizeof(double) * 8));
    DSGD_CUDA(cudaMemset(c->norm_max, 0, sizeof(double) * 8));
    c->scratch = c->norm_max + 4;
  }
  DSGD_CUDA(cudaMallocHost(&c->norm_host, sizeof(double) * kMaxLocal));
  DSGD_CUDA(cudaMalloc(&c->arrive, 256));
  DSGD_CUDA(cudaMemset(c->arrive, 0, 256));
  DSGD_CUDA(cudaMalloc(&c->lt_flags, sizeof(unsigned long long) * 4096));
  DSGD_CUDA(cudaMemset(c->lt_flags, 0, sizeof(unsigned long long) * 4096));
  if (c->trace_cap) {
    DSGD_CUDA(cudaMalloc(&c->trace_dev, sizeof(unsigned long long) * 3 * c->trace_cap));
    DSGD_CUDA(cudaMemset(c->trace_dev, 0, sizeof(unsigned long long) * 3 * c->trace_cap));
  }
  if (c->n_local < c->p) {
    for (int h = 0; h < 4; ++h)
      DSGD_CUDA(cudaStreamCreateWithFlags(&c->pipe_stream[h], cudaStreamNonBlocking));
    for (int h = 0; h < 9; ++h)
      DSGD_CUDA(cudaEventCreateWithFlags(&c->pipe_event[h], cudaEventDisableTiming));
  }
  c->error = c->arrive + 32;
  // local nodes are addressable peers of themselves
  c->peers.resize(c->p);
  for (uint32_t i = 0; i < c->n_local; ++i) {
    PeerNode& pn = c->peers[c->first + i];
    pn.theta[0] = c->theta_ptr(i, 0);
    pn.theta[1] = c->theta_ptr(i, 1);
    pn.round = c->round_ptr(i);
    if (c->off_x) {
      pn.x = c->arena + c->off_x;
      pn.avg = c->arena + c->off_a;
      pn.ar = reinterpret_cast<unsigned long long*>(c->arena + c->off_ar);
      pn.x2 = c->arena + c->off_x2;
      pn.hb = reinterpret_cast<unsigned long long*>(c->arena + c->off_hb);
    }
    if (i == 0 && (c->flags & DSGD_CTX_CENTER)) {
      pn.c_in = c->arena + c->off_c_in;
      pn.flags = reinterpret_cast<unsigned long long*>(c->arena + c->off_flags);
    }
  }
  c->connected = !c->distributed();
  *out = c.release();
  return DSGD_OK;
}

void dsgd_ctx_destroy(dsgd_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  dsgd::mc_release(&c->mc, c->device);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  for (uint32_t i = 0; i < c->n_local; ++i) {
    cudaFree(c->delta[i]);
    cudaFree(c->grad[i]);
    cudaFree(c->noise[i]);
    cudaFree(c->aux[i]);
  }
  cudaFree(c->spec);
  cudaFree(c->opt);
  cudaFree(c->norm);
  cudaFree(c->norm_max);
  cudaFreeHost(c->norm_host);
  cudaFree(c->arrive);
  cudaFree(c->lt_flags);
  cudaFree(c->trace_dev);
  cudaFreeHost(c->staging);
  cudaFree(c->arena);
  for (auto* s : c->partner_streams) dsgd_stream_destroy(s);
  for (auto* s : c->noise_streams) dsgd_stream_destroy(s);
  for (auto* s : c->sample_streams) dsgd_stream_destroy(s);
  if (c->clock_stream) dsgd_stream_destroy(c->clock_stream);
  delete[] c->noise_host;
  cudaFree(c->lg_X);
  cudaFree(c->lg_y);
  cudaFree(c->lg_rows);
  cudaFree(c->lg_scratch);
  for (int k = 0; k < 4; ++k) {
    cudaFreeHost(c->lg_pin[k]);
    if (c->lg_ev[k]) cudaEventDestroy(c->lg_ev[k]);
  }
  for (const Prof& p : c->prof_pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  for (int h = 0; h < 4; ++h)
    if (c->pipe_stream[h] && c->pipe_stream[h] != c->stream) {
      cudaStreamSynchronize(c->pipe_stream[h]);
      cudaStreamDestroy(c->pipe_stream[h]);
    }
  for (int h = 0; h < 9; ++h)
    if (c->pipe_event[h]) cudaEventDestroy(c->pipe_event[h]);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

dsgd_status dsgd_ctx_stream(dsgd_ctx* c, void** stream) {
  DSGD_TRY(check_ctx(c));
  *stream = c->stream;
  return DSGD_OK;
}

dsgd_status dsgd_ctx_sync(dsgd_ctx* c) {
  DSGD_TRY(check_ctx(c));
  DeviceGuard g(c->device);
  DSGD_TRY(norm_read(c));
  DSGD_TRY(join_pipes(c));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  unsigned int err = 0;
  DSGD_CUDA(cudaMemcpy(&err, c->error, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) return set_error(DSGD_ETIMEOUT, "a peer flag wait timed out inside a kernel");
  return DSGD_OK;
}

dsgd_status dsgd_grad_norm_flush(dsgd_ctx* c) {
  DSGD_TRY(check_ctx(c));
  DeviceGuard g(c->device);
  return norm_read(c);
}

dsgd_status dsgd_ctx_set_timeout(dsgd_ctx* c, double seconds) {
  DSGD_TRY(check_ctx(c));
  if (!(seconds > 0)) return set_error(DSGD_EINVAL, "timeout must be positive");
  c->timeout_ns = (unsigned long long)(seconds * 1e9);
  return DSGD_OK;
}

dsgd_status dsgd_buffer_ptr(dsgd_ctx* c, uint32_t local, dsgd_buffer which, void** dev) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  *dev = p;
  return DSGD_OK;
}

dsgd_status dsgd_set_state(dsgd_ctx* c, uint32_t local, const double* theta,
                           const double* delta_prev, uint64_t t) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  DeviceGuard g(c->device);
  if (theta) DSGD_TRY(upload_vec(c, c->theta_ptr(local, c->cur), theta));
  if (delta_prev) DSGD_TRY(upload_vec(c, c->delta[local], delta_prev));
  c->t[local] = t;
  return DSGD_OK;
}

dsgd_status dsgd_get_state(dsgd_ctx* c, uint32_t local, double* theta, double* delta_prev,
                           uint64_t* t) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  DeviceGuard g(c->device);
  DSGD_TRY(dsgd_ctx_sync(c));
  if (theta) DSGD_TRY(download_vec(c, c->theta_ptr(local, c->cur), theta));
  if (delta_prev) DSGD_TRY(download_vec(c, c->delta[local], delta_prev));
  if (t) *t = c->t[local];
  return DSGD_OK;
}

dsgd_status dsgd_set_vector(dsgd_ctx* c, uint32_t local, dsgd_buffer which, const double* host) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  DeviceGuard g(c->device);
  return upload_vec(c, p, host);
}

dsgd_status dsgd_set_logistic(dsgd_ctx* c, const double* features, const int32_t* labels,
                              uint64_t n_samples, double l2) {
  DSGD_TRY(check_ctx(c));
  // the LogisticObjective constructor's checks, objectives.cpp:83-101
  if (n_samples == 0 || !features || !labels)
    return set_error(DSGD_EINVAL, "logistic dataset is empty");
  if (!(l2 > 0.0))
    return set_error(DSGD_EINVAL, "logistic l2 must be positive (strong convexity)");
  for (uint64_t r = 0; r < n_samples; ++r)
    if (labels[r] != 0 && labels[r] != 1)
      return set_error(DSGD_EINVAL, "logistic labels must be 0 or 1");
  DeviceGuard g(c->device);
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  const size_t vb = c->d * c->es;
  for (uint32_t i = 0; i < c->n_local; ++i)
    if (!c->grad[i]) {  // the produced gradient lands in the node's gradient buffer
      DSGD_CUDA(cudaMalloc(&c->grad[i], vb));
      DSGD_CUDA(cudaMemset(c->grad[i], 0, vb));
    }
  cudaFree(c->lg_X);
  cudaFree(c->lg_y);
  c->lg_X = nullptr;
  c->lg_y = nullptr;
  DSGD_CUDA(cudaMalloc(&c->lg_X, n_samples * vb));
  DSGD_CUDA(cudaMalloc(&c->lg_y, n_samples * sizeof(int32_t)));
  if (c->dtype == DSGD_F64) {
    DSGD_CUDA(cudaMemcpy(c->lg_X, features, n_samples * vb, cudaMemcpyHostToDevice));
  } else {  // the context dtype: round each feature to fp32 once, on the host
    std::vector<float> f32(n_samples * c->d);
    for (size_t k = 0; k < f32.size(); ++k) f32[k] = (float)features[k];
    DSGD_CUDA(cudaMemcpy(c->lg_X, f32.data(), n_samples * vb, cudaMemcpyHostToDevice));
  }
  DSGD_CUDA(cudaMemcpy(c->lg_y, labels, n_samples * sizeof(int32_t), cudaMemcpyHostToDevice));
  c->lg_n = n_samples;
  c->lg_l2 = l2;
  c->lg_begin.assign(c->n_local, 0);
  c->lg_end.assign(c->n_local, n_samples);
  return DSGD_OK;
}

dsgd_status dsgd_logistic_set_sample_range(dsgd_ctx* c, uint32_t local, uint64_t begin,
                                           uint64_t end) {
  DSGD_TRY(check_ctx(c));
  if (!c->lg_X) return set_error(DSGD_ESTATE, "no logistic dataset (dsgd_set_logistic)");
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  if (begin >= end || end > c->lg_n) return set_error(DSGD_EINVAL, "invalid sample range");
  c->lg_begin[local] = begin;
  c->lg_end[local] = end;
  return DSGD_OK;
}

// Rank 0 of a multi-GPU EASGD chain holds the center in its c_in, written
// chunk by chunk by rank p-1's last gated round: wait (on the device,
// bounded) until every chunk of that round has arrived.
// (enqueue only: the context stream waits on the device)
dsgd_status center_wait_enqueue(dsgd_ctx* c) {
  if (!c->distributed() || c->first != 0 || c->ea_seq == 0 || !c->connected) return DSGD_OK;
  const uint64_t n = (c->d + c->ea_chunk_used - 1) / c->ea_chunk_used;
  DSGD_CUDA(dsgd::launch_wait_chunks(reinterpret_cast<const unsigned long long*>(c->arena + c->off_flags),
                                     n, c->ea_seq, c->timeout_ns, c->error, c->stream));
  return DSGD_OK;
}

dsgd_status center_arrived(dsgd_ctx* c) {
  if (!c->distributed() || c->first != 0 || c->ea_seq == 0 || !c->connected) return DSGD_OK;
  DSGD_TRY(center_wait_enqueue(c));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  unsigned int err = 0;
  DSGD_CUDA(cudaMemcpy(&err, c->error, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) return set_error(DSGD_ETIMEOUT, "the EASGD center never arrived from the last rank");
  return DSGD_OK;
}

dsgd_status dsgd_get_vector(dsgd_ctx* c, uint32_t local, dsgd_buffer which, double* host) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  DeviceGuard g(c->device);
  if (which == DSGD_BUF_CENTER) DSGD_TRY(center_arrived(c));
  return download_vec(c, p, host);
}

dsgd_status dsgd_upload_async(dsgd_ctx* c, uint32_t local, dsgd_buffer which, const void* host,
                              uint64_t count) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local || count > c->d) return set_error(DSGD_EINVAL, "range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  DeviceGuard g(c->device);
  DSGD_CUDA(cudaMemcpyAsync(p, host, count * c->es, cudaMemcpyHostToDevice, c->stream));
  return DSGD_OK;
}

dsgd_status dsgd_download_async(dsgd_ctx* c, uint32_t local, dsgd_buffer which, void* host,
                                uint64_t count) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local || count > c->d) return set_error(DSGD_EINVAL, "range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  DeviceGuard g(c->device);
  if (which == DSGD_BUF_CENTER) DSGD_TRY(center_wait_enqueue(c));  // as dsgd_get_vector
  DSGD_CUDA(cudaMemcpyAsync(host, p, count * c->es, cudaMemcpyDeviceToHost, c->stream));
  return DSGD_OK;
}

dsgd_status dsgd_copy_in_async(dsgd_ctx* c, uint32_t local, dsgd_buffer which, const void* src,
                               uint64_t count) {
  DSGD_TRY(check_ctx(c));
  if (which == DSGD_BUF_THETA || which == DSGD_BUF_DELTA) DSGD_TRY(flush_pending(c));
  if (local >= c->n_local || count > c->d || !src) return set_error(DSGD_EINVAL, "range");
  char* p = buffer_of(c, local, which);
  if (!p) return set_error(DSGD_ESTATE, "buffer not allocated for this context");
  DeviceGuard g(c->device);
  DSGD_CUDA(cudaMemcpyAsync(p, src, count * c->es, cudaMemcpyDefault, c->stream));
  return DSGD_OK;
}

dsgd_status dsgd_get_t(dsgd_ctx* c, uint32_t local, uint64_t* t) {
  DSGD_TRY(check_ctx(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  *t = c->t[local];
  return DSGD_OK;
}

dsgd_status dsgd_set_t(dsgd_ctx* c, uint32_t local, uint64_t t) {
  DSGD_TRY(check_ctx(c));
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  c->t[local] = t;
  return DSGD_OK;
}

// ----------------------------------------------------------- update rules
dsgd_status dsgd_local_sgd_step(dsgd_ctx* c, const dsgd_hyperparams* h, const dsgd_grad_spec* g) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
    DSGD_TRY(do_local_step<T>(c, h, gs));
    finish_round(c, true);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_allreduce_round(dsgd_ctx* c, const dsgd_hyperparams* h, const dsgd_grad_spec* g,
                                 dsgd_momentum_scope scope) {
  DSGD_TRY(check_ctx(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_common_round(c));
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  if (gs.logistic) DSGD_TRY(flush_pending(c));  // the gradient reads the applied theta
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
    DSGD_TRY(do_allreduce<T>(c, h, gs, scope));
    finish_round(c, !c->distributed());  // multi-GPU: do_allreduce tracks the buffers
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_ea_round(dsgd_ctx* c, const dsgd_hyperparams* h, const dsgd_grad_spec* g,
                          int gated) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    if (gs.logistic && gated) {
      // client/server half, then the minibatch gradient at the moved theta,
      // then the step (ea_client_step protocols.cpp:146-151)
      DSGD_TRY(do_ea<T>(c, h, gs, gated, true));
      finish_round(c, true, false);
      c->rounds_done -= 1;
      DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
      DSGD_TRY(do_local_step<T>(c, h, gs));
    } else {
      DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
      DSGD_TRY(do_ea<T>(c, h, gs, gated));
    }
    finish_round(c, true);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_pull_gossip_round(dsgd_ctx* c, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, const uint32_t* partner_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_common_round(c));
  if (partner_of) DSGD_TRY(check_map(c, partner_of));
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    if (partner_of && gs.logistic) {
      // pull_mix, then the minibatch gradient at the mixed theta, then the
      // step (protocols.cpp:173-185)
      DSGD_TRY(do_pull<T>(c, nullptr, gs, partner_of, dsgd::kModeMix, T(0.5)));
      finish_round(c, true, false);
      c->rounds_done -= 1;
      DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
      DSGD_TRY(do_local_step<T>(c, h, gs));
    } else if (partner_of) {
      DSGD_TRY(do_pull<T>(c, h, gs, partner_of, dsgd::kModePull, T(0.5)));
    } else {
      DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
      DSGD_TRY(do_local_step<T>(c, h, gs));
    }
    finish_round(c, true);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_push_gossip_round(dsgd_ctx* c, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, const uint32_t* target_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_common_round(c));
  DSGD_TRY(check_map(c, target_of));
  for (uint32_t k = 0; k < c->p; ++k)
    if (target_of[k] == k) return set_error(DSGD_EINVAL, "push target must differ from sender");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    if (gs.logistic) {  // push_mix, gradient at the mixed theta, step (230-242)
      DSGD_TRY(do_push<T>(c, nullptr, nullptr, target_of));
      finish_round(c, true, false);
      c->rounds_done -= 1;
      DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
      DSGD_TRY(do_local_step<T>(c, h, gs));
    } else {
      DSGD_TRY(do_push<T>(c, h, &gs, target_of));
    }
    finish_round(c, true);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_gossip_stale_round(dsgd_ctx* c, const dsgd_hyperparams* h,
                                    const dsgd_grad_spec* g, const uint32_t* partner_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_map(c, partner_of));
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
    DSGD_TRY(do_pull<T>(c, h, gs, partner_of, dsgd::kModeStale, (T)h->beta_gossip));
    finish_round(c, true);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_gossip_fresh_round(dsgd_ctx* c, const dsgd_hyperparams* h,
                                    const dsgd_grad_spec* g, const uint32_t* partner_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_map(c, partner_of));
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    // every node steps (theta' into the other buffer), then mixes with the
    // partner's post-step theta' (simulator.cpp:305-319)
    DSGD_TRY(produce_logistic<T>(c, h, gs, all_local(c), true));
    DSGD_TRY(do_local_step<T>(c, h, gs));
    finish_round(c, true, true);
    c->rounds_done -= 1;
    if (c->grp && c->distributed()) {
      // in-process group: the mix reads the partner's post-step theta of this
      // round, so every rank's step is issued before any mix; the last rank
      // issues the mixes of all ranks, in rank order
      c->fresh_map.assign(partner_of, partner_of + c->p);
      c->fresh_beta = h->beta_gossip;
      if (c->first + 1 == c->p)
        for (dsgd_ctx* r : c->grp->ctx) {
          DeviceGuard dg(r->device);
          GradSel none;
          none.quad = 1;
          DSGD_TRY(do_pull<T>(r, nullptr, none, r->fresh_map.data(), dsgd::kModeMix,
                              (T)r->fresh_beta));
          finish_round(r, true, false);
        }
      return norm_end(c, gs, g);
    }
    DSGD_TRY(do_pull<T>(c, nullptr, gs, partner_of, dsgd::kModeMix, (T)h->beta_gossip));
    finish_round(c, true, false);
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_async_pull_event(dsgd_ctx* c, const dsgd_hyperparams* h,
                                  const dsgd_grad_spec* g, uint32_t i, uint32_t j) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (c->distributed()) return set_error(DSGD_EINVAL, "async-pull runs on a single context");
  if (i >= c->p || j >= c->p)
    return set_error(DSGD_EINVAL, "async_pull_event node index out of range");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    // model_gradient at theta_i itself (protocols.cpp:287: no lookahead)
    DSGD_TRY(produce_logistic<T>(c, h, gs, {i}, false));
    // in place on node i (only node i changes; j == i reads the pre-event value)
    dsgd::StepArgs<T> a{};
    fill_node<T>(c, i, gs, h, &a.node[0], true);
    a.node[0].theta_out = as<T>(c->theta_ptr(i, c->cur));
    a.node[0].partner = as<T>(c->theta_ptr(j, c->cur));
    a.node[0].norm = gs.norm ? c->norm + (size_t)c->norm_slot * c->n_local : nullptr;
    fill_common(c, h, gs, &a);
    a.beta = (T)h->beta_gossip;
    a.n_local = 1;
    const bool vec = (gs.quad || aligned16(gs.grad[i]));
    if (!gs.quad) a.node[0].grad = static_cast<const T*>(gs.grad[i]);
    if (gs.noise) a.node[0].noise = as<T>(c->noise[i]);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
    a.tma_partner = c->ar_tma;  // every stream staged through smem (k_step_tma2<Async>)
    {
      LaunchScope ls(c, DSGD_K_STEP);
      DSGD_CUDA(dsgd::launch_step<T>(dsgd::kModeAsync, a, vec, a.blocks_per_node, c->stream));
    }
    c->t[i] += 1;
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_gossip_stale_step(dsgd_ctx* c, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, uint32_t local, const void* partner) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (c->distributed()) return set_error(DSGD_EINVAL, "single-node rules run on a single context");
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  if (!partner) return set_error(DSGD_EINVAL, "null partner vector");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  if (gs.logistic) return set_error(DSGD_EINVAL, "single-node rules take a quadratic or buffer gradient");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    DSGD_TRY(node_step<T>(c, dsgd::kModeStale, h, &gs, local, partner, (T)h->beta_gossip));
    c->t[local] += 1;
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_eval_point(dsgd_ctx* c, const dsgd_hyperparams* h, uint32_t local, void* out) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  if (!out) return set_error(DSGD_EINVAL, "null output buffer");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    dsgd::StepArgs<T> a{};
    a.node[0].theta_in = as<T>(c->theta_ptr(local, c->cur));
    a.node[0].theta_out = static_cast<T*>(out);
    a.node[0].delta = as<T>(c->delta[local]);
    a.d = c->d;
    a.mu = (T)h->mu;
    a.mu_nz = h->mu != 0.0;
    a.n_local = 1;
    const bool vec = aligned16(out);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
    LaunchScope ls(c, DSGD_K_OTHER);
    DSGD_CUDA(dsgd::launch_step<T>(dsgd::kModeLookahead, a, vec, a.blocks_per_node, c->stream));
    return DSGD_OK;
  });
}

dsgd_status dsgd_mix_toward(dsgd_ctx* c, uint32_t local, const void* partner, double beta) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (c->distributed()) return set_error(DSGD_EINVAL, "single-node rules run on a single context");
  if (local >= c->n_local) return set_error(DSGD_EINVAL, "local node out of range");
  if (!partner) return set_error(DSGD_EINVAL, "null partner vector");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    return node_step<T>(c, dsgd::kModeMix, nullptr, nullptr, local, partner, (T)beta);
  });
}

dsgd_status dsgd_pull_mix(dsgd_ctx* c, const uint32_t* partner_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_map(c, partner_of));
  GradSel gs;
  gs.quad = 1;
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(do_pull<T>(c, nullptr, gs, partner_of, dsgd::kModeMix, T(0.5)));
    finish_round(c, true, false);
    return DSGD_OK;
  });
}

dsgd_status dsgd_push_mix(dsgd_ctx* c, const uint32_t* target_of) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_map(c, target_of));
  for (uint32_t k = 0; k < c->p; ++k)
    if (target_of[k] == k) return set_error(DSGD_EINVAL, "push target must differ from sender");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(do_push<T>(c, nullptr, nullptr, target_of));
    finish_round(c, true, false);
    return DSGD_OK;
  });
}

dsgd_status dsgd_gossip_fresh_mix(dsgd_ctx* c, const uint32_t* partner_of, double beta) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  DSGD_TRY(check_map(c, partner_of));
  GradSel gs;
  gs.quad = 1;
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(do_pull<T>(c, nullptr, gs, partner_of, dsgd::kModeMix, (T)beta));
    finish_round(c, true, false);
    return DSGD_OK;
  });
}

dsgd_status dsgd_ea_set_update_out(dsgd_ctx* c, void* const* update_out) {
  DSGD_TRY(check_ctx(c));
  for (uint32_t i = 0; i < c->n_local; ++i) c->ea_update_out[i] = update_out ? update_out[i] : nullptr;
  return DSGD_OK;
}

dsgd_status dsgd_ea_server_apply(dsgd_ctx* c, const void* update) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!(c->flags & DSGD_CTX_CENTER) || c->first != 0)
    return set_error(DSGD_ESTATE, "the server center lives on the context hosting node 0");
  if (!update) return set_error(DSGD_EINVAL, "null update");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    dsgd::StepArgs<T> a{};
    T* center = as<T>(c->arena + c->off_c_in);
    a.node[0].theta_in = center;
    a.node[0].theta_out = center;  // in place: each element read then written by one thread
    a.node[0].aux = static_cast<T*>(const_cast<void*>(update));
    a.d = c->d;
    a.n_local = 1;
    const bool vec = aligned16(update);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    a.blocks_per_node = blocks_for(c, (c->d / W + 1) / 2, 1);
    LaunchScope ls(c, DSGD_K_OTHER);
    DSGD_CUDA(dsgd::launch_step<T>(dsgd::kModeApply, a, vec, a.blocks_per_node, c->stream));
    return DSGD_OK;
  });
}

dsgd_status dsgd_ea_client_event(dsgd_ctx* c, const dsgd_hyperparams* h,
                                 const dsgd_grad_spec* g, uint32_t i, int gated) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!h) return set_error(DSGD_EINVAL, "null hyperparams");
  if (c->distributed()) return set_error(DSGD_EINVAL, "async EASGD runs on a single context");
  if (i >= c->p) return set_error(DSGD_EINVAL, "client index out of range");
  if (!(c->flags & DSGD_CTX_CENTER)) return set_error(DSGD_ESTATE, "no center (DSGD_CTX_CENTER)");
  GradSel gs;
  DSGD_TRY(resolve_grad(c, g, &gs));
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    DSGD_TRY(norm_begin(c, gs, g));
    dsgd::EaArgs<T> a{};
    fill_node<T>(c, i, gs, h, &a.node[0]);
    a.node[0].theta_out = as<T>(c->theta_ptr(i, c->cur));  // in place: only node i moves
    a.node[0].aux = static_cast<T*>(c->ea_update_out[i]);  // ea_client_step's update
    if (!gs.quad) a.node[0].grad = static_cast<const T*>(gs.grad[i]);
    a.node[0].noise = gs.noise ? as<T>(c->noise[i]) : nullptr;
    a.node[0].norm = gs.norm ? c->norm + (size_t)c->norm_slot * c->n_local : nullptr;
    fill_common(c, h, gs, &a);
    a.center = as<T>(c->arena + c->off_c_in);
    a.beta = (T)h->beta_ea;
    a.gated = gated;
    a.p = 1;
    const bool vec = gs.quad || aligned16(gs.grad[i]);
    const uint64_t W = vec ? 16 / sizeof(T) : 1;
    if (gs.logistic && gated) {  // client/server half in place, then the gradient
      LaunchScope ls(c, DSGD_K_EA);
      DSGD_CUDA(dsgd::launch_ea_local<T>(a, 0, 0, blocks_for(c, c->d, 1), c->stream, true));
      a.gated = 0;
    }
    DSGD_TRY(produce_logistic<T>(c, h, gs, {i}, true));
    {
      LaunchScope ls(c, DSGD_K_EA);
      DSGD_CUDA(dsgd::launch_ea_local<T>(a, vec, gs.norm, blocks_for(c, c->d / W, 1), c->stream));
    }
    c->t[i] += 1;
    return norm_end(c, gs, g);
  });
}

dsgd_status dsgd_trace(dsgd_ctx* c, double* sq_err_consensus, double* loss_mean,
                       double* sq_err_opt) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
  if (c->p > (uint32_t)kMaxLocal) return set_error(DSGD_EINVAL, "trace supports p <= 32");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    dsgd::TraceArgs<T> a{};
    for (uint32_t k = 0; k < c->p; ++k) a.x[k] = as<T>(c->peers[k].theta[c->cur]);
    a.spec = c->spec ? as<T>(c->spec) : nullptr;
    a.opt = c->spec ? as<T>(c->opt) : nullptr;
    a.p = c->p;
    a.d = c->d;
    a.out = c->scratch;
    // every peer's current theta is final once its last launch published
    DSGD_TRY(all_peer_waits(c, c->seq, &a.wait));
    DSGD_CUDA(cudaMemsetAsync(c->scratch, 0, 4 * sizeof(double), c->stream));
    {
      LaunchScope ls(c, DSGD_K_OTHER);
      DSGD_CUDA(dsgd::launch_trace<T>(a, blocks_for(c, c->d, 1), c->stream));
    }
    DSGD_CUDA(cudaMemcpyAsync(c->norm_host, c->scratch, 4 * sizeof(double),
                              cudaMemcpyDeviceToHost, c->stream));
    DSGD_CUDA(cudaStreamSynchronize(c->stream));
    if (c->norm_host[3] != 0.0)
      return set_error(DSGD_ESTATE, "non-finite parameter encountered at t=" +
                                        std::to_string(c->t[0]));
    if (sq_err_consensus) *sq_err_consensus = c->norm_host[0];
    if (loss_mean) *loss_mean = c->spec ? 0.5 * c->norm_host[1] / c->p : 0.0;
    if (sq_err_opt) *sq_err_opt = c->spec ? c->norm_host[2] : 0.0;
    if (loss_mean && c->lg_X) {
      // LogisticObjective::value objectives.cpp:116-125 of every node:
      // mean over rows of log1pexp(z) - y z, plus 0.5 l2 ||theta||^2 (the
      // trace kernel's sum of squares with no optimum)
      double data = 0.0;
      DSGD_TRY(logistic_values<T>(c, &data));
      *loss_mean = (data + 0.5 * c->lg_l2 * c->norm_host[2]) / c->p;
    }
    return DSGD_OK;
  });
}

dsgd_status dsgd_ea_init_center(dsgd_ctx* c) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!(c->flags & DSGD_CTX_CENTER)) return set_error(DSGD_ESTATE, "no center (DSGD_CTX_CENTER)");
  return dispatch(c, [&](auto z) -> dsgd_status {
    using T = decltype(z);
    T* center = as<T>(c->arena + c->off_c_in);
    if (!c->distributed()) {
      const T* xs[kMaxLocal];
      for (uint32_t i = 0; i < c->n_local; ++i) xs[i] = as<T>(c->theta_ptr(i, c->cur));
      LaunchScope ls(c, DSGD_K_OTHER);
      DSGD_CUDA(dsgd::launch_spatial_mean<T>(xs, c->p, c->d, center, c->stream));
      return DSGD_OK;
    }
    // only node 0's context owns the server center (other ranks' c_in are
    // written by their chain predecessor): it reads every rank's theta over
    // NVLink and forms the reference's pivot-form mean (param_vec.cpp:19-40)
    if (!c->connected) return set_error(DSGD_ESTATE, "peers not connected");
    if (c->first != 0) return DSGD_OK;
    const T* xs[kMaxLocal];
    for (uint32_t k = 0; k < c->p; ++k) xs[k] = as<T>(c->peers[k].theta[c->cur]);
    LaunchScope ls(c, DSGD_K_OTHER);
    DSGD_CUDA(dsgd::launch_spatial_mean<T>(xs, c->p, c->d, center, c->stream));
    return DSGD_OK;
  });
}

// --------------------------------------------------------- worker loop
dsgd_status dsgd_ctx_seed_streams(dsgd_ctx* c, uint64_t seed, const char* run_id) {
  DSGD_TRY(check_ctx(c));
  for (auto* s : c->partner_streams) dsgd_stream_destroy(s);
  for (auto* s : c->noise_streams) dsgd_stream_destroy(s);
  c->partner_streams.assign(c->p, nullptr);
  c->noise_streams.assign(c->n_local, nullptr);
  for (auto* s : c->sample_streams) dsgd_stream_destroy(s);
  c->sample_streams.assign(c->n_local, nullptr);
  if (c->clock_stream) dsgd_stream_destroy(c->clock_stream);
  c->clock_stream = nullptr;
  // run-level stream: node id kRunLevelNode = 0xFFFFFFFF (simulator.cpp:398)
  DSGD_TRY(dsgd_stream_make(seed, run_id, 0xFFFFFFFFu, DSGD_PURPOSE_CLOCK, &c->clock_stream));
  for (uint32_t i = 0; i < c->n_local; ++i)
    DSGD_TRY(dsgd_stream_make(seed, run_id, c->first + i, DSGD_PURPOSE_SAMPLE,
                              &c->sample_streams[i]));
  for (uint32_t i = 0; i < c->p; ++i)
    DSGD_TRY(dsgd_stream_make(seed, run_id, i, DSGD_PURPOSE_PARTNER, &c->partner_streams[i]));
  for (uint32_t i = 0; i < c->n_local; ++i)
    DSGD_TRY(dsgd_stream_make(seed, run_id, c->first + i, DSGD_PURPOSE_NOISE,
                              &c->noise_streams[i]));
  return DSGD_OK;
}

dsgd_status dsgd_run_events(dsgd_ctx* c, const dsgd_run_desc* run, uint64_t events,
                            double rate_per_node, double* sim_time, double* alpha) {
  DSGD_TRY(check_ctx(c));
  if (!run) return set_error(DSGD_EINVAL, "null run descriptor");
  DSGD_TRY(dsgd_hyperparams_validate(&run->hyper));
  const dsgd_protocol proto = run->protocol;
  if (proto != DSGD_ASYNC_PULL && proto != DSGD_ELASTIC_AVG)
    return set_error(DSGD_EINVAL, "asynchronous driver supports async-pull and elastic-avg");
  if (c->distributed()) return set_error(DSGD_EINVAL, "the asynchronous driver runs on one context");
  if (!c->clock_stream || c->partner_streams.size() != c->p ||
      c->noise_streams.size() != c->n_local)
    return set_error(DSGD_ESTATE, "dsgd_ctx_seed_streams first");
  if (!(rate_per_node > 0.0)) return set_error(DSGD_EINVAL, "poisson rate must be positive");
  if (run->host_noise_sigma > 0.0) {
    if (!c->noise[0]) return set_error(DSGD_ESTATE, "host noise needs DSGD_CTX_NOISE");
    if (!c->noise_host) c->noise_host = new double[c->d];
  }
  const dsgd_hyperparams* h = &run->hyper;
  double now = sim_time ? *sim_time : 0.0;
  double last_alpha = alpha ? *alpha : 0.0;
  for (uint64_t k = 0; k < events; ++k) {
    // sample_next_event simulator.cpp:128-140: gap, then the ticking node
    double gap = 0.0;
    DSGD_TRY(dsgd_stream_exponential(c->clock_stream, (double)c->p * rate_per_node, &gap));
    uint32_t i = 0;
    DSGD_TRY(dsgd_stream_uniform_index(c->clock_stream, c->p, &i));
    now += gap;
    last_alpha = dsgd_step_size_at(h, c->t[i]);
    dsgd_grad_spec g = run->grad;
    uint32_t j = 0;
    if (proto == DSGD_ASYNC_PULL)  // partner from the ticking node's stream (416-417)
      DSGD_TRY(dsgd_stream_uniform_index(c->partner_streams[i], c->p, &j));
    if (run->host_noise_sigma > 0.0) {  // NoiseModel::sample on node i's noise stream
      dsgd_stream_fill_normal(c->noise_streams[i], run->host_noise_sigma, c->noise_host, c->d);
      DSGD_TRY(dsgd_set_vector(c, i, DSGD_BUF_NOISE, c->noise_host));
      g.use_noise = 1;
    }
    dsgd_status st;
    if (proto == DSGD_ASYNC_PULL) {
      st = dsgd_async_pull_event(c, h, &g, i, j);
    } else {
      const uint64_t ti = c->t[i];
      st = dsgd_ea_client_event(c, h, &g, i, (ti > 0 && ti % h->tau == 0) ? 1 : 0);
    }
    if (st != DSGD_OK) return st;
  }
  if (sim_time) *sim_time = now;
  if (alpha) *alpha = last_alpha;
  return norm_read(c);  // grad_norm_out: one host read per run, not per event
}

dsgd_status dsgd_ctx_round(dsgd_ctx* c, uint64_t* round) {
  DSGD_TRY(check_ctx(c));
  *round = c->rounds_done;
  return DSGD_OK;
}

namespace {

dsgd_status run_check(dsgd_ctx* c, const dsgd_run_desc* run) {
  DSGD_TRY(check_ctx(c));
  if (!run) return set_error(DSGD_EINVAL, "null run descriptor");
  DSGD_TRY(dsgd_hyperparams_validate(&run->hyper));
  const dsgd_protocol proto = run->protocol;
  const bool needs_partners = proto == DSGD_PULL_GOSSIP || proto == DSGD_GOSSIP_STALE ||
                              proto == DSGD_GOSSIP_FRESH || proto == DSGD_PUSH_GOSSIP;
  if (needs_partners && c->partner_streams.size() != c->p)
    return set_error(DSGD_ESTATE, "dsgd_ctx_seed_streams first");
  if (proto == DSGD_ASYNC_PULL) return set_error(DSGD_EINVAL, "async-pull is event-driven");
  if (proto > DSGD_ASYNC_PULL) return set_error(DSGD_EINVAL, "unknown protocol");
  if (run->host_noise_sigma > 0.0) {
    if (!c->noise[0]) return set_error(DSGD_ESTATE, "host noise needs DSGD_CTX_NOISE");
    if (c->noise_streams.size() != c->n_local)
      return set_error(DSGD_ESTATE, "dsgd_ctx_seed_streams first");
    if (!c->noise_host) c->noise_host = new double[c->d];
  }
  return DSGD_OK;
}

// One round of run_sync's loop (simulator.cpp:234-369) on one context.
dsgd_status run_one_round(dsgd_ctx* c, const dsgd_run_desc* run) {
  const dsgd_protocol proto = run->protocol;
  const dsgd_hyperparams* h = &run->hyper;
  std::vector<uint32_t> map(c->p);
  const void* grads[kMaxLocal];
  const uint64_t t = c->t[0];
  const bool gated = t > 0 && t % h->tau == 0;  // simulator.cpp:25
  dsgd_grad_spec g = run->grad;
  if (run->n_grad_pool > 0) {
    const uint64_t slot = c->rounds_done % run->n_grad_pool;
    for (uint32_t i = 0; i < c->n_local; ++i) grads[i] = run->grad_pool[slot * c->n_local + i];
    g.source = DSGD_GRAD_BUFFER;
    g.grad = grads;
  }
  if (run->host_noise_sigma > 0.0) {
    // NoiseModel::sample on each local node's reference noise stream
    for (uint32_t i = 0; i < c->n_local; ++i) {
      dsgd_stream_fill_normal(c->noise_streams[i], run->host_noise_sigma, c->noise_host, c->d);
      DSGD_TRY(dsgd_set_vector(c, i, DSGD_BUF_NOISE, c->noise_host));
    }
    g.use_noise = 1;
  }
  switch (proto) {
    case DSGD_ALLREDUCE:
      return dsgd_allreduce_round(c, h, &g, run->scope);
    case DSGD_ELASTIC_AVG:
      return dsgd_ea_round(c, h, &g, gated ? 1 : 0);
    case DSGD_PULL_GOSSIP:
    case DSGD_GOSSIP_STALE:
    case DSGD_GOSSIP_FRESH:
      if (!gated) return dsgd_pull_gossip_round(c, h, &g, nullptr);
      DSGD_TRY(dsgd_draw_pull_partners(c->partner_streams.data(), c->p, map.data()));
      return proto == DSGD_PULL_GOSSIP    ? dsgd_pull_gossip_round(c, h, &g, map.data())
             : proto == DSGD_GOSSIP_STALE ? dsgd_gossip_stale_round(c, h, &g, map.data())
                                          : dsgd_gossip_fresh_round(c, h, &g, map.data());
    case DSGD_PUSH_GOSSIP:
      if (!(gated && c->p > 1)) return dsgd_pull_gossip_round(c, h, &g, nullptr);
      DSGD_TRY(dsgd_draw_push_targets(c->partner_streams.data(), c->p, map.data()));
      return dsgd_push_gossip_round(c, h, &g, map.data());
    default:
      return set_error(DSGD_EINVAL, "unknown protocol");
  }
}

// Leaves the context in its logical state (the timed work of `rounds`
// rounds includes the last deferred apply) and settles grad_norm_out: one
// host read per run, not per round.
dsgd_status run_finish(dsgd_ctx* c) {
  DSGD_TRY(flush_pending(c));
  DeviceGuard dg(c->device);
  return norm_read(c);
}

}  // namespace

dsgd_status dsgd_run_rounds(dsgd_ctx* c, const dsgd_run_desc* run) {
  DSGD_TRY(run_check(c, run));
  if (c->grp && c->p > 1)
    return set_error(DSGD_EINVAL, "in-process group: use dsgd_group_run_rounds");
  c->lt_run = true;
  c->lt_prev = false;
  dsgd_status st = DSGD_OK;
  for (uint64_t r = 0; r < run->rounds && st == DSGD_OK; ++r) st = run_one_round(c, run);
  c->lt_run = c->lt_prev = false;
  DSGD_TRY(st);
  return run_finish(c);
}

dsgd_status dsgd_group_run_rounds(dsgd_ctx* const* ctxs, uint32_t n, const dsgd_run_desc* runs) {
  if (!ctxs || !runs || n == 0) return set_error(DSGD_EINVAL, "null group");
  for (uint32_t k = 0; k < n; ++k) {
    DSGD_TRY(run_check(ctxs[k], &runs[k]));
    if (!ctxs[k]->grp || ctxs[k]->grp->ctx.size() != n || ctxs[k]->grp->ctx[k] != ctxs[k])
      return set_error(DSGD_EINVAL, "contexts must be one in-process group in node order");
    if (runs[k].rounds != runs[0].rounds || runs[k].protocol != runs[0].protocol)
      return set_error(DSGD_EINVAL, "every rank runs the same rounds and protocol");
  }
  for (uint64_t r = 0; r < runs[0].rounds; ++r)
    for (uint32_t k = 0; k < n; ++k) {  // host order = rank order inside every round
      DeviceGuard dg(ctxs[k]->device);
      DSGD_TRY(run_one_round(ctxs[k], &runs[k]));
    }
  for (uint32_t k = 0; k < n; ++k) DSGD_TRY(run_finish(ctxs[k]));
  return DSGD_OK;
}

// -------------------------------------------------------- multi-GPU wiring
dsgd_status dsgd_ctx_export_handle(dsgd_ctx* c, void* blob) {
  DSGD_TRY(check_ctx(c));
  if (!blob) return set_error(DSGD_EINVAL, "null blob");
  DeviceGuard g(c->device);
  HandleBlob b{};
  b.magic = kMagic;
  b.abi = DSGD_B200_ABI_VERSION;
  b.first_node = c->first;
  b.n_local = c->n_local;
  b.dtype = c->dtype;
  b.flags = c->flags;
  b.d = c->d;
  b.device = c->device;
  DSGD_CUDA(cudaIpcGetMemHandle(&b.handle, c->arena));
  b.arena_bytes = c->arena_bytes;
  b.off_theta[0] = c->off_theta[0][0];
  b.off_theta[1] = c->off_theta[0][1];
  b.off_c_in = c->off_c_in;
  b.off_flags = c->off_flags;
  b.off_round = c->off_round;
  b.off_x = c->off_x;
  b.off_a = c->off_a;
  b.off_ar = c->off_ar;
  b.off_x2 = c->off_x2;
  b.off_hb = c->off_hb;
  // NVLS: rank 0 creates the multicast object every rank joins in
  // dsgd_ctx_connect_peers (the decision is the same on every rank)
  if (c->first == 0 && wants_nvls(c) && c->mc.mc == 0) {
    if (!dsgd::mc_supported(c->device)) {
      c->nvls_note = "the GPU reports no multicast (NVLS) support";
    } else {
      int fd = -1;
      const dsgd_status s1 = dsgd::mc_create(&c->mc, c->device, c->p, nvls_bytes(c), true);
      const dsgd_status s2 = s1 == DSGD_OK ? dsgd::mc_export_fd(&c->mc, &fd) : s1;
      if (s2 != DSGD_OK) {
        c->nvls_note = dsgd::g_error;
        dsgd::mc_release(&c->mc, c->device);
      }
    }
  }
  if (c->first == 0 && c->mc.mc && c->mc.export_fd >= 0) {
    b.mc_kind = 2;
    b.mc_pid = (int32_t)getpid();
    b.mc_fd = c->mc.export_fd;
    b.mc_size = c->mc.size;
  }
  std::memset(blob, 0, DSGD_HANDLE_BYTES);
  std::memcpy(blob, &b, sizeof(b));
  return DSGD_OK;
}

dsgd_status dsgd_ctx_connect_peers(dsgd_ctx* c, const void* blobs) {
  DSGD_TRY(check_ctx(c));
  if (!blobs) return set_error(DSGD_EINVAL, "null blobs");
  if (!c->distributed()) {
    c->connected = true;
    return DSGD_OK;
  }
  DeviceGuard g(c->device);
  const char* base = static_cast<const char*>(blobs);
  for (uint32_t k = 0; k < c->p; ++k) {
    HandleBlob b;
    std::memcpy(&b, base + (size_t)k * DSGD_HANDLE_BYTES, sizeof(b));
    if (b.magic != kMagic || b.abi != DSGD_B200_ABI_VERSION)
      return set_error(DSGD_EINVAL, "bad handle blob");
    if (b.first_node != k || b.n_local != 1)
      return set_error(DSGD_EINVAL, "blob order must be node order, one node per context");
    if (b.d != c->d || b.dtype != (uint32_t)c->dtype)
      return set_error(DSGD_EINVAL, "peer dimension/dtype mismatch");
    if ((b.flags & DSGD_CTX_CENTER) != (c->flags & DSGD_CTX_CENTER))
      return set_error(DSGD_EINVAL, "DSGD_CTX_CENTER must match on every rank");
    if (k == c->first) continue;
    if (b.device != c->device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, c->device, b.device);
      if (can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return set_error(DSGD_ECUDA, std::string("enable peer access: ") + cudaGetErrorString(e));
        cudaGetLastError();
      }
    }
    void* mapped = nullptr;
    DSGD_CUDA(cudaIpcOpenMemHandle(&mapped, b.handle, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(mapped);
    char* m = static_cast<char*>(mapped);
    PeerNode& pn = c->peers[k];
    pn.theta[0] = m + b.off_theta[0];
    pn.theta[1] = m + b.off_theta[1];
    pn.round = reinterpret_cast<unsigned long long*>(m + b.off_round);
    if (b.off_x) {
      pn.x = m + b.off_x;
      pn.avg = m + b.off_a;
      pn.ar = reinterpret_cast<unsigned long long*>(m + b.off_ar);
      pn.x2 = m + b.off_x2;
      pn.hb = reinterpret_cast<unsigned long long*>(m + b.off_hb);
    }
    if (b.flags & DSGD_CTX_CENTER) {
      pn.c_in = m + b.off_c_in;
      pn.flags = reinterpret_cast<unsigned long long*>(m + b.off_flags);
    }
  }
  c->connected = true;
  HandleBlob b0;
  std::memcpy(&b0, base, sizeof(b0));
  if (b0.mc_kind == 2 && wants_nvls(c)) return join_nvls(c, b0);
  if (wants_nvls(c) && c->nvls_note.empty())
    c->nvls_note = "rank 0 created no multicast object";
  return DSGD_OK;
}

dsgd_status dsgd_group_create_inproc(const dsgd_ctx_desc* base, uint32_t p, const int* devices,
                                     dsgd_ctx** out) {
  if (!base || !out) return set_error(DSGD_EINVAL, "null argument");
  if (p == 0 || p > (uint32_t)kMaxWait) return set_error(DSGD_EINVAL, "in-process group: 1 <= p <= 16");
  auto grp = std::make_shared<InprocGroup>();
  std::vector<int> dev(p);
  for (uint32_t r = 0; r < p; ++r) dev[r] = devices ? devices[r] : base->device;
  auto stream_of = [&](int d, cudaStream_t* s) -> dsgd_status {
    for (auto& e : grp->streams)
      if (e.first == d) {
        *s = e.second;
        return DSGD_OK;
      }
    DeviceGuard g(d);
    DSGD_CUDA(cudaSetDevice(d));
    cudaStream_t ns = nullptr;
    DSGD_CUDA(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
    grp->streams.emplace_back(d, ns);
    *s = ns;
    return DSGD_OK;
  };
  auto fail = [&](dsgd_status st) {
    const std::string msg = dsgd::g_error;
    for (dsgd_ctx* c : grp->ctx) dsgd_ctx_destroy(c);
    grp->ctx.clear();
    return set_error(st, msg);
  };
  for (uint32_t r = 0; r < p; ++r) {
    dsgd_ctx_desc d = *base;
    d.device = dev[r];
    d.p = p;
    d.first_node = r;
    d.n_local = 1;
    cudaStream_t s = nullptr;
    dsgd_status st = stream_of(dev[r], &s);
    if (st != DSGD_OK) return fail(st);
    d.stream = s;
    dsgd_ctx* c = nullptr;
    st = dsgd_ctx_create(&d, &c);
    if (st != DSGD_OK) return fail(st);
    grp->ctx.push_back(c);
  }
  for (uint32_t r = 0; r < p; ++r) {
    dsgd_ctx* c = grp->ctx[r];
    DeviceGuard g(c->device);
    const bool shared = std::count(dev.begin(), dev.end(), c->device) > 1;
    if (shared) {
      // ranks of one GPU: one stream, no pipeline streams (nothing of two
      // ranks may run concurrently on one device), and a short flag timeout
      // (a wait host order cannot satisfy never will be)
      for (int h = 0; h < 4; ++h) {
        if (c->pipe_stream[h] && c->pipe_stream[h] != c->stream) cudaStreamDestroy(c->pipe_stream[h]);
        c->pipe_stream[h] = c->stream;
      }
      c->timeout_ns = 5ull * 1000 * 1000 * 1000;
    }
    for (uint32_t k = 0; k < p; ++k) {
      if (k == r) continue;
      dsgd_ctx* o = grp->ctx[k];
      if (o->device != c->device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, c->device, o->device);
        if (!can) return fail(set_error(DSGD_ECUDA, "no peer access between the group's GPUs"));
        cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(set_error(DSGD_ECUDA, std::string("enable peer access: ") + cudaGetErrorString(e)));
        cudaGetLastError();
      }
      c->peers[k] = o->peers[k];  // the owner's own view of its arena
    }
    c->connected = true;
    c->grp = grp;
  }
  {
    const dsgd_status st = inproc_nvls(grp.get());
    if (st != DSGD_OK) return fail(st);
  }
  for (uint32_t r = 0; r < p; ++r) out[r] = grp->ctx[r];
  return DSGD_OK;
}

dsgd_status dsgd_ctx_attach_multicast(dsgd_ctx* c, void* x, void* x_mc, void* avg, void* avg_mc) {
  DSGD_TRY(check_ctx(c));
  DSGD_TRY(flush_pending(c));
  if (!c->distributed() || !c->connected)
    return set_error(DSGD_ESTATE, "multicast all-reduce needs a connected one-node-per-GPU group");
  if (!x || !x_mc || !avg || !avg_mc) return set_error(DSGD_EINVAL, "null multicast buffer");
  for (void* q : {x, x_mc, avg, avg_mc})
    if (!aligned16(q)) return set_error(DSGD_EINVAL, "multicast buffers must be 16-byte aligned");
  if (c->mc.mc) return set_error(DSGD_ESTATE, "the library already set up multicast buffers");
  attach_nvls(c, static_cast<char*>(x), static_cast<char*>(x_mc), static_cast<char*>(avg),
              static_cast<char*>(avg_mc));
  return DSGD_OK;
}

dsgd_status dsgd_ctx_allreduce_backend(dsgd_ctx* c, const char** name, const char** note) {
  DSGD_TRY(check_ctx(c));
  const char* n = !c->distributed()       ? "local"
                  : !c->p2p_allreduce     ? "nccl"
                  : c->ar_oneshot         ? "oneshot"
                  : c->ar_nvls            ? "nvls"
                                          : "p2p";
  if (name) *name = n;
  if (note) *note = c->nvls_note.c_str();
  return DSGD_OK;
}

dsgd_status dsgd_nccl_unique_id(void* id) {
  if (!id) return set_error(DSGD_EINVAL, "null id");
  static_assert(sizeof(ncclUniqueId) == DSGD_NCCL_ID_BYTES, "nccl id size");
  ncclUniqueId u;
  DSGD_NCCL(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return DSGD_OK;
}

dsgd_status dsgd_ctx_init_nccl(dsgd_ctx* c, const void* id, int rank, int nranks) {
  DSGD_TRY(check_ctx(c));
  if (!id || nranks <= 0 || rank < 0 || rank >= nranks)
    return set_error(DSGD_EINVAL, "bad nccl rank/size");
  if ((uint32_t)nranks != c->p || (uint32_t)rank != c->first)
    return set_error(DSGD_EINVAL, "NCCL ranks must equal node ids (one node per context)");
  DeviceGuard g(c->device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  DSGD_NCCL(ncclCommInitRank(&c->comm, nranks, u, rank));
  return DSGD_OK;
}

// ------------------------------------------------------------ measurement
dsgd_status dsgd_profile_enable(dsgd_ctx* c, int enable) {
  DSGD_TRY(check_ctx(c));
  DeviceGuard g(c->device);
  if (!enable) DSGD_TRY(collect_profile(c));
  c->profile = enable != 0;
  return DSGD_OK;
}

dsgd_status dsgd_profile_read(dsgd_ctx* c, dsgd_kernel_id k, double* total_ms, uint64_t* launches,
                              int reset) {
  DSGD_TRY(check_ctx(c));
  if ((int)k < 0 || k >= DSGD_K_COUNT) return set_error(DSGD_EINVAL, "kernel id");
  DeviceGuard g(c->device);
  DSGD_TRY(collect_profile(c));
  if (total_ms) *total_ms = c->prof_ms[k];
  if (launches) *launches = c->prof_launches[k];
  if (reset) {
    c->prof_ms[k] = 0;
    c->prof_launches[k] = 0;
  }
  return DSGD_OK;
}

dsgd_status dsgd_trace_dump(dsgd_ctx* c, uint64_t* out, uint32_t max_records, uint32_t* n) {
  DSGD_TRY(check_ctx(c));
  DeviceGuard g(c->device);
  DSGD_TRY(join_pipes(c));
  DSGD_CUDA(cudaStreamSynchronize(c->stream));
  const uint32_t m = std::min(max_records, c->trace_n);
  std::vector<unsigned long long> buf(3ull * std::max<uint32_t>(1, m));
  if (m) DSGD_CUDA(cudaMemcpy(buf.data(), c->trace_dev, 24ull * m, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < m; ++i) {
    out[5ull * i + 0] = c->trace_kind[i];
    out[5ull * i + 1] = c->trace_round[i];
    out[5ull * i + 2] = buf[3ull * i + 0];
    out[5ull * i + 3] = buf[3ull * i + 1];
    out[5ull * i + 4] = buf[3ull * i + 2];
  }
  *n = m;
  return DSGD_OK;
}

dsgd_status dsgd_launch_count(dsgd_ctx* c, uint64_t* kernels, uint64_t* nccl_calls) {
  DSGD_TRY(check_ctx(c));
  if (kernels) *kernels = c->kernels;
  if (nccl_calls) *nccl_calls = c->nccl_calls;
  return DSGD_OK;
}

}  // extern "C"
