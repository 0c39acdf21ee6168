/*
 * dsgd_b200.h -- C ABI of the B200-native parameter-aggregation and update
 * path of arXiv 1611.04581 (synchronous all-reduce SGD, elastic averaging SGD
 * and gossiping SGD, all with Nesterov momentum).
 *
 * Drop-in boundary.  The reference has no FFI; its boundary is the C++
 * update-rule interface /root/reference/proj/include/dsgd/protocols.hpp:45-152
 * plus the per-step worker loops that call it
 * (src/simulator.cpp:234-369 run_sync, src/transport.cpp:342-479
 * run_transport worker).  Each entry point below names the reference
 * function it replaces.  State lives on the device (SoA buffers per node);
 * the host passes hyperparameters, partner maps and gate bits, exactly the
 * arguments the reference functions take besides the NodeState vectors.
 *
 * Conventions
 *  - Every function returns dsgd_status; no C++ exception crosses the ABI.
 *    DSGD_EINVAL mirrors the reference's std::invalid_argument
 *    (protocols.cpp:43-77, 198-202, 282-284), DSGD_ETIMEOUT its
 *    TransportError (transport.hpp:57-60); dsgd_last_error() gives the text
 *    (thread-local).
 *  - A context (dsgd_ctx) is one process's view of one GPU; it hosts
 *    n_local nodes (workers).  Group calls are lock-step: every context of a
 *    group makes the same sequence of round calls (like NCCL collectives).
 *    A group is either all p nodes in one context (p workers on one GPU) or
 *    one node per context, one context per GPU (one process per GPU), wired
 *    with dsgd_ctx_export_handle / dsgd_ctx_connect_peers (CUDA IPC peer
 *    memory over NVLink) and dsgd_ctx_init_nccl.
 *  - Arithmetic: DSGD_F64 reproduces the reference fp64 operation order
 *    bit-for-bit (explicit round-to-nearest intrinsics, no FMA contraction);
 *    DSGD_F32 runs the same operation order in binary32.
 */
#ifndef DSGD_B200_H_
#define DSGD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSGD_B200_ABI_VERSION 2
#define DSGD_MAX_LOCAL_NODES 32
#define DSGD_HANDLE_BYTES 512 /* size of one dsgd_ctx_export_handle blob */
#define DSGD_NCCL_ID_BYTES 128

typedef enum {
  DSGD_OK = 0,
  DSGD_EINVAL = 1,   /* std::invalid_argument in the reference */
  DSGD_ECUDA = 2,    /* CUDA runtime error */
  DSGD_ENCCL = 3,    /* NCCL error */
  DSGD_ETIMEOUT = 4, /* TransportError: a peer never arrived */
  DSGD_ENOMEM = 5,
  DSGD_ESTATE = 6 /* call out of order (e.g. peers not connected) */
} dsgd_status;

typedef enum { DSGD_F32 = 0, DSGD_F64 = 1 } dsgd_dtype;

/* ProtocolKind core.hpp:31-39 (same numbering) */
typedef enum {
  DSGD_ALLREDUCE = 0,
  DSGD_ELASTIC_AVG = 1,
  DSGD_PULL_GOSSIP = 2,
  DSGD_PUSH_GOSSIP = 3,
  DSGD_GOSSIP_STALE = 4,
  DSGD_GOSSIP_FRESH = 5,
  DSGD_ASYNC_PULL = 6
} dsgd_protocol;

/* MomentumScope core.hpp:46 */
typedef enum { DSGD_SCOPE_AGGREGATE = 0, DSGD_SCOPE_PER_NODE = 1 } dsgd_momentum_scope;

/* StreamPurpose rng.hpp:30-37 */
typedef enum {
  DSGD_PURPOSE_NOISE = 0,
  DSGD_PURPOSE_SAMPLE = 1,
  DSGD_PURPOSE_PARTNER = 2,
  DSGD_PURPOSE_CLOCK = 3,
  DSGD_PURPOSE_STRAGGLER = 4,
  DSGD_PURPOSE_INIT = 5
} dsgd_purpose;

/* Hyperparams core.hpp:54-70 (anneal_at sorted ascending, n_anneal entries) */
typedef struct {
  double alpha0;
  double anneal_factor;
  const uint64_t* anneal_at;
  uint32_t n_anneal;
  double mu;
  double weight_decay;
  double beta_gossip;
  double beta_ea;
  uint32_t tau;
  uint32_t batch;
} dsgd_hyperparams;

const char* dsgd_last_error(void);
int dsgd_abi_version(void);

/* ------------------------------------------------------------------ host
 * Deterministic streams: rng.hpp:50-95 / rng.cpp:24-112 (std::mt19937_64,
 * explicit samplers).  Peer schedules are drawn on the host, bit-exact. */
typedef struct dsgd_stream dsgd_stream;
uint64_t dsgd_derive_stream_seed(uint64_t root_seed, const char* run_id, uint32_t node_id,
                                 dsgd_purpose purpose);                 /* rng.cpp:93 */
dsgd_status dsgd_stream_create(uint64_t engine_seed, dsgd_stream** out); /* RngStream(seed) */
dsgd_status dsgd_stream_make(uint64_t root_seed, const char* run_id, uint32_t node_id,
                             dsgd_purpose purpose, dsgd_stream** out); /* make_stream */
dsgd_status dsgd_stream_clone(const dsgd_stream* s, dsgd_stream** out);
void dsgd_stream_destroy(dsgd_stream* s);
uint64_t dsgd_stream_next_u64(dsgd_stream* s);
double dsgd_stream_uniform01(dsgd_stream* s);
double dsgd_stream_normal(dsgd_stream* s);
dsgd_status dsgd_stream_uniform_index(dsgd_stream* s, uint32_t n, uint32_t* out);
dsgd_status dsgd_stream_exponential(dsgd_stream* s, double rate, double* out);
/* NoiseModel::sample objectives.cpp:175-183: out[k] = sigma * normal() */
void dsgd_stream_fill_normal(dsgd_stream* s, double sigma, double* out, uint64_t n);

double dsgd_step_size_at(const dsgd_hyperparams* h, uint64_t t); /* core.cpp:82-92 */
dsgd_status dsgd_hyperparams_validate(const dsgd_hyperparams* h); /* core.cpp:62-80 */
/* draw_pull_partners / draw_push_targets simulator.cpp:69-88 */
dsgd_status dsgd_draw_pull_partners(dsgd_stream* const* partner_streams, uint32_t p,
                                    uint32_t* out);
dsgd_status dsgd_draw_push_targets(dsgd_stream* const* partner_streams, uint32_t p,
                                   uint32_t* out);

/* --------------------------------------------------------------- context */
typedef struct dsgd_ctx dsgd_ctx;

enum {
  DSGD_CTX_QUADRATIC = 1u << 0, /* device-resident diagonal quadratic objective (s, opt) */
  DSGD_CTX_GRAD = 1u << 1,      /* own gradient buffer per node (DSGD_BUF_GRAD) */
  DSGD_CTX_NOISE = 1u << 2,     /* own additive-noise buffer per node (DSGD_BUF_NOISE) */
  DSGD_CTX_CENTER = 1u << 3     /* EASGD center (on the context hosting node 0) */
};

typedef struct {
  int device;
  uint64_t dim;        /* d */
  dsgd_dtype dtype;
  uint32_t p;          /* nodes in the whole group */
  uint32_t first_node; /* global id of this context's node 0 */
  uint32_t n_local;    /* nodes hosted here (p, or 1 with one context per GPU) */
  uint32_t flags;      /* DSGD_CTX_* */
  void* stream;        /* cudaStream_t to launch on; NULL: the context creates one */
} dsgd_ctx_desc;

dsgd_status dsgd_ctx_create(const dsgd_ctx_desc* desc, dsgd_ctx** out);
void dsgd_ctx_destroy(dsgd_ctx* ctx);
dsgd_status dsgd_ctx_stream(dsgd_ctx* ctx, void** stream);
/* Waits for the context's stream and reports device-side failures (a peer
 * timeout inside a kernel -> DSGD_ETIMEOUT). */
dsgd_status dsgd_ctx_sync(dsgd_ctx* ctx);
/* Raises the grad_norm_out of the rounds run since the last read to the
 * device-side running max (one host wait). */
dsgd_status dsgd_grad_norm_flush(dsgd_ctx* ctx);

/* Buffers (device pointers, dtype elements, d per node). */
typedef enum {
  DSGD_BUF_THETA = 0, /* current parameters */
  DSGD_BUF_DELTA = 1, /* delta_prev (momentum memory) */
  DSGD_BUF_GRAD = 2,
  DSGD_BUF_NOISE = 3,
  DSGD_BUF_SPECTRUM = 4,
  DSGD_BUF_OPT = 5,
  DSGD_BUF_CENTER = 6
} dsgd_buffer;
dsgd_status dsgd_buffer_ptr(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which, void** dev);

/* NodeState io: host fp64 vectors converted to the context dtype. */
dsgd_status dsgd_set_state(dsgd_ctx* ctx, uint32_t local, const double* theta,
                           const double* delta_prev, uint64_t t);
dsgd_status dsgd_get_state(dsgd_ctx* ctx, uint32_t local, double* theta, double* delta_prev,
                           uint64_t* t);
dsgd_status dsgd_set_vector(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which,
                            const double* host);
/* DSGD_BUF_CENTER on rank 0 of a multi-GPU EASGD chain: waits (bounded by
 * the context timeout -> DSGD_ETIMEOUT) until the last gated round's center
 * has fully arrived from rank p-1, so no host barrier is needed first. */
dsgd_status dsgd_get_vector(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which, double* host);
/* Raw asynchronous copies in the context dtype on the context stream (host
 * memory should be pinned); used by the end-to-end path.  A DSGD_BUF_CENTER
 * download on rank 0 of a multi-GPU EASGD chain is ordered after the last
 * round's center chunks on the device (no host wait). */
dsgd_status dsgd_upload_async(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which,
                              const void* host, uint64_t count);
dsgd_status dsgd_download_async(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which, void* host,
                                uint64_t count);
/* Copy `count` elements from any device/pinned pointer (cudaMemcpyDefault)
 * into a context buffer on the context stream, e.g. parameters held by a
 * framework tensor. */
dsgd_status dsgd_copy_in_async(dsgd_ctx* ctx, uint32_t local, dsgd_buffer which,
                               const void* src, uint64_t count);
dsgd_status dsgd_get_t(dsgd_ctx* ctx, uint32_t local, uint64_t* t);
dsgd_status dsgd_set_t(dsgd_ctx* ctx, uint32_t local, uint64_t t);

/* ------------------------------------------------------- gradient source
 * The reference's Objective plugin (objectives.hpp:33-53) evaluated at the
 * lookahead point theta + mu*delta_prev.  DSGD_GRAD_QUADRATIC evaluates
 * QuadraticObjective::gradient (objectives.cpp:71-78) inside the update
 * kernel; DSGD_GRAD_BUFFER reads a per-node device buffer holding the
 * minibatch gradient (the caller's model fills it).  Weight decay and the
 * additive noise draw are always applied inside the kernel, in the
 * reference order (protocols.cpp:27-38, 98). */
typedef enum {
  DSGD_GRAD_QUADRATIC = 0,
  DSGD_GRAD_BUFFER = 1,
  /* LogisticObjective::stochastic_gradient (objectives.cpp:147-162) on the
   * device-resident dataset of dsgd_set_logistic, evaluated at the point the
   * rule evaluates its gradient (after the pull/push/EASGD mix, at the
   * lookahead theta + mu*delta_prev, or at theta for async-pull), h->batch
   * rows per node.  Written into each node's DSGD_BUF_GRAD, then consumed as
   * DSGD_GRAD_BUFFER. */
  DSGD_GRAD_LOGISTIC = 2
} dsgd_grad_source;

typedef struct {
  dsgd_grad_source source;
  const void* const* grad; /* GRAD_BUFFER: n_local device pointers, or NULL for DSGD_BUF_GRAD */
  uint32_t use_noise;      /* 0: add +0.0 (NoiseModel::zero); 1: add DSGD_BUF_NOISE (e.g. the
                              reference noise stream drawn on the host); 2: N(0, noise_sigma^2)
                              drawn inside the kernel (Philox keyed by noise_seed, node, t) */
  double* grad_norm_out;   /* optional: raised to max ||g_i|| over nodes and rounds like
                              protocols.cpp:34-36.  Accumulated on the device without a host
                              wait; *grad_norm_out is raised lazily, when the call that
                              needs it returns: dsgd_grad_norm_flush, dsgd_ctx_sync,
                              dsgd_get_state, the end of dsgd_run_rounds / dsgd_run_events,
                              or a round passing a different grad_norm_out pointer */
  double noise_sigma;      /* use_noise == 2 */
  uint64_t noise_seed;     /* use_noise == 2 */
  const uint64_t* rows;    /* GRAD_LOGISTIC: n_local * batch global row indices (host), node
                              i's at [i * batch]; NULL: drawn from each node's sample stream
                              (dsgd_ctx_seed_streams), row = begin + uniform_index(end - begin)
                              objectives.cpp:154-157 */
} dsgd_grad_spec;

/* LogisticObjective (objectives.cpp:80-106): features n_samples x d row-major
 * (host, fp64; stored in the context dtype), labels 0/1, l2 > 0.  Replicated
 * per context; every local node samples all rows until
 * dsgd_logistic_set_sample_range.  Errors (DSGD_EINVAL) carry the
 * constructor's messages. */
dsgd_status dsgd_set_logistic(dsgd_ctx* ctx, const double* features, const int32_t* labels,
                              uint64_t n_samples, double l2);
/* LogisticObjective::set_sample_range objectives.cpp:108-114 for one local node */
dsgd_status dsgd_logistic_set_sample_range(dsgd_ctx* ctx, uint32_t local, uint64_t begin,
                                           uint64_t end);

/* ----------------------------------------------------------- update rules
 * All are lock-step over every node of the group and advance each node's t. */

/* local_sgd_step protocols.cpp:102-108, on every node */
dsgd_status dsgd_local_sgd_step(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                const dsgd_grad_spec* g);
/* allreduce_round protocols.cpp:110-131 (one context: pivot-form
 * spatial_mean, bit-exact with param_vec.cpp:19-40; one context per GPU:
 * the mean over NVLink replacing ring_allreduce transport.cpp:183-248 --
 * a one-shot peer-memory kernel (p <= 2, reference ring order, bit-exact),
 * an NVSwitch multimem two-shot (p > 2), a two-shot over peer memory (ring
 * order, bit-exact) or ncclAllReduce (DSGD_ALLREDUCE); theta += avg is
 * deferred into the next round's delta kernel and materialised by any other
 * call). */
dsgd_status dsgd_allreduce_round(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                 const dsgd_grad_spec* g, dsgd_momentum_scope scope);
/* Synchronous EASGD sweep simulator.cpp:332-351 = ea_client_step
 * protocols.cpp:140-153 + ea_server_apply 155-159 in node order; center on
 * the context hosting node 0.  gated = (t > 0 && t % tau == 0). */
dsgd_status dsgd_ea_round(dsgd_ctx* ctx, const dsgd_hyperparams* h, const dsgd_grad_spec* g,
                          int gated);
/* pull_gossip_round protocols.cpp:173-185 (partner_of: p entries);
 * partner_of == NULL runs the ungated branch (local step on every node). */
dsgd_status dsgd_pull_gossip_round(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, const uint32_t* partner_of);
/* push_gossip_round protocols.cpp:230-242 (target_of: p entries, no self) */
dsgd_status dsgd_push_gossip_round(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, const uint32_t* target_of);
/* gated gossip-stale round simulator.cpp:283-292 (gossip_stale_step 252-263) */
dsgd_status dsgd_gossip_stale_round(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                    const dsgd_grad_spec* g, const uint32_t* partner_of);
/* gated gossip-fresh round simulator.cpp:305-319 (gossip_fresh_step 271-276) */
dsgd_status dsgd_gossip_fresh_round(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                    const dsgd_grad_spec* g, const uint32_t* partner_of);
/* async_pull_event protocols.cpp:278-297 (nodes i, j global ids; one context) */
dsgd_status dsgd_async_pull_event(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                  const dsgd_grad_spec* g, uint32_t i, uint32_t j);
/* gossip_stale_step protocols.cpp:252-263 for ONE local node of a single
 * context against an arbitrary device vector `partner` (dtype elements, d):
 * delta' = compute_local_delta(theta_i); theta_i = mix_toward(theta_i,
 * partner, beta_gossip) + delta'; in place, t_i += 1.  (The reference's
 * single-node signature; simulator.cpp:283-292 calls it per node.) */
dsgd_status dsgd_gossip_stale_step(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                   const dsgd_grad_spec* g, uint32_t local, const void* partner);
/* mix_toward protocols.cpp:42-51 for ONE local node, in place:
 * theta_i += beta * (partner - theta_i) (gossip_fresh_mix 265-269). */
dsgd_status dsgd_mix_toward(dsgd_ctx* ctx, uint32_t local, const void* partner, double beta);
/* The point a host Objective is evaluated at by compute_local_delta
 * (protocols.cpp:90-93): out = theta + mu * delta_prev (theta when mu == 0),
 * for one local node, into a device buffer of d dtype elements on the
 * context stream -- the input of an Objective::stochastic_gradient plugin
 * (objectives.hpp:44-49) whose result comes back as DSGD_GRAD_BUFFER. */
dsgd_status dsgd_eval_point(dsgd_ctx* ctx, const dsgd_hyperparams* h, uint32_t local, void* out);
/* pull_mix 161-171 / push_mix 195-228 without the SGD step */
dsgd_status dsgd_pull_mix(dsgd_ctx* ctx, const uint32_t* partner_of);
dsgd_status dsgd_push_mix(dsgd_ctx* ctx, const uint32_t* target_of);
/* gossip_fresh_mix protocols.cpp:265-269 (mix_toward with beta, no step) */
dsgd_status dsgd_gossip_fresh_mix(dsgd_ctx* ctx, const uint32_t* partner_of, double beta);
/* ea_client_step's update output: when update_out != NULL (n_local device
 * pointers), dsgd_ea_round / dsgd_ea_client_event on a single context also
 * write each client's update u_i = beta*(theta_i - c) there. */
dsgd_status dsgd_ea_set_update_out(dsgd_ctx* ctx, void* const* update_out);
/* ea_server_apply protocols.cpp:155-159: center += update (device vector) */
dsgd_status dsgd_ea_server_apply(dsgd_ctx* ctx, const void* update);
/* EASGD center = spatial_mean of the nodes' current theta (simulator.cpp:62-67,
 * pivot form param_vec.cpp:19-40).  One context per GPU: node 0's context reads
 * every rank's theta over NVLink (call after every rank's dsgd_set_state, e.g.
 * behind a host barrier); the others return at once. */
dsgd_status dsgd_ea_init_center(dsgd_ctx* ctx);
/* One client tick of asynchronous EASGD (run_async simulator.cpp:419-428):
 * node i (global id, single context) runs ea_client_step against the center
 * and the server applies its update (gated), or a plain local step. */
dsgd_status dsgd_ea_client_event(dsgd_ctx* ctx, const dsgd_hyperparams* h,
                                 const dsgd_grad_spec* g, uint32_t i, int gated);
/* make_trace_record simulator.cpp:92-123 over all p nodes: consensus error
 * sum_i ||theta_i - mean||^2, mean objective value (quadratic contexts) and
 * sum_i ||theta_i - theta*||^2, fp64 accumulation.  A non-finite parameter
 * returns DSGD_ESTATE ("non-finite parameter", the reference's
 * runtime_error).  One context per GPU: reads every peer's current theta over
 * NVLink once every peer has published its last round (device-side wait). */
dsgd_status dsgd_trace(dsgd_ctx* ctx, double* sq_err_consensus, double* loss_mean,
                       double* sq_err_opt);

/* ------------------------------------------------------ per-step worker loop
 * run_sync simulator.cpp:234-369 / the run_transport worker
 * transport.cpp:342-479, per context: alpha from step_size_at, the gate,
 * partner draws from the reference partner streams (all p, so every
 * context knows the full map), optional reference noise drawn on the host
 * and uploaded, the protocol's fused kernels.  Streams are keyed by
 * (seed, run_id) and persist in the context across calls. */
typedef struct {
  dsgd_protocol protocol;
  dsgd_hyperparams hyper;
  dsgd_momentum_scope scope;
  dsgd_grad_spec grad;
  uint32_t n_grad_pool;          /* >0: round r reads grad_pool[(r % n) * n_local + i] */
  const void* const* grad_pool;
  double host_noise_sigma;       /* >0: reference Gaussian noise drawn on the host per step */
  uint64_t rounds;
} dsgd_run_desc;
dsgd_status dsgd_ctx_seed_streams(dsgd_ctx* ctx, uint64_t seed, const char* run_id);
dsgd_status dsgd_run_rounds(dsgd_ctx* ctx, const dsgd_run_desc* run);
dsgd_status dsgd_ctx_round(dsgd_ctx* ctx, uint64_t* round); /* rounds completed */
/* run_async simulator.cpp:380-449 on one context (all p nodes): `events`
 * ticks of the Poisson master clock (the run-level clock stream of
 * dsgd_ctx_seed_streams: gap ~ Exp(p * rate_per_node), then the ticking
 * node), each one async_pull_event (run->protocol DSGD_ASYNC_PULL; partner
 * from the node's partner stream) or one EASGD client tick (DSGD_ELASTIC_AVG;
 * ea_client_step + ea_server_apply when gated on the node's own t, else a
 * local step).  The clock persists across calls; *sim_time accumulates the
 * gaps and *alpha receives the step size of the last event (the trace
 * record's alpha, simulator.cpp:411). */
dsgd_status dsgd_run_events(dsgd_ctx* ctx, const dsgd_run_desc* run, uint64_t events,
                            double rate_per_node, double* sim_time, double* alpha);

/* ---------------------------------------------- multi-GPU group wiring
 * One context per GPU (n_local == 1).  Each context exports a fixed-size
 * blob (CUDA IPC handle of its state arena + layout; on node 0, when the
 * all-reduce backend is NVLS, the NVSwitch multicast object it created, as
 * its pid + POSIX fd); the host exchanges blobs out of band (e.g.
 * torch.distributed all_gather, a shared mapping) and connects.  Connecting
 * maps every peer's arena and -- for NVLS -- makes every rank join the
 * multicast object (pidfd_getfd, cuMulticastAddDevice, cuMulticastBindMem),
 * agreeing over the mapped peer memory; when any GPU cannot join, every rank
 * stays on the peer-memory two-shot ("p2p").  All ranks call it together. */
dsgd_status dsgd_ctx_export_handle(dsgd_ctx* ctx, void* blob /* DSGD_HANDLE_BYTES */);
dsgd_status dsgd_ctx_connect_peers(dsgd_ctx* ctx, const void* blobs /* p blobs */);
/* In-process group: p one-node contexts (rank r on devices[r], or all on
 * base->device when devices == NULL) created and wired to each other by raw
 * device pointers in this process -- no IPC, no second process.  The host
 * issues every round in node order (rank 0..p-1; the two-shot all-reduce's
 * reduce kernels after every rank's exchange kernel), so every cross-rank
 * flag wait is already satisfied when a kernel starts.  Ranks on one GPU
 * share one stream: the multi-GPU kernels (ring-order all-reduce, EASGD
 * chain, peer-read gossip) then run -- and can be checked -- on a single
 * GPU; ranks on distinct GPUs run over NVLink exactly as with one process
 * per GPU (the shape a single-process profiler capture needs).  out: p
 * contexts in node order (destroy each).  Same-GPU ranks use a 5 s flag
 * timeout. */
dsgd_status dsgd_group_create_inproc(const dsgd_ctx_desc* base, uint32_t p, const int* devices,
                                     dsgd_ctx** out);
/* dsgd_run_rounds over an in-process group: round r of every rank, in node
 * order, then round r+1 (runs: one descriptor per rank, same protocol and
 * round count). */
dsgd_status dsgd_group_run_rounds(dsgd_ctx* const* ctxs, uint32_t n, const dsgd_run_desc* runs);
/* NVLS (in-switch) all-reduce with CALLER-provided buffers (the library sets
 * up its own in dsgd_ctx_connect_peers): `x` and `avg` are this context's
 * d-element slices of a multicast-mapped allocation and `x_mc` / `avg_mc`
 * their multicast addresses.  The multi-GPU all-reduce then reduces with
 * multimem.ld_reduce and broadcasts with multimem.st (summation order: the
 * switch's). */
dsgd_status dsgd_ctx_attach_multicast(dsgd_ctx* ctx, void* x, void* x_mc, void* avg,
                                      void* avg_mc);
/* The multi-GPU all-reduce this context runs: "local" (one context),
 * "oneshot", "nvls", "p2p" or "nccl"; *note says why NVLS is not in use when
 * it was requested (empty otherwise).  Strings owned by the context. */
dsgd_status dsgd_ctx_allreduce_backend(dsgd_ctx* ctx, const char** name, const char** note);
dsgd_status dsgd_nccl_unique_id(void* id /* DSGD_NCCL_ID_BYTES */);
dsgd_status dsgd_ctx_init_nccl(dsgd_ctx* ctx, const void* id, int rank, int nranks);
/* Spin-wait bound for cross-GPU flags (default 30 s). */
dsgd_status dsgd_ctx_set_timeout(dsgd_ctx* ctx, double seconds);

/* ----------------------------------------------------------- measurement */
typedef enum {
  DSGD_K_STEP = 0,       /* fused local step / pull / stale / mix kernels */
  DSGD_K_ALLREDUCE = 1,  /* single-context fused all-reduce round */
  DSGD_K_AR_DELTA = 2,   /* multi-GPU all-reduce: delta kernel */
  DSGD_K_AR_APPLY = 3,   /* multi-GPU all-reduce: apply kernel */
  DSGD_K_NCCL = 4,       /* all-reduce exchange: ncclAllReduce or the peer-memory reduce kernel */
  DSGD_K_EA = 5,         /* EASGD fused chain */
  DSGD_K_PUSH = 6,
  DSGD_K_OTHER = 7,
  DSGD_K_COUNT = 8
} dsgd_kernel_id;
/* When enabled, every launch is bracketed by CUDA events on the context
 * stream; read accumulates device time per kernel id (and syncs). */
dsgd_status dsgd_profile_enable(dsgd_ctx* ctx, int enable);
dsgd_status dsgd_profile_read(dsgd_ctx* ctx, dsgd_kernel_id k, double* total_ms,
                              uint64_t* launches, int reset);
/* DSGD_TRACE=<n> (environment) records up to n launches of the multi-GPU
 * kernels: 5 u64 per record {kernel id (+16 * pipeline), round, %globaltimer
 * at entry, after the cross-GPU wait, when the last CTA signalled}. */
dsgd_status dsgd_trace_dump(dsgd_ctx* ctx, uint64_t* out, uint32_t max_records, uint32_t* n);
/* Number of kernels (and NCCL calls) this context has launched. */
dsgd_status dsgd_launch_count(dsgd_ctx* ctx, uint64_t* kernels, uint64_t* nccl_calls);

#ifdef __cplusplus
}
#endif

#endif /* DSGD_B200_H_ */
