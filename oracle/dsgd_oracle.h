/*
 * dsgd_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference `dsgd` update rules (arXiv 1611.04581
 * reference, /root/reference/proj) used as the CHECKER for the B200 product
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product
 * (paper_1611_04581_b200/) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit (fp64) against
 * the reference sources compiled in oracle/_ref (oracle/Makefile) and against
 * the reference's own golden values (tests/test_oracle_golden.py).
 *
 * Two precisions are provided: *_f64 follows the reference arithmetic exactly
 * (no FMA contraction: built with -ffp-contract=off, the reference objects
 * contain no vfmadd), *_f32 runs the identical operation order in binary32,
 * which is what the GPU fp32 kernels must reproduce bit-for-bit.
 */
#ifndef DSGD_ORACLE_H_
#define DSGD_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + reference samplers (rng.hpp:50-85, rng.cpp) */
typedef struct {
  uint64_t mt[312];
  uint32_t idx;
} dsgdo_rng;

enum {
  DSGDO_PURPOSE_NOISE = 0,   /* "gradient-noise" */
  DSGDO_PURPOSE_SAMPLE = 1,  /* "sample" */
  DSGDO_PURPOSE_PARTNER = 2, /* "partner-choice" */
  DSGDO_PURPOSE_CLOCK = 3,   /* "clock" */
  DSGDO_PURPOSE_STRAGGLER = 4,
  DSGDO_PURPOSE_INIT = 5
};

void dsgdo_rng_seed(dsgdo_rng* r, uint64_t seed);
uint64_t dsgdo_rng_next(dsgdo_rng* r);
double dsgdo_uniform01(dsgdo_rng* r);
double dsgdo_normal(dsgdo_rng* r);
double dsgdo_exponential(dsgdo_rng* r, double rate);
void dsgdo_fill_normal(dsgdo_rng* r, double sigma, double* out, uint64_t n);
uint32_t dsgdo_uniform_index(dsgdo_rng* r, uint32_t n);
uint64_t dsgdo_derive_stream_seed(uint64_t root_seed, const char* run_id,
                                  uint32_t node_id, int purpose);
void dsgdo_make_stream(dsgdo_rng* r, uint64_t root_seed, const char* run_id,
                       uint32_t node_id, int purpose);

/* ---- hyperparameters (core.hpp:54-70) and schedule (core.cpp:82-92) */
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
  uint32_t batch; /* minibatch size b (core.hpp:63; LogisticObjective only) */
} dsgdo_hyper;

double dsgdo_step_size_at(const dsgdo_hyper* h, uint64_t t);

/* Partner draws (simulator.cpp:69-88): out[i] for each node in order from
 * that node's partner stream. */
void dsgdo_draw_pull_partners(dsgdo_rng* partner_streams, uint32_t p, uint32_t* out);
void dsgdo_draw_push_targets(dsgdo_rng* partner_streams, uint32_t p, uint32_t* out);

/* Schedule generator used by the tests: partners for `rounds` rounds of a
 * pull-gossip run_sync (gated rounds only draw; ungated rows are all
 * 0xffffffff). out is rounds*p. */
void dsgdo_pull_schedule(uint64_t seed, const char* run_id, uint32_t p, uint32_t tau,
                         uint64_t rounds, uint32_t* out);

/* ---- objective / noise selection for the primitives.
 * kind 0 = diagonal quadratic g = s*(x - opt) (objectives.cpp:71-78),
 * kind 1 = fixed gradient (an Objective whose stochastic_gradient returns
 *          a given vector; the plugin slot the GPU's external-gradient mode
 *          fills).  For per-node objectives `grad` is p*d. */
enum { DSGDO_OBJ_QUADRATIC = 0, DSGDO_OBJ_FIXED = 1, DSGDO_OBJ_LOGISTIC = 2 /* ref_shim only */ };

/* ---- LogisticObjective (objectives.cpp:80-162).  Minibatch rows are drawn
 * by the caller from the node's sample stream, in batch order:
 *   row = begin + uniform_index(end - begin)          (objectives.cpp:154-157)
 * dsgdo_draw_rows does exactly that.  The logistic gradient itself is
 * dsgdo_logistic_grad_{f64,f32} below. */
void dsgdo_draw_rows(dsgdo_rng* sample, uint64_t begin, uint64_t end, uint32_t batch,
                     uint64_t* rows);
double dsgdo_sigmoid(double z);
/* LogisticObjective::value objectives.cpp:116-125 (fp64): mean over all rows
 * of log1pexp(z) - y z, plus 0.5 l2 ||theta||^2 */
double dsgdo_logistic_value(uint64_t n, uint64_t d, const double* X, const int32_t* y, double l2,
                            const double* theta);

/* ---- run drivers (simulator.cpp run_sync 214-374 / run_async 380-449) */
enum {
  DSGDO_ALLREDUCE = 0,
  DSGDO_ELASTIC = 1,
  DSGDO_PULL = 2,
  DSGDO_PUSH = 3,
  DSGDO_STALE = 4,
  DSGDO_FRESH = 5,
  DSGDO_ASYNC_PULL = 6
};
enum { DSGDO_INIT_ZEROS = 0, DSGDO_INIT_OFFSET_ONES = 1, DSGDO_INIT_GAUSSIAN = 2, DSGDO_INIT_EXPLICIT = 3 };

typedef struct {
  int protocol;
  uint32_t p;
  uint64_t d;
  dsgdo_hyper hyper;
  int noise_gaussian; /* 0: NoiseModel::zero, 1: gaussian with per-coord sigma */
  double sigma;
  const double* spectrum; /* quadratic objective, d entries */
  const double* opt;      /* d entries */
  int init_kind;
  double target_sq_err;
  double init_scale;
  const double* init_values; /* explicit init, d entries */
  int scope_per_node;        /* all-reduce momentum scope: 0 aggregate, 1 per-node */
  int poisson;               /* elastic-avg: run under the poisson clock (run_async) */
  uint64_t rounds;           /* sync horizon */
  uint64_t events;           /* async horizon */
  double rate_per_node;
  uint64_t seed;
  const char* run_id;
} dsgdo_sim;

#define DSGDO_DECLARE(SFX, R)                                                              \
  void dsgdo_local_delta_##SFX(uint64_t d, const R* theta, const R* dprev, int obj_kind,  \
                               const R* spec, const R* opt, const R* gfixed,              \
                               const R* noise, double alpha, double mu, double wd,        \
                               R* out);                                                   \
  void dsgdo_local_sgd_step_##SFX(uint64_t d, R* theta, R* dprev, uint64_t* t,           \
                                  int obj_kind, const R* spec, const R* opt,             \
                                  const R* gfixed, const R* noise,                        \
                                  const dsgdo_hyper* h);                                  \
  void dsgdo_spatial_mean_##SFX(uint32_t p, uint64_t d, const R* x, R* out);             \
  void dsgdo_allreduce_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev,           \
                                   uint64_t* t, int obj_kind, const R* spec,              \
                                   const R* opt, const R* gfixed, const R* noise,         \
                                   const dsgdo_hyper* h, int per_node, R* avg_out);       \
  void dsgdo_ring_allreduce_##SFX(uint32_t p, uint64_t d, const R* in, R* out);          \
  void dsgdo_ea_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev, uint64_t* t,     \
                            R* center, int gated, int obj_kind, const R* spec,            \
                            const R* opt, const R* gfixed, const R* noise,                \
                            const dsgdo_hyper* h);                                        \
  void dsgdo_pull_mix_##SFX(uint32_t p, uint64_t d, R* theta, const uint32_t* partner);  \
  void dsgdo_pull_gossip_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev,         \
                                     uint64_t* t, const uint32_t* partner, int obj_kind,  \
                                     const R* spec, const R* opt, const R* gfixed,        \
                                     const R* noise, const dsgdo_hyper* h);               \
  int dsgdo_push_mix_##SFX(uint32_t p, uint64_t d, R* theta, const uint32_t* target);    \
  int dsgdo_push_gossip_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev,          \
                                    uint64_t* t, const uint32_t* target, int obj_kind,    \
                                    const R* spec, const R* opt, const R* gfixed,         \
                                    const R* noise, const dsgdo_hyper* h);                \
  void dsgdo_stale_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev, uint64_t* t,  \
                               const uint32_t* partner, int obj_kind, const R* spec,      \
                               const R* opt, const R* gfixed, const R* noise,             \
                               const dsgdo_hyper* h);                                     \
  void dsgdo_fresh_round_##SFX(uint32_t p, uint64_t d, R* theta, R* dprev, uint64_t* t,  \
                               const uint32_t* partner, int obj_kind, const R* spec,      \
                               const R* opt, const R* gfixed, const R* noise,             \
                               const dsgdo_hyper* h);                                     \
  void dsgdo_async_pull_event_##SFX(uint32_t p, uint64_t d, R* theta, uint64_t* t,       \
                                    uint32_t i, uint32_t j, int obj_kind, const R* spec,  \
                                    const R* opt, const R* gfixed, const R* noise,        \
                                    const dsgdo_hyper* h);                                \
  void dsgdo_logistic_grad_##SFX(uint64_t d, const R* X, const int32_t* y, double l2,    \
                                  const R* theta, uint32_t batch, const uint64_t* rows,   \
                                  R* out);                                                \
  int dsgdo_run_##SFX(const dsgdo_sim* cfg, R* theta_out, R* dprev_out, uint64_t* t_out, \
                      R* center_out);                                                     \
  void dsgdo_trace_##SFX(uint32_t p, uint64_t d, const R* theta, const R* spec,          \
                         const R* opt, double* sq_err_consensus, double* loss_mean,       \
                         double* sq_err_opt);

DSGDO_DECLARE(f64, double)
DSGDO_DECLARE(f32, float)

#ifdef __cplusplus
}
#endif

#endif /* DSGD_ORACLE_H_ */
