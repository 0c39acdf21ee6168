// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference sources
// (/root/reference/proj/src/{rng,param_vec,core,objectives,protocols,
// simulator,transport}.cpp), compiled by oracle/Makefile into
// oracle/_ref/libdsgd_ref.so.  Used (a) to pin the C restatement in
// oracle/dsgd_oracle.c bit-for-bit and (b) as the reference CPU arm of
// bench.py.  Nothing here is product code; nothing is copied from the
// reference -- this file only calls its public API (protocols.hpp,
// simulator.hpp, transport.hpp).
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "dsgd/core.hpp"
#include "dsgd/objectives.hpp"
#include "dsgd/protocols.hpp"
#include "dsgd/rng.hpp"
#include "dsgd/simulator.hpp"
#include "dsgd/transport.hpp"
#include "dsgd_oracle.h"
#ifdef REF_HAVE_TRACE_IO
#include "dsgd/trace_io.hpp"
#endif
#ifdef REF_B200_RESIDENT  // the integration harness: run_sync with the state on the GPU
#include "run_sync_b200.hpp"
#endif

using namespace dsgd;

namespace {

// An Objective whose stochastic gradient is a fixed vector: the reference's
// plugin slot (objectives.hpp:33-53) filled the way the GPU path's external
// gradient buffer fills it.
class FixedGradientObjective : public Objective {
 public:
  explicit FixedGradientObjective(std::vector<double> g) : g_(std::move(g)) {}
  std::size_t dim() const override { return g_.size(); }
  double value(const ParamVec&) const override { return 0.0; }
  ParamVec gradient(const ParamVec&) const override { return ParamVec(g_); }
  std::pair<double, double> convexity_params() const override { return {1.0, 1.0}; }

 private:
  std::vector<double> g_;
};

// A pool of synthetic N(0, 1) gradient vectors served in turn through the
// plugin slot (thread-safe: run_transport's workers share one objective).
class PoolGradientObjective : public Objective {
 public:
  PoolGradientObjective(std::size_t d, std::size_t n) : d_(d) {
    for (std::size_t k = 0; k < n; ++k) {
      RngStream s(0x9001 + k);
      std::vector<double> g(d);
      for (double& x : g) x = s.normal();
      pool_.emplace_back(std::move(g));
    }
  }
  std::size_t dim() const override { return d_; }
  double value(const ParamVec&) const override { return 0.0; }
  ParamVec gradient(const ParamVec&) const override {
    return pool_[next_.fetch_add(1) % pool_.size()];
  }
  std::pair<double, double> convexity_params() const override { return {1.0, 1.0}; }

 private:
  std::size_t d_;
  std::vector<ParamVec> pool_;
  mutable std::atomic<std::size_t> next_{0};
};

thread_local std::string g_err;

Hyperparams to_hyper(const dsgdo_hyper& h) {
  Hyperparams out;
  out.alpha0 = h.alpha0;
  out.anneal_factor = h.anneal_factor;
  out.anneal_at.assign(h.anneal_at, h.anneal_at + h.n_anneal);
  out.mu = h.mu;
  out.weight_decay = h.weight_decay;
  out.beta_gossip = h.beta_gossip;
  out.beta_ea = h.beta_ea;
  out.tau = h.tau;
  out.batch = h.batch == 0 ? 1 : h.batch;
  return out;
}

ProtocolKind to_protocol(int p) {
  switch (p) {
    case DSGDO_ALLREDUCE: return ProtocolKind::kAllReduce;
    case DSGDO_ELASTIC: return ProtocolKind::kElasticAvg;
    case DSGDO_PULL: return ProtocolKind::kPullGossip;
    case DSGDO_PUSH: return ProtocolKind::kPushGossip;
    case DSGDO_STALE: return ProtocolKind::kGossipStale;
    case DSGDO_FRESH: return ProtocolKind::kGossipFresh;
    default: return ProtocolKind::kAsyncPull;
  }
}

SimConfig to_sim(const dsgdo_sim& c) {
  SimConfig cfg;
  cfg.protocol = to_protocol(c.protocol);
  cfg.p = c.p;
  cfg.hyper = to_hyper(c.hyper);
  cfg.noise = c.noise_gaussian ? NoiseModel::gaussian_per_coord(c.sigma, c.d)
                               : NoiseModel::zero(c.d);
  switch (c.init_kind) {
    case DSGDO_INIT_ZEROS: cfg.init.kind = InitSpec::Kind::kZeros; break;
    case DSGDO_INIT_OFFSET_ONES: cfg.init.kind = InitSpec::Kind::kOffsetOnes; break;
    case DSGDO_INIT_GAUSSIAN: cfg.init.kind = InitSpec::Kind::kGaussianSpread; break;
    default:
      cfg.init.kind = InitSpec::Kind::kExplicit;
      cfg.init.values.assign(c.init_values, c.init_values + c.d);
  }
  cfg.init.target_sq_err = c.target_sq_err;
  cfg.init.scale = c.init_scale;
  cfg.momentum_scope = c.scope_per_node ? MomentumScope::kPerNode : MomentumScope::kAggregate;
  if (c.protocol == DSGDO_ASYNC_PULL || c.poisson) {
    cfg.clock.kind = ClockModel::Kind::kPoisson;
    cfg.clock.rate_per_node = c.rate_per_node;
  }
  cfg.rounds = c.rounds;
  cfg.events = c.events;
  cfg.trace_every = 1u << 30;
  cfg.seed = c.seed;
  cfg.run_id = c.run_id;
  return cfg;
}

// LogisticObjective dataset for obj_kind DSGDO_OBJ_LOGISTIC (ref_set_logistic);
// node i samples rows [ranges[2i], ranges[2i+1]) (LogisticObjective::set_sample_range).
struct LogisticData {
  bool set = false;
  std::vector<std::vector<double>> X;
  std::vector<int> y;
  double l2 = 0.0;
  std::vector<std::uint64_t> ranges;
};
LogisticData g_logistic;

std::unique_ptr<LogisticObjective> logistic_for(std::uint32_t node) {
  auto o = std::make_unique<LogisticObjective>(g_logistic.X, g_logistic.y, g_logistic.l2);
  if (!g_logistic.ranges.empty())
    o->set_sample_range(g_logistic.ranges[2 * node], g_logistic.ranges[2 * node + 1]);
  return o;
}

void export_nodes(const std::vector<NodeState>& nodes, std::uint64_t d, double* theta,
                  double* dprev, std::uint64_t* t) {
  for (std::size_t i = 0; i < nodes.size(); ++i) {
    std::memcpy(theta + i * d, nodes[i].theta.raw(), sizeof(double) * d);
    if (dprev) std::memcpy(dprev + i * d, nodes[i].delta_prev.raw(), sizeof(double) * d);
    if (t) t[i] = nodes[i].t;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_derive_stream_seed(std::uint64_t seed, const char* run_id, std::uint32_t node,
                                     int purpose) {
  return derive_stream_seed(seed, run_id, node, static_cast<StreamPurpose>(purpose));
}

// Raw draws and samplers from one stream: kind 0 next_u64 (as bits in a
// double array via memcpy), 1 uniform01, 2 normal, 3 uniform_index(n),
// 4 exponential(rate = n).
void ref_stream_draws(std::uint64_t seed, int kind, std::uint32_t n, std::uint64_t count,
                      void* out) {
  RngStream s(seed);
  for (std::uint64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: static_cast<std::uint64_t*>(out)[i] = s.next_u64(); break;
      case 1: static_cast<double*>(out)[i] = s.uniform01(); break;
      case 2: static_cast<double*>(out)[i] = s.normal(); break;
      case 3: static_cast<std::uint64_t*>(out)[i] = s.uniform_index(n); break;
      default: static_cast<double*>(out)[i] = s.exponential(static_cast<double>(n)); break;
    }
  }
}

// LogisticObjective dataset used by ref_round (obj_kind 2) and ref_run while
// set: X is n*d row-major, labels 0/1, ranges (optional) 2*p sample ranges.
int ref_set_logistic(const double* X, const std::int32_t* y, std::uint64_t n, std::uint64_t d,
                     double l2, const std::uint64_t* ranges, std::uint32_t p) {
  try {
    g_logistic = LogisticData{};
    for (std::uint64_t r = 0; r < n; ++r) {
      g_logistic.X.emplace_back(X + r * d, X + (r + 1) * d);
      g_logistic.y.push_back(y[r]);
    }
    g_logistic.l2 = l2;
    if (ranges) g_logistic.ranges.assign(ranges, ranges + 2 * p);
    (void)LogisticObjective(g_logistic.X, g_logistic.y, l2);  // the constructor's checks
    g_logistic.set = true;
    return 0;
  } catch (const std::exception& e) {
    g_logistic = LogisticData{};
    g_err = e.what();
    return -1;
  }
}

void ref_clear_logistic() { g_logistic = LogisticData{}; }

// LogisticObjective::stochastic_gradient(theta, batch, RngStream(sample_seed))
// on rows [begin, end).
int ref_logistic_grad(const double* theta, std::uint64_t d, std::uint32_t batch,
                      std::uint64_t sample_seed, std::uint64_t begin, std::uint64_t end,
                      double* out) {
  try {
    LogisticObjective o(g_logistic.X, g_logistic.y, g_logistic.l2);
    o.set_sample_range(begin, end);
    RngStream s(sample_seed);
    const ParamVec g =
        o.stochastic_gradient(ParamVec(std::vector<double>(theta, theta + d)), batch, s);
    std::memcpy(out, g.raw(), sizeof(double) * d);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// LogisticObjective::value on the installed dataset.
double ref_logistic_value(const double* theta, std::uint64_t d) {
  LogisticObjective o(g_logistic.X, g_logistic.y, g_logistic.l2);
  return o.value(ParamVec(std::vector<double>(theta, theta + d)));
}

// Full run through the reference drivers (run_simulation). Returns 0, or -1
// with ref_last_error() set when the reference throws.
int ref_run(const dsgdo_sim* c, double* theta, double* dprev, std::uint64_t* t,
            double* center) {
  try {
    const SimConfig cfg = to_sim(*c);
    RunResult r;
    if (g_logistic.set) {  // sharded logistic objectives (runner.cpp:100-115 shape)
      LogisticObjective eval(g_logistic.X, g_logistic.y, g_logistic.l2);
      std::vector<std::unique_ptr<LogisticObjective>> own;
      std::vector<const Objective*> objs;
      for (std::uint32_t i = 0; i < c->p; ++i) {
        own.push_back(logistic_for(i));
        objs.push_back(own.back().get());
      }
      r = (cfg.clock.kind == ClockModel::Kind::kPoisson) ? run_async(cfg, eval, objs)
                                                         : run_sync(cfg, eval, objs);
    } else {
      QuadraticObjective obj(std::vector<double>(c->spectrum, c->spectrum + c->d),
                             ParamVec(std::vector<double>(c->opt, c->opt + c->d)));
      r = run_simulation(cfg, obj);
    }
    export_nodes(r.final_nodes, c->d, theta, dprev, t);
    if (center && r.final_server) {
      std::memcpy(center, r.final_server->theta_center.raw(), sizeof(double) * c->d);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_simulation with trace_every: the trace records as rows of
// {t, sim_time (NaN: none), sq_err_opt (NaN: none), sq_err_consensus,
// loss_mean, alpha} and, when trace_io.cpp is compiled in, the JSONL text
// of write_trace_jsonl (trace_io.cpp:40-51).  Returns the record count or -1.
long ref_run_traced(const dsgdo_sim* c, std::uint64_t trace_every, double* rec,
                    std::uint64_t max_rec, char* jsonl, std::uint64_t jsonl_cap) {
  try {
    SimConfig cfg = to_sim(*c);
    cfg.trace_every = trace_every;
    RunResult r;
    if (g_logistic.set) {
      LogisticObjective eval(g_logistic.X, g_logistic.y, g_logistic.l2);
      std::vector<std::unique_ptr<LogisticObjective>> own;
      std::vector<const Objective*> objs;
      for (std::uint32_t i = 0; i < c->p; ++i) {
        own.push_back(logistic_for(i));
        objs.push_back(own.back().get());
      }
      r = (cfg.clock.kind == ClockModel::Kind::kPoisson) ? run_async(cfg, eval, objs)
                                                         : run_sync(cfg, eval, objs);
    } else {
      QuadraticObjective obj(std::vector<double>(c->spectrum, c->spectrum + c->d),
                             ParamVec(std::vector<double>(c->opt, c->opt + c->d)));
      r = run_simulation(cfg, obj);
    }
    const double nan = std::numeric_limits<double>::quiet_NaN();
    std::string text;
    for (std::size_t k = 0; k < r.trace.size() && k < max_rec; ++k) {
      const TraceRecord& t = r.trace[k];
      double* o = rec + 6 * k;
      o[0] = static_cast<double>(t.t);
      o[1] = t.sim_time.value_or(nan);
      o[2] = t.sq_err_opt.value_or(nan);
      o[3] = t.sq_err_consensus;
      o[4] = t.loss_mean;
      o[5] = t.alpha;
#ifdef REF_HAVE_TRACE_IO
      text += trace_record_to_json_line(t);
      text += "\n";
#endif
    }
    if (jsonl && jsonl_cap) {
      const std::size_t n = std::min<std::size_t>(text.size(), jsonl_cap - 1);
      std::memcpy(jsonl, text.data(), n);
      jsonl[n] = 0;
    }
    return static_cast<long>(r.trace.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

#ifdef REF_B200_RESIDENT
// integration/run_sync_b200.cpp: run_sync with the node state resident on
// the GPU (one dsgd_run_rounds); also returns max_grad_norm.
int ref_run_resident(const dsgdo_sim* c, double* theta, double* dprev, std::uint64_t* t,
                     double* center, double* max_grad_norm) {
  try {
    const SimConfig cfg = to_sim(*c);
    QuadraticObjective obj(std::vector<double>(c->spectrum, c->spectrum + c->d),
                           ParamVec(std::vector<double>(c->opt, c->opt + c->d)));
    const RunResult r = dsgd_b200::run_sync_resident(cfg, obj);
    export_nodes(r.final_nodes, c->d, theta, dprev, t);
    if (center && r.final_server)
      std::memcpy(center, r.final_server->theta_center.raw(), sizeof(double) * c->d);
    if (max_grad_norm) *max_grad_norm = r.max_grad_norm;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
#endif

// run_simulation's max_grad_norm (run_sync passes &result.max_grad_norm
// to every rule, simulator.cpp:239-344).
int ref_run_max_grad_norm(const dsgdo_sim* c, double* max_grad_norm) {
  try {
    const SimConfig cfg = to_sim(*c);
    QuadraticObjective obj(std::vector<double>(c->spectrum, c->spectrum + c->d),
                           ParamVec(std::vector<double>(c->opt, c->opt + c->d)));
    *max_grad_norm = run_simulation(cfg, obj).max_grad_norm;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Threaded transport backend (run_transport): the reference's own parallel
// per-rank worker loop.
int ref_run_transport(const dsgdo_sim* c, double* theta, double* dprev, std::uint64_t* t,
                      double* center, std::uint64_t chaos_seed) {
  try {
    const SimConfig cfg = to_sim(*c);
    QuadraticObjective obj(std::vector<double>(c->spectrum, c->spectrum + c->d),
                           ParamVec(std::vector<double>(c->opt, c->opt + c->d)));
    TransportOptions opt;
    opt.chaos_seed = chaos_seed;
    const RunResult r = run_transport(cfg, obj, opt);
    export_nodes(r.final_nodes, c->d, theta, dprev, t);
    if (center && r.final_server) {
      std::memcpy(center, r.final_server->theta_center.raw(), sizeof(double) * c->d);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One round of a protocol from explicit node states.  Node i's streams are
// make_node(i, theta, seed, run_id)'s, so noise draws are the first ones of
// (seed, run_id, i, gradient-noise).  obj_kind 0: shared quadratic (spec,
// opt); 1: per-node fixed gradients gfixed (p*d).  protocol selects:
//   0 allreduce_round(scope), 1 EA sweep (gated), 2 pull_gossip_round,
//   3 push_gossip_round, 4 stale (per node vs snapshot), 5 fresh,
//   6 async_pull_event(i = aux0, j = aux1), 7 local_sgd_step on every node,
//   8 pull_mix, 9 push_mix.
int ref_round(int protocol, std::uint32_t p, std::uint64_t d, double* theta, double* dprev,
              std::uint64_t* t, const std::uint32_t* partner, int obj_kind, const double* spec,
              const double* opt, const double* gfixed, int noise_gaussian, double sigma,
              std::uint64_t seed, const char* run_id, const dsgdo_hyper* hp, int per_node,
              double* center, int gated, std::uint32_t aux0, std::uint32_t aux1) {
  try {
    const Hyperparams h = to_hyper(*hp);
    const NoiseModel noise =
        noise_gaussian ? NoiseModel::gaussian_per_coord(sigma, d) : NoiseModel::zero(d);
    std::vector<std::unique_ptr<Objective>> own;
    std::vector<const Objective*> objs;
    for (std::uint32_t i = 0; i < p; ++i) {
      if (obj_kind == DSGDO_OBJ_QUADRATIC) {
        own.push_back(std::make_unique<QuadraticObjective>(
            std::vector<double>(spec, spec + d), ParamVec(std::vector<double>(opt, opt + d))));
      } else if (obj_kind == DSGDO_OBJ_LOGISTIC) {
        own.push_back(logistic_for(i));
      } else {
        own.push_back(std::make_unique<FixedGradientObjective>(
            std::vector<double>(gfixed + i * d, gfixed + (i + 1) * d)));
      }
      objs.push_back(own.back().get());
    }
    std::vector<NodeState> nodes;
    for (std::uint32_t i = 0; i < p; ++i) {
      NodeState n = make_node(i, ParamVec(std::vector<double>(theta + i * d, theta + (i + 1) * d)),
                              seed, run_id);
      n.delta_prev = ParamVec(std::vector<double>(dprev + i * d, dprev + (i + 1) * d));
      n.t = t[i];
      nodes.push_back(std::move(n));
    }
    const std::span<const Objective* const> objspan(objs);
    const std::span<const std::uint32_t> pm(partner, partner ? p : 0);
    switch (protocol) {
      case 0:
        nodes = allreduce_round(std::move(nodes), objspan, noise, h,
                                per_node ? MomentumScope::kPerNode : MomentumScope::kAggregate);
        break;
      case 1: {
        ServerState server{ParamVec(std::vector<double>(center, center + d)), 0};
        for (std::uint32_t i = 0; i < p; ++i) {
          if (gated) {
            auto [node, update] = ea_client_step(std::move(nodes[i]), server.theta_center,
                                                 *objs[i], noise, h);
            nodes[i] = std::move(node);
            server = ea_server_apply(std::move(server), update);
          } else {
            nodes[i] = local_sgd_step(std::move(nodes[i]), *objs[i], noise, h);
          }
        }
        std::memcpy(center, server.theta_center.raw(), sizeof(double) * d);
        break;
      }
      case 2: nodes = pull_gossip_round(std::move(nodes), pm, objspan, noise, h); break;
      case 3: nodes = push_gossip_round(std::move(nodes), pm, objspan, noise, h); break;
      case 4: {
        std::vector<ParamVec> snap;
        for (const NodeState& n : nodes) snap.push_back(n.theta);
        for (std::uint32_t i = 0; i < p; ++i)
          nodes[i] = gossip_stale_step(std::move(nodes[i]), snap[partner[i]], *objs[i], noise, h);
        break;
      }
      case 5: {
        for (std::uint32_t i = 0; i < p; ++i)
          nodes[i] = local_sgd_step(std::move(nodes[i]), *objs[i], noise, h);
        std::vector<ParamVec> stepped;
        for (const NodeState& n : nodes) stepped.push_back(n.theta);
        for (std::uint32_t i = 0; i < p; ++i)
          nodes[i] = gossip_fresh_mix(std::move(nodes[i]), stepped[partner[i]], h.beta_gossip);
        break;
      }
      case 6:
        nodes = async_pull_event(std::move(nodes), aux0, aux1, *objs[aux0], noise, h);
        break;
      case 7:
        for (std::uint32_t i = 0; i < p; ++i)
          nodes[i] = local_sgd_step(std::move(nodes[i]), *objs[i], noise, h);
        break;
      case 8: nodes = pull_mix(std::move(nodes), pm); break;
      case 9: nodes = push_mix(std::move(nodes), pm); break;
      default: g_err = "bad protocol"; return -1;
    }
    export_nodes(nodes, d, theta, dprev, t);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ring_allreduce over p threads on an in-process Network (transport.cpp
// 183-248); in/out are p*d.
int ref_ring_allreduce(std::uint32_t p, std::uint64_t d, const double* in, double* out,
                       std::uint64_t chaos_seed) {
  try {
    Network net(p);
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errs(p);
    for (std::uint32_t r = 0; r < p; ++r) {
      threads.emplace_back([&, r] {
        try {
          Endpoint ep(&net, r, std::chrono::milliseconds(60000), chaos_seed);
          const auto res =
              ring_allreduce(ep, p, std::vector<double>(in + r * d, in + (r + 1) * d), 0);
          std::memcpy(out + r * d, res.data(), sizeof(double) * d);
        } catch (...) {
          errs[r] = std::current_exception();
        }
      });
    }
    for (auto& th : threads) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CPU-baseline timing: `rounds` rounds of one protocol through the reference
// update rules on p nodes of dimension d (quadratic objective, spectrum 1,
// optimum 0; nodes at N(0,1) spread; zero noise; the bench's hyperparams).
// mode 0: single-thread simulator rules (allreduce_round / pull_gossip_round
// with the seeded partner streams / EA sweep, gated every round after 0);
// mode 1: the threaded transport backend run_transport (p worker threads,
// +1 EA server thread).  Returns seconds for all rounds, or -1.
}  // extern "C"

namespace {
// Rounds of the compiled reference, timed.  `sync` (sharded runs): every
// shard's thread arrives there right before its first timed round and right
// after its last, so the clock covers the rounds of all shards together.
double time_rounds_impl(int protocol, std::uint32_t p, std::uint64_t d, std::uint64_t rounds,
                        int mode, const dsgdo_hyper* hp, int grad_kind,
                        std::barrier<>* sync) {
  try {
    dsgdo_sim c{};
    c.protocol = protocol;
    c.p = p;
    c.d = d;
    c.hyper = *hp;
    std::vector<double> spec(d, 1.0), opt(d, 0.0);
    c.spectrum = spec.data();
    c.opt = opt.data();
    c.init_kind = DSGDO_INIT_GAUSSIAN;
    c.init_scale = 1.0;
    c.rounds = rounds;
    c.seed = 1;
    c.run_id = "run/trial0";
    SimConfig cfg = to_sim(c);
    // grad_kind 0: QuadraticObjective(spectrum 1, optimum 0); 1: a pool of 4
    // synthetic N(0, 1) gradient vectors served in turn through the
    // Objective plugin slot (the GPU bench's external-gradient pool)
    QuadraticObjective quad(spec, ParamVec(opt));
    std::unique_ptr<PoolGradientObjective> pool;
    if (grad_kind == 1) pool = std::make_unique<PoolGradientObjective>(d, 4);
    const Objective& obj = grad_kind == 1 ? static_cast<const Objective&>(*pool)
                                          : static_cast<const Objective&>(quad);
    using clk = std::chrono::steady_clock;
    if (mode == 1) {
      // run_transport also builds the initial nodes and trace records; time
      // `rounds + 1` and 1 round and keep the difference (per-round cost).
      cfg.rounds = rounds + 1;
      auto t0 = clk::now();
      (void)run_transport(cfg, obj);
      const double tl = std::chrono::duration<double>(clk::now() - t0).count();
      cfg.rounds = 1;
      t0 = clk::now();
      (void)run_transport(cfg, obj);
      const double ts = std::chrono::duration<double>(clk::now() - t0).count();
      return tl - ts;
    }
    // Single-thread simulator rules, dispatched exactly as run_sync does
    // (simulator.cpp:234-351) on gated rounds; nodes built outside the clock.
    std::vector<NodeState> nodes = make_initial_nodes(cfg, obj);
    ServerState server;
    {
      std::vector<ParamVec> th;
      for (const NodeState& n : nodes) th.push_back(n.theta);
      server = ServerState{spatial_mean(th), 0};
    }
    const Hyperparams& h = cfg.hyper;
    std::vector<std::uint32_t> partners(p);
    if (sync) sync->arrive_and_wait();
    const auto t0 = clk::now();
    for (std::uint64_t r = 1; r <= rounds; ++r) {  // r > 0: every round gated (tau = 1)
      switch (protocol) {
        case DSGDO_ALLREDUCE:
          nodes = allreduce_round(std::move(nodes), obj, cfg.noise, h, cfg.momentum_scope);
          break;
        case DSGDO_PULL:
          for (std::uint32_t i = 0; i < p; ++i) partners[i] = nodes[i].rng.partner.uniform_index(p);
          nodes = pull_gossip_round(std::move(nodes), partners, obj, cfg.noise, h);
          break;
        case DSGDO_ELASTIC:
          for (std::uint32_t i = 0; i < p; ++i) {
            auto [node, update] =
                ea_client_step(std::move(nodes[i]), server.theta_center, obj, cfg.noise, h);
            nodes[i] = std::move(node);
            server = ea_server_apply(std::move(server), update);
          }
          break;
        default:
          for (NodeState& n : nodes) n = local_sgd_step(std::move(n), obj, cfg.noise, h);
      }
    }
    if (sync) sync->arrive_and_wait();
    return std::chrono::duration<double>(clk::now() - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    if (sync) sync->arrive_and_drop();
    return -1.0;
  }
}
}  // namespace

extern "C" {

double ref_time_rounds(int protocol, std::uint32_t p, std::uint64_t d, std::uint64_t rounds,
                       int mode, const dsgdo_hyper* hp, int grad_kind) {
  return time_rounds_impl(protocol, p, d, rounds, mode, hp, grad_kind, nullptr);
}

// The same rounds on every host thread: d split into `shards` coordinate
// ranges (every rule of this path is coordinate-separable), each shard an
// independent reference run on its own thread -- the reference's own code
// using all the cores a host gives it.  Simulator rules only (mode 0): the
// clock spans the rounds of all shards (start / end barriers).
double ref_time_rounds_sharded(int protocol, std::uint32_t p, std::uint64_t d,
                               std::uint64_t rounds, int mode, const dsgdo_hyper* hp,
                               int grad_kind, std::uint32_t shards) {
  if (shards <= 1 || d < shards) return ref_time_rounds(protocol, p, d, rounds, mode, hp, grad_kind);
  using clk = std::chrono::steady_clock;
  auto size_of = [&](std::uint32_t i) { return d / shards + (i + 1 == shards ? d % shards : 0); };
  std::vector<double> secs(shards, 0.0);
  if (mode == 0) {
    std::barrier<> sync((std::ptrdiff_t)shards);
    std::vector<std::thread> th;
    for (std::uint32_t i = 0; i < shards; ++i)
      th.emplace_back([&, i] {
        secs[i] = time_rounds_impl(protocol, p, size_of(i), rounds, 0, hp, grad_kind, &sync);
      });
    for (auto& t : th) t.join();
    double m = 0.0;
    for (double v : secs) {
      if (v < 0) return -1.0;
      m = std::max(m, v);
    }
    return m;
  }
  // the threaded transport is timed unsharded (ref_time_rounds): concurrent
  // whole run_transport calls cannot keep node construction out of the clock
  g_err = "sharded timing supports the simulator rules (mode 0) only";
  return -1.0;
}

}  // extern "C"
