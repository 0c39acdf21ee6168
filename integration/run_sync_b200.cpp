// run_sync_b200.cpp -- the reference's synchronous driver (run_sync,
// /root/reference/proj/src/simulator.cpp:214-376) with the node state
// RESIDENT on the GPU for the whole run: one dsgd_run_rounds call replaces
// the per-round loop (gating, step sizes, partner draws from the reference
// partner streams, NoiseModel draws from the noise streams, one fused
// kernel per round), so no state crosses PCIe between rounds.  Compiled
// against the reference headers next to protocols_b200.cpp
// (integration/Makefile) -- the example of INTEGRATION.md section 2.
//
// Scope: the quadratic objective (QuadraticObjective, fused in the kernel),
// every synchronous protocol, both momentum scopes.  Returns the final
// nodes, the EASGD server, max_grad_norm and the first and last trace
// records (make_trace_record, simulator.cpp:92-123); the straggler clock
// (node_time) models time, not arithmetic, and stays zero.
#include "run_sync_b200.hpp"

#include <stdexcept>
#include <string>
#include <vector>

#include "dsgd_b200.h"

namespace dsgd_b200 {

namespace {

void check(dsgd_status s) {
  if (s == DSGD_OK) return;
  const std::string msg = dsgd_last_error();
  if (s == DSGD_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("dsgd_b200: " + msg);
}

struct Ctx {
  dsgd_ctx* c = nullptr;
  ~Ctx() {
    if (c) dsgd_ctx_destroy(c);
  }
};

}  // namespace

dsgd::RunResult run_sync_resident(const dsgd::SimConfig& cfg, const dsgd::QuadraticObjective& obj,
                                  int device) {
  if (cfg.protocol == dsgd::ProtocolKind::kAsyncPull)
    throw std::invalid_argument("async-pull requires the asynchronous driver");
  if (cfg.noise.dim != obj.dim())
    throw std::invalid_argument("noise dimension must match objective dimension");
  if (cfg.rounds == 0) throw std::invalid_argument("rounds must be >= 1");
  std::vector<dsgd::NodeState> nodes = dsgd::make_initial_nodes(cfg, obj);  // unchanged
  const uint64_t d = obj.dim();
  const bool ea = cfg.protocol == dsgd::ProtocolKind::kElasticAvg;
  const bool noisy = cfg.noise.kind == dsgd::NoiseModel::Kind::kGaussian;
  Ctx x;
  const dsgd_ctx_desc desc{device, d, DSGD_F64, cfg.p, 0, cfg.p,
                           DSGD_CTX_QUADRATIC | (noisy ? DSGD_CTX_NOISE : 0u) |
                               (ea ? DSGD_CTX_CENTER : 0u),
                           nullptr};
  check(dsgd_ctx_create(&desc, &x.c));
  check(dsgd_set_vector(x.c, 0, DSGD_BUF_SPECTRUM, obj.spectrum().data()));
  check(dsgd_set_vector(x.c, 0, DSGD_BUF_OPT, obj.optimum()->values().data()));
  for (uint32_t i = 0; i < cfg.p; ++i)
    check(dsgd_set_state(x.c, i, nodes[i].theta.raw(), nodes[i].delta_prev.raw(), nodes[i].t));
  if (ea) check(dsgd_ea_init_center(x.c));  // make_server: spatial_mean (simulator.cpp:62-67)
  check(dsgd_ctx_seed_streams(x.c, cfg.seed, cfg.run_id.c_str()));

  dsgd::RunResult result;
  result.node_time.assign(cfg.p, 0.0);
  std::vector<dsgd::ParamVec> thetas;
  for (const auto& n : nodes) thetas.push_back(n.theta);
  result.trace.push_back(dsgd::make_trace_record(cfg, obj, thetas, 0, 0.0,
                                                 dsgd::step_size_at(cfg.hyper, 0)));

  const dsgd::Hyperparams& hp = cfg.hyper;
  dsgd_run_desc run{};
  run.protocol = static_cast<dsgd_protocol>(cfg.protocol);  // ProtocolKind numbering
  run.hyper = dsgd_hyperparams{hp.alpha0, hp.anneal_factor, hp.anneal_at.data(),
                               static_cast<uint32_t>(hp.anneal_at.size()), hp.mu, hp.weight_decay,
                               hp.beta_gossip, hp.beta_ea, hp.tau, hp.batch};
  run.scope = cfg.momentum_scope == dsgd::MomentumScope::kAggregate ? DSGD_SCOPE_AGGREGATE
                                                                    : DSGD_SCOPE_PER_NODE;
  run.grad = dsgd_grad_spec{DSGD_GRAD_QUADRATIC, nullptr, 0, &result.max_grad_norm, 0.0, 0,
                            nullptr};
  run.host_noise_sigma = noisy ? cfg.noise.sigma : 0.0;
  run.rounds = cfg.rounds;
  check(dsgd_run_rounds(x.c, &run));  // max_grad_norm is read once, here

  thetas.clear();
  for (uint32_t i = 0; i < cfg.p; ++i) {
    check(dsgd_get_state(x.c, i, nodes[i].theta.raw(), nodes[i].delta_prev.raw(), &nodes[i].t));
    thetas.push_back(nodes[i].theta);
  }
  result.trace.push_back(dsgd::make_trace_record(cfg, obj, thetas, cfg.rounds, 0.0,
                                                 dsgd::step_size_at(hp, cfg.rounds)));
  if (ea) {
    dsgd::ServerState server;
    server.theta_center = dsgd::ParamVec(d);
    check(dsgd_get_vector(x.c, 0, DSGD_BUF_CENTER, server.theta_center.raw()));
    uint64_t gated = 0;
    for (uint64_t t = 1; t < cfg.rounds; ++t) gated += (t % hp.tau == 0) ? 1 : 0;
    server.applied_updates = gated * cfg.p;
    result.final_server = std::move(server);
  }
  result.final_nodes = std::move(nodes);
  return result;
}

}  // namespace dsgd_b200
