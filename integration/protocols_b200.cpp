// protocols_b200.cpp -- the reference's update-rule interface
// (/root/reference/proj/include/dsgd/protocols.hpp:45-152) with the SAME
// C++ signatures, implemented over the B200 C ABI (include/dsgd_b200.h).
//
// A reference build links this file INSTEAD of src/protocols.cpp; its own
// simulator.cpp (run_sync / run_async), transport.cpp (run_transport) and
// every other caller stay unmodified and now run each rule on the GPU
// (integration/Makefile builds exactly that: the unmodified reference
// sources + this file -> libdsgd_reference_b200.so).
//
// Value semantics are kept: each call uploads the nodes it is given (fp64,
// bit-exact mode), runs the fused rule kernel and writes the new state back
// into the returned NodeState values.  The gradient plugin:
//  * an exact QuadraticObjective (objectives.cpp:71-78) is evaluated inside
//    the fused kernel from its device-resident spectrum / optimum;
//  * any other Objective (LogisticObjective, a user's model ...) is called on
//    the host as the reference calls it -- stochastic_gradient(eval_point,
//    h.batch, node.rng.sample) at the rule's evaluation point, which the host
//    forms with the reference's own operation order -- and the result enters
//    the kernel as its gradient buffer (weight decay, noise, momentum, mix
//    and apply stay on the device).
// NoiseModel draws come from each node's noise stream on the host (so the
// streams the caller gets back are advanced exactly as the reference's).
// Errors keep the reference's types and messages (std::invalid_argument).
// Thread-compatible like the reference: device contexts are
// cached per thread, so run_transport's p worker threads each drive their own.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <typeinfo>
#include <utility>
#include <vector>

#include "dsgd/core.hpp"
#include "dsgd/objectives.hpp"
#include "dsgd/protocols.hpp"
#include "dsgd_b200.h"

namespace dsgd {

namespace {

void check(dsgd_status s) {
  if (s == DSGD_OK) return;
  const std::string msg = dsgd_last_error();
  if (s == DSGD_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("dsgd_b200: " + msg);
}

// ------------------------------------------------------- device contexts
struct DevCtx {
  dsgd_ctx* c = nullptr;
  uint32_t p = 0;
  uint64_t d = 0;
  std::vector<double> spec, opt;  // the quadratic objective last uploaded
  bool quad_set = false;
  ~DevCtx() {
    if (c) dsgd_ctx_destroy(c);
  }
};

// A few contexts per thread, most recently used first.
thread_local std::list<std::unique_ptr<DevCtx>> t_ctx;

DevCtx& ctx_for(uint32_t p, uint64_t d) {
  for (auto it = t_ctx.begin(); it != t_ctx.end(); ++it)
    if ((*it)->p == p && (*it)->d == d) {
      t_ctx.splice(t_ctx.begin(), t_ctx, it);
      return *t_ctx.front();
    }
  auto x = std::make_unique<DevCtx>();
  const char* dev = std::getenv("DSGD_B200_DEVICE");
  dsgd_ctx_desc desc{dev ? std::atoi(dev) : 0, d, DSGD_F64, p, 0, p,
                     DSGD_CTX_QUADRATIC | DSGD_CTX_GRAD | DSGD_CTX_NOISE | DSGD_CTX_CENTER,
                     nullptr};
  check(dsgd_ctx_create(&desc, &x->c));
  x->p = p;
  x->d = d;
  t_ctx.push_front(std::move(x));
  if (t_ctx.size() > 4) t_ctx.pop_back();
  return *t_ctx.front();
}

const QuadraticObjective* as_quadratic(const Objective* o) {
  // exactly the reference's QuadraticObjective (a subclass may override
  // stochastic_gradient: it then takes the host-plugin path)
  if (o && typeid(*o) == typeid(QuadraticObjective)) return static_cast<const QuadraticObjective*>(o);
  return nullptr;
}

bool same_quadratic(std::span<const Objective* const> objs) {
  const QuadraticObjective* q0 = as_quadratic(objs[0]);
  if (!q0) return false;
  for (const Objective* o : objs) {
    if (o == objs[0]) continue;
    const QuadraticObjective* q = as_quadratic(o);
    if (!q || q->spectrum() != q0->spectrum() || q->optimum()->values() != q0->optimum()->values())
      return false;
  }
  return true;
}

// The gradient source of one call.  eval(i) returns node i's evaluation
// point (only called for host-plugin objectives, in node order).
template <typename Eval>
dsgd_grad_spec prepare(DevCtx& x, std::span<NodeState> nodes, std::span<const Objective* const> objs,
                       const NoiseModel& noise, const Hyperparams& h, double* grad_norm_out,
                       Eval&& eval) {
  dsgd_grad_spec g{};
  const uint64_t d = x.d;
  if (same_quadratic(objs)) {
    const QuadraticObjective* q = as_quadratic(objs[0]);
    if (q->dim() != d) throw std::invalid_argument("ParamVec dimension mismatch");
    const std::vector<double>& s = q->spectrum();
    // optimum() returns the optional by value: keep it alive while `o` is used
    const std::optional<ParamVec> opt = q->optimum();
    const std::vector<double>& o = opt->values();
    if (!x.quad_set || x.spec != s || x.opt != o) {
      check(dsgd_set_vector(x.c, 0, DSGD_BUF_SPECTRUM, s.data()));
      check(dsgd_set_vector(x.c, 0, DSGD_BUF_OPT, o.data()));
      x.spec = s;
      x.opt = o;
      x.quad_set = true;
    }
    g.source = DSGD_GRAD_QUADRATIC;
  } else {
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const ParamVec point = eval(i);
      const ParamVec gi = objs[i]->stochastic_gradient(point, h.batch, nodes[i].rng.sample);
      if (gi.dim() != d) throw std::invalid_argument("ParamVec dimension mismatch");
      check(dsgd_set_vector(x.c, static_cast<uint32_t>(i), DSGD_BUF_GRAD, gi.raw()));
    }
    g.source = DSGD_GRAD_BUFFER;
  }
  if (noise.kind == NoiseModel::Kind::kGaussian) {
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const ParamVec xi = noise.sample(nodes[i].rng.noise);  // objectives.cpp:175-183
      check(dsgd_set_vector(x.c, static_cast<uint32_t>(i), DSGD_BUF_NOISE, xi.raw()));
    }
    g.use_noise = 1;
  }
  g.grad_norm_out = grad_norm_out;  // raised when get_state reads the device max
  return g;
}

dsgd_hyperparams to_c(const Hyperparams& h) {
  return dsgd_hyperparams{h.alpha0, h.anneal_factor, h.anneal_at.data(),
                          static_cast<uint32_t>(h.anneal_at.size()), h.mu, h.weight_decay,
                          h.beta_gossip, h.beta_ea, h.tau, h.batch};
}

void put(DevCtx& x, uint32_t i, const NodeState& n) {
  if (n.theta.dim() != x.d || n.delta_prev.dim() != x.d)
    throw std::invalid_argument("ParamVec dimension mismatch");
  check(dsgd_set_state(x.c, i, n.theta.raw(), n.delta_prev.raw(), n.t));
}

void get(DevCtx& x, uint32_t i, NodeState& n, bool delta = true) {
  uint64_t t = 0;
  std::vector<double> dp;
  if (!delta) dp.resize(x.d);
  check(dsgd_get_state(x.c, i, n.theta.raw(), delta ? n.delta_prev.raw() : dp.data(), &t));
  n.t = t;
}

uint64_t common_dim(const std::vector<NodeState>& nodes) {
  const uint64_t d = nodes[0].theta.dim();
  for (const NodeState& n : nodes)
    if (n.theta.dim() != d) throw std::invalid_argument("mixing dimension mismatch");
  return d;
}

// Lookahead point of compute_local_delta (protocols.cpp:90-96), the
// reference's own operations.
ParamVec lookahead(const ParamVec& theta, const NodeState& n, const Hyperparams& h) {
  if (h.mu == 0.0) return theta;
  ParamVec la = theta;
  la.axpy(h.mu, n.delta_prev);
  return la;
}

ParamVec mix_point(const ParamVec& own, const ParamVec& other, double beta) {
  ParamVec out = own;  // mix_toward protocols.cpp:42-51 (centred form)
  for (std::size_t k = 0; k < out.dim(); ++k) out[k] += beta * (other[k] - own[k]);
  return out;
}

void check_common_round(const std::vector<NodeState>& nodes) {
  for (const NodeState& n : nodes)
    if (n.t != nodes[0].t)
      throw std::invalid_argument("synchronous round requires equal node clocks");
}

void check_partners(std::size_t p, std::span<const std::uint32_t> m) {
  if (m.size() != p) throw std::invalid_argument("partner map size must equal node count");
  for (std::uint32_t j : m)
    if (j >= p) throw std::invalid_argument("partner index out of range");
}

void check_objectives(std::size_t p, std::span<const Objective* const> objs) {
  if (objs.size() != p) throw std::invalid_argument("objective list size must equal node count");
  for (const Objective* o : objs)
    if (o == nullptr) throw std::invalid_argument("null objective");
}

std::vector<const Objective*> replicate(const Objective& obj, std::size_t p) {
  return std::vector<const Objective*>(p, &obj);
}

// Slot 1 of a two-node context holds an explicit vector (a partner's theta)
// for the single-node rules; it is never stepped.
NodeState carrier(const NodeState& n, const ParamVec& theta) {
  NodeState c;
  c.theta = theta;
  c.delta_prev = ParamVec::zeros(theta.dim());
  c.t = n.t;
  return c;
}

}  // namespace

// ------------------------------------------------------------ local step
ParamVec compute_local_delta(NodeState& node, const Objective& obj, const NoiseModel& noise,
                             const Hyperparams& h, double* grad_norm_out) {
  DevCtx& x = ctx_for(1, node.theta.dim());
  put(x, 0, node);
  const Objective* objs[1] = {&obj};
  std::span<NodeState> one(&node, 1);
  const dsgd_grad_spec g = prepare(x, one, objs, noise, h, grad_norm_out,
                                   [&](std::size_t) { return lookahead(node.theta, node, h); });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_local_sgd_step(x.c, &hc, &g));
  ParamVec delta(node.theta.dim());
  check(dsgd_get_state(x.c, 0, nullptr, delta.raw(), nullptr));  // theta, t untouched
  return delta;
}

NodeState local_sgd_step(NodeState node, const Objective& obj, const NoiseModel& noise,
                         const Hyperparams& h, double* grad_norm_out) {
  DevCtx& x = ctx_for(1, node.theta.dim());
  put(x, 0, node);
  const Objective* objs[1] = {&obj};
  std::span<NodeState> one(&node, 1);
  const dsgd_grad_spec g = prepare(x, one, objs, noise, h, grad_norm_out,
                                   [&](std::size_t) { return lookahead(node.theta, node, h); });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_local_sgd_step(x.c, &hc, &g));
  get(x, 0, node);
  return node;
}

// ------------------------------------------------------------- all-reduce
std::vector<NodeState> allreduce_round(std::vector<NodeState> nodes,
                                       std::span<const Objective* const> objs,
                                       const NoiseModel& noise, const Hyperparams& h,
                                       MomentumScope scope, double* grad_norm_out) {
  if (nodes.empty()) throw std::invalid_argument("allreduce_round on empty node set");
  check_common_round(nodes);
  check_objectives(nodes.size(), objs);
  const uint64_t d = common_dim(nodes);
  const uint32_t p = static_cast<uint32_t>(nodes.size());
  DevCtx& x = ctx_for(p, d);
  for (uint32_t i = 0; i < p; ++i) put(x, i, nodes[i]);
  const dsgd_grad_spec g =
      prepare(x, nodes, objs, noise, h, grad_norm_out,
              [&](std::size_t i) { return lookahead(nodes[i].theta, nodes[i], h); });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_allreduce_round(x.c, &hc, &g,
                             scope == MomentumScope::kAggregate ? DSGD_SCOPE_AGGREGATE
                                                                : DSGD_SCOPE_PER_NODE));
  for (uint32_t i = 0; i < p; ++i) get(x, i, nodes[i]);
  return nodes;
}

std::vector<NodeState> allreduce_round(std::vector<NodeState> nodes, const Objective& obj,
                                       const NoiseModel& noise, const Hyperparams& h,
                                       MomentumScope scope, double* grad_norm_out) {
  const auto objs = replicate(obj, nodes.size());
  return allreduce_round(std::move(nodes), objs, noise, h, scope, grad_norm_out);
}

// ------------------------------------------------------------------ EASGD
std::pair<NodeState, ParamVec> ea_client_step(NodeState node, const ParamVec& center,
                                              const Objective& obj, const NoiseModel& noise,
                                              const Hyperparams& h, double* grad_norm_out) {
  if (center.dim() != node.theta.dim())
    throw std::invalid_argument("ea_client_step center dimension mismatch");
  const uint64_t d = node.theta.dim();
  DevCtx& x = ctx_for(2, d);
  put(x, 0, node);
  check(dsgd_set_vector(x.c, 0, DSGD_BUF_CENTER, center.raw()));
  const Objective* objs[1] = {&obj};
  std::span<NodeState> one(&node, 1);
  const dsgd_grad_spec g = prepare(x, one, objs, noise, h, grad_norm_out, [&](std::size_t) {
    ParamVec moved = node.theta;  // theta -= beta_ea * (theta - c)  (protocols.cpp:146-150)
    for (std::size_t k = 0; k < d; ++k) moved[k] -= h.beta_ea * (node.theta[k] - center[k]);
    return lookahead(moved, node, h);
  });
  // one client tick on slot 0 (dsgd_ea_client_event: the client update,
  // the step, in place); the update u -- ea_client_step's second result --
  // is written into slot 1's parameter buffer, the center copy is discarded
  void* sink = nullptr;
  check(dsgd_buffer_ptr(x.c, 1, DSGD_BUF_THETA, &sink));
  void* outs[2] = {sink, nullptr};
  check(dsgd_ea_set_update_out(x.c, outs));
  const dsgd_hyperparams hc = to_c(h);
  const dsgd_status st = dsgd_ea_client_event(x.c, &hc, &g, 0, 1);
  dsgd_ea_set_update_out(x.c, nullptr);
  check(st);
  get(x, 0, node);
  ParamVec update(d);
  check(dsgd_get_vector(x.c, 1, DSGD_BUF_THETA, update.raw()));
  return {std::move(node), std::move(update)};
}

ServerState ea_server_apply(ServerState server, const ParamVec& update) {
  if (update.dim() != server.theta_center.dim())
    throw std::invalid_argument("ParamVec dimension mismatch");
  const uint64_t d = update.dim();
  DevCtx& x = ctx_for(1, d);
  check(dsgd_set_vector(x.c, 0, DSGD_BUF_CENTER, server.theta_center.raw()));
  check(dsgd_set_vector(x.c, 0, DSGD_BUF_GRAD, update.raw()));
  void* u = nullptr;
  check(dsgd_buffer_ptr(x.c, 0, DSGD_BUF_GRAD, &u));
  check(dsgd_ea_server_apply(x.c, u));  // center += update (protocols.cpp:156)
  check(dsgd_get_vector(x.c, 0, DSGD_BUF_CENTER, server.theta_center.raw()));
  server.applied_updates += 1;
  return server;
}

// ------------------------------------------------------------ pull gossip
std::vector<NodeState> pull_mix(std::vector<NodeState> nodes,
                                std::span<const std::uint32_t> partner_of) {
  check_partners(nodes.size(), partner_of);
  if (nodes.empty()) return nodes;
  const uint64_t d = common_dim(nodes);
  const uint32_t p = static_cast<uint32_t>(nodes.size());
  DevCtx& x = ctx_for(p, d);
  for (uint32_t i = 0; i < p; ++i) put(x, i, nodes[i]);
  check(dsgd_pull_mix(x.c, partner_of.data()));
  for (uint32_t i = 0; i < p; ++i) get(x, i, nodes[i]);
  return nodes;
}

std::vector<NodeState> pull_gossip_round(std::vector<NodeState> nodes,
                                         std::span<const std::uint32_t> partner_of,
                                         std::span<const Objective* const> objs,
                                         const NoiseModel& noise, const Hyperparams& h,
                                         double* grad_norm_out) {
  check_common_round(nodes);
  check_objectives(nodes.size(), objs);
  check_partners(nodes.size(), partner_of);
  if (nodes.empty()) return nodes;
  const uint64_t d = common_dim(nodes);
  const uint32_t p = static_cast<uint32_t>(nodes.size());
  DevCtx& x = ctx_for(p, d);
  for (uint32_t i = 0; i < p; ++i) put(x, i, nodes[i]);
  const dsgd_grad_spec g = prepare(x, nodes, objs, noise, h, grad_norm_out, [&](std::size_t i) {
    // the gradient is taken at the mixed theta (protocols.cpp:180-183)
    return lookahead(mix_point(nodes[i].theta, nodes[partner_of[i]].theta, 0.5), nodes[i], h);
  });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_pull_gossip_round(x.c, &hc, &g, partner_of.data()));
  for (uint32_t i = 0; i < p; ++i) get(x, i, nodes[i]);
  return nodes;
}

std::vector<NodeState> pull_gossip_round(std::vector<NodeState> nodes,
                                         std::span<const std::uint32_t> partner_of,
                                         const Objective& obj, const NoiseModel& noise,
                                         const Hyperparams& h, double* grad_norm_out) {
  const auto objs = replicate(obj, nodes.size());
  return pull_gossip_round(std::move(nodes), partner_of, objs, noise, h, grad_norm_out);
}

// ------------------------------------------------------------ push gossip
namespace {
void check_targets(std::size_t p, std::span<const std::uint32_t> target_of) {
  check_partners(p, target_of);
  for (std::size_t k = 0; k < p; ++k)
    if (target_of[k] == k) throw std::invalid_argument("push target must differ from sender");
}

ParamVec push_point(const std::vector<NodeState>& nodes, std::span<const std::uint32_t> target_of,
                    std::size_t i) {
  // push_mix protocols.cpp:207-225: centred average of the received set
  ParamVec acc = ParamVec::zeros(nodes[i].theta.dim());
  std::size_t count = 1;
  for (std::size_t k = 0; k < nodes.size(); ++k)
    if (target_of[k] == i) {
      for (std::size_t c = 0; c < acc.dim(); ++c) acc[c] += nodes[k].theta[c] - nodes[i].theta[c];
      ++count;
    }
  ParamVec mixed = nodes[i].theta;
  const double inv = 1.0 / static_cast<double>(count);
  for (std::size_t c = 0; c < mixed.dim(); ++c) mixed[c] += acc[c] * inv;
  return mixed;
}
}  // namespace

std::vector<NodeState> push_mix(std::vector<NodeState> nodes,
                                std::span<const std::uint32_t> target_of) {
  check_targets(nodes.size(), target_of);
  if (nodes.empty()) return nodes;
  const uint64_t d = common_dim(nodes);
  const uint32_t p = static_cast<uint32_t>(nodes.size());
  DevCtx& x = ctx_for(p, d);
  for (uint32_t i = 0; i < p; ++i) put(x, i, nodes[i]);
  check(dsgd_push_mix(x.c, target_of.data()));
  for (uint32_t i = 0; i < p; ++i) get(x, i, nodes[i]);
  return nodes;
}

std::vector<NodeState> push_gossip_round(std::vector<NodeState> nodes,
                                         std::span<const std::uint32_t> target_of,
                                         std::span<const Objective* const> objs,
                                         const NoiseModel& noise, const Hyperparams& h,
                                         double* grad_norm_out) {
  check_common_round(nodes);
  check_objectives(nodes.size(), objs);
  check_targets(nodes.size(), target_of);
  if (nodes.empty()) return nodes;
  const uint64_t d = common_dim(nodes);
  const uint32_t p = static_cast<uint32_t>(nodes.size());
  DevCtx& x = ctx_for(p, d);
  for (uint32_t i = 0; i < p; ++i) put(x, i, nodes[i]);
  const dsgd_grad_spec g = prepare(x, nodes, objs, noise, h, grad_norm_out, [&](std::size_t i) {
    return lookahead(push_point(nodes, target_of, i), nodes[i], h);
  });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_push_gossip_round(x.c, &hc, &g, target_of.data()));
  for (uint32_t i = 0; i < p; ++i) get(x, i, nodes[i]);
  return nodes;
}

std::vector<NodeState> push_gossip_round(std::vector<NodeState> nodes,
                                         std::span<const std::uint32_t> target_of,
                                         const Objective& obj, const NoiseModel& noise,
                                         const Hyperparams& h, double* grad_norm_out) {
  const auto objs = replicate(obj, nodes.size());
  return push_gossip_round(std::move(nodes), target_of, objs, noise, h, grad_norm_out);
}

// ---------------------------------------------------- stale / fresh gossip
NodeState gossip_stale_step(NodeState node, const ParamVec& partner_theta, const Objective& obj,
                            const NoiseModel& noise, const Hyperparams& h,
                            double* grad_norm_out) {
  if (partner_theta.dim() != node.theta.dim())
    throw std::invalid_argument("mixing dimension mismatch");
  const uint64_t d = node.theta.dim();
  DevCtx& x = ctx_for(2, d);
  put(x, 0, node);
  put(x, 1, carrier(node, partner_theta));  // slot 1 only holds the partner vector
  void* partner = nullptr;
  check(dsgd_buffer_ptr(x.c, 1, DSGD_BUF_THETA, &partner));
  const Objective* objs[1] = {&obj};
  std::span<NodeState> one(&node, 1);
  // the delta uses the pre-mix theta (protocols.cpp:255-258)
  const dsgd_grad_spec g = prepare(x, one, objs, noise, h, grad_norm_out,
                                   [&](std::size_t) { return lookahead(node.theta, node, h); });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_gossip_stale_step(x.c, &hc, &g, 0, partner));
  get(x, 0, node);
  return node;
}

NodeState gossip_fresh_mix(NodeState stepped, const ParamVec& partner_theta_fresh, double beta) {
  if (partner_theta_fresh.dim() != stepped.theta.dim())
    throw std::invalid_argument("mixing dimension mismatch");
  DevCtx& x = ctx_for(2, stepped.theta.dim());
  put(x, 0, stepped);
  put(x, 1, carrier(stepped, partner_theta_fresh));
  void* partner = nullptr;
  check(dsgd_buffer_ptr(x.c, 1, DSGD_BUF_THETA, &partner));
  check(dsgd_mix_toward(x.c, 0, partner, beta));
  get(x, 0, stepped);
  return stepped;
}

NodeState gossip_fresh_step(NodeState node, const ParamVec& partner_theta_fresh,
                            const Objective& obj, const NoiseModel& noise, const Hyperparams& h,
                            double* grad_norm_out) {
  node = local_sgd_step(std::move(node), obj, noise, h, grad_norm_out);
  return gossip_fresh_mix(std::move(node), partner_theta_fresh, h.beta_gossip);
}

// -------------------------------------------------------------- async pull
std::vector<NodeState> async_pull_event(std::vector<NodeState> nodes, std::uint32_t i,
                                        std::uint32_t j, const Objective& obj,
                                        const NoiseModel& noise, const Hyperparams& h,
                                        double* grad_norm_out) {
  if (i >= nodes.size() || j >= nodes.size())
    throw std::invalid_argument("async_pull_event node index out of range");
  const uint64_t d = common_dim(nodes);
  DevCtx& x = ctx_for(2, d);
  // node i in slot 0, node j's current theta in slot 1 (j == i: the own
  // pre-step theta, protocols.cpp:290)
  put(x, 0, nodes[i]);
  put(x, 1, carrier(nodes[i], nodes[j].theta));
  const Objective* objs[1] = {&obj};
  std::span<NodeState> one(&nodes[i], 1);
  // model_gradient at theta_i itself: no lookahead (protocols.cpp:287)
  const dsgd_grad_spec g =
      prepare(x, one, objs, noise, h, grad_norm_out, [&](std::size_t) { return nodes[i].theta; });
  const dsgd_hyperparams hc = to_c(h);
  check(dsgd_async_pull_event(x.c, &hc, &g, 0, 1));
  get(x, 0, nodes[i]);
  return nodes;
}

}  // namespace dsgd
