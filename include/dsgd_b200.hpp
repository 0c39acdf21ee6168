// dsgd_b200.hpp -- header-only C++ host wrapper over the C ABI in
// dsgd_b200.h, for callers of the reference's update-rule interface
// (/root/reference/proj/include/dsgd/protocols.hpp:45-152).
//
// Error conventions follow the reference: invalid arguments throw
// std::invalid_argument (protocols.cpp:43-77), a peer that never arrives
// throws dsgd_b200::TransportError (transport.hpp:57-60), CUDA/NCCL failures
// throw std::runtime_error.  State lives on the GPU; a Context is one
// process's view of one GPU hosting all p nodes or exactly one of them.
#ifndef DSGD_B200_HPP_
#define DSGD_B200_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dsgd_b200.h"

namespace dsgd_b200 {

class TransportError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(dsgd_status s) {
  if (s == DSGD_OK) return;
  const std::string msg = dsgd_last_error();
  if (s == DSGD_EINVAL) throw std::invalid_argument(msg);
  if (s == DSGD_ETIMEOUT) throw TransportError(msg);
  throw std::runtime_error("dsgd_b200: " + msg);
}

// dsgd::Hyperparams (core.hpp:54-70) with its defaults.
struct Hyperparams {
  double alpha0 = 0.1;
  double anneal_factor = 0.1;
  std::vector<std::uint64_t> anneal_at = {150000, 300000};
  double mu = 0.9;
  double weight_decay = 1e-4;
  double beta_gossip = 0.5;
  double beta_ea = 0.1;
  std::uint32_t tau = 1;
  std::uint32_t batch = 1;

  dsgd_hyperparams c() const {
    return dsgd_hyperparams{alpha0,      anneal_factor, anneal_at.data(), (uint32_t)anneal_at.size(),
                            mu,          weight_decay,  beta_gossip,      beta_ea,
                            tau,         batch};
  }
  void validate() const {
    const dsgd_hyperparams h = c();
    check(dsgd_hyperparams_validate(&h));
  }
};

inline double step_size_at(const Hyperparams& h, std::uint64_t t) {
  const dsgd_hyperparams c = h.c();
  return dsgd_step_size_at(&c, t);
}

// RAII RngStream (rng.hpp:50-85).
class Stream {
 public:
  Stream(std::uint64_t root_seed, const std::string& run_id, std::uint32_t node,
         dsgd_purpose purpose) {
    check(dsgd_stream_make(root_seed, run_id.c_str(), node, purpose, &s_));
  }
  explicit Stream(std::uint64_t engine_seed) { check(dsgd_stream_create(engine_seed, &s_)); }
  Stream(const Stream& o) { check(dsgd_stream_clone(o.s_, &s_)); }
  Stream(Stream&& o) noexcept : s_(std::exchange(o.s_, nullptr)) {}
  Stream& operator=(Stream o) {
    std::swap(s_, o.s_);
    return *this;
  }
  ~Stream() { dsgd_stream_destroy(s_); }
  std::uint64_t next_u64() { return dsgd_stream_next_u64(s_); }
  double normal() { return dsgd_stream_normal(s_); }
  std::uint32_t uniform_index(std::uint32_t n) {
    std::uint32_t out = 0;
    check(dsgd_stream_uniform_index(s_, n, &out));
    return out;
  }
  dsgd_stream* get() const { return s_; }

 private:
  dsgd_stream* s_ = nullptr;
};

// Gradient source of one call: the device quadratic objective, or per-node
// device gradient buffers (the Objective plugin evaluated by the caller).
struct Gradient {
  dsgd_grad_source source = DSGD_GRAD_QUADRATIC;
  std::vector<const void*> buffers;  // empty: the context's own DSGD_BUF_GRAD
  bool noise = false;                // add DSGD_BUF_NOISE
  double* grad_norm_out = nullptr;
  double device_noise_sigma = 0.0;   // > 0: N(0, sigma^2) drawn inside the kernel
  std::uint64_t device_noise_seed = 0;
  std::vector<std::uint64_t> rows;   // DSGD_GRAD_LOGISTIC: n_local * batch rows (empty: streams)

  dsgd_grad_spec c() const {
    const uint32_t mode = noise ? 1u : (device_noise_sigma > 0.0 ? 2u : 0u);
    return dsgd_grad_spec{source,        buffers.empty() ? nullptr : buffers.data(),
                          mode,          grad_norm_out,
                          device_noise_sigma, device_noise_seed,
                          rows.empty() ? nullptr : rows.data()};
  }
};

class Context {
 public:
  Context(std::uint64_t dim, std::uint32_t p, dsgd_dtype dtype = DSGD_F32, int device = 0,
          std::uint32_t flags = 0, std::uint32_t first_node = 0, std::uint32_t n_local = 0,
          void* stream = nullptr) {
    dsgd_ctx_desc d{device, dim, dtype, p, first_node, n_local ? n_local : p, flags, stream};
    check(dsgd_ctx_create(&d, &ctx_));
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ~Context() { dsgd_ctx_destroy(ctx_); }
  dsgd_ctx* get() const { return ctx_; }

  void set_state(std::uint32_t local, const std::vector<double>& theta,
                 const std::vector<double>& delta_prev, std::uint64_t t) {
    check(dsgd_set_state(ctx_, local, theta.data(),
                         delta_prev.empty() ? nullptr : delta_prev.data(), t));
  }
  void get_state(std::uint32_t local, std::vector<double>* theta, std::vector<double>* delta_prev,
                 std::uint64_t* t) {
    check(dsgd_get_state(ctx_, local, theta ? theta->data() : nullptr,
                         delta_prev ? delta_prev->data() : nullptr, t));
  }
  void set_vector(std::uint32_t local, dsgd_buffer which, const std::vector<double>& v) {
    check(dsgd_set_vector(ctx_, local, which, v.data()));
  }
  std::vector<double> get_vector(std::uint32_t local, dsgd_buffer which, std::uint64_t dim) {
    std::vector<double> v(dim);
    check(dsgd_get_vector(ctx_, local, which, v.data()));
    return v;
  }
  // LogisticObjective(features, labels, l2) objectives.cpp:80-106 (features row-major)
  void set_logistic(const std::vector<std::vector<double>>& features,
                    const std::vector<int>& labels, double l2) {
    std::vector<double> flat;
    for (const auto& r : features) {
      if (r.size() != features[0].size())
        throw std::invalid_argument("logistic feature rows have inconsistent width");
      flat.insert(flat.end(), r.begin(), r.end());
    }
    if (features.size() != labels.size())
      throw std::invalid_argument("logistic features/labels size mismatch");
    std::vector<int32_t> y(labels.begin(), labels.end());
    check(dsgd_set_logistic(ctx_, flat.empty() ? nullptr : flat.data(),
                            y.empty() ? nullptr : y.data(), features.size(), l2));
  }
  void set_sample_range(std::uint32_t local, std::uint64_t begin, std::uint64_t end) {
    check(dsgd_logistic_set_sample_range(ctx_, local, begin, end));
  }
  void sync() { check(dsgd_ctx_sync(ctx_)); }

  // protocols.hpp:45-152, lock-step over every node of the group.
  void local_sgd_step(const Hyperparams& h, const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_local_sgd_step(ctx_, &hc, &gc));
  }
  void allreduce_round(const Hyperparams& h, const Gradient& g = {},
                       dsgd_momentum_scope scope = DSGD_SCOPE_AGGREGATE) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_allreduce_round(ctx_, &hc, &gc, scope));
  }
  void ea_round(const Hyperparams& h, bool gated, const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_ea_round(ctx_, &hc, &gc, gated ? 1 : 0));
  }
  void pull_gossip_round(const Hyperparams& h, const std::vector<std::uint32_t>& partner_of,
                         const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_pull_gossip_round(ctx_, &hc, &gc, partner_of.data()));
  }
  void push_gossip_round(const Hyperparams& h, const std::vector<std::uint32_t>& target_of,
                         const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_push_gossip_round(ctx_, &hc, &gc, target_of.data()));
  }
  void gossip_stale_round(const Hyperparams& h, const std::vector<std::uint32_t>& partner_of,
                          const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_gossip_stale_round(ctx_, &hc, &gc, partner_of.data()));
  }
  void gossip_fresh_round(const Hyperparams& h, const std::vector<std::uint32_t>& partner_of,
                          const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_gossip_fresh_round(ctx_, &hc, &gc, partner_of.data()));
  }
  void async_pull_event(const Hyperparams& h, std::uint32_t i, std::uint32_t j,
                        const Gradient& g = {}) {
    const auto hc = h.c();
    const auto gc = g.c();
    check(dsgd_async_pull_event(ctx_, &hc, &gc, i, j));
  }

 private:
  dsgd_ctx* ctx_ = nullptr;
};

}  // namespace dsgd_b200

#endif  // DSGD_B200_HPP_
