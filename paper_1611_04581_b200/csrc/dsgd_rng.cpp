// dsgd_rng.cpp -- host-side deterministic streams and schedule (C ABI).
//
// The peer schedule must be bit-exact with the reference, so it is drawn on
// the host exactly as rng.hpp:50-95 / rng.cpp:24-112 specify:
// std::mt19937_64 (its sequence is fixed by the C++ standard) keyed by
// splitmix64(FNV-1a(seed || run_id || 0 || purpose || 0 || node)), and the
// explicit samplers uniform01 (53-bit centred), Box-Muller normal,
// exponential and rejection-sampled uniform_index (n == 1 draws nothing).
#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "dsgd_b200.h"
#include "dsgd_internal.h"

struct dsgd_stream {
  std::mt19937_64 engine;
};

namespace {

const char* purpose_name(dsgd_purpose p) {
  switch (p) {
    case DSGD_PURPOSE_NOISE: return "gradient-noise";
    case DSGD_PURPOSE_SAMPLE: return "sample";
    case DSGD_PURPOSE_PARTNER: return "partner-choice";
    case DSGD_PURPOSE_CLOCK: return "clock";
    case DSGD_PURPOSE_STRAGGLER: return "straggler";
    case DSGD_PURPOSE_INIT: return "init";
  }
  return "unknown";
}

inline uint64_t fnv(uint64_t h, uint8_t b) { return (h ^ b) * 1099511628211ull; }

}  // namespace

extern "C" {

uint64_t dsgd_derive_stream_seed(uint64_t root_seed, const char* run_id, uint32_t node_id,
                                 dsgd_purpose purpose) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < 8; ++i) h = fnv(h, uint8_t(root_seed >> (8 * i)));
  for (const char* c = run_id ? run_id : ""; *c; ++c) h = fnv(h, uint8_t(*c));
  h = fnv(h, 0);
  for (const char* c = purpose_name(purpose); *c; ++c) h = fnv(h, uint8_t(*c));
  h = fnv(h, 0);
  for (int i = 0; i < 8; ++i) h = fnv(h, uint8_t(uint64_t(node_id) >> (8 * i)));
  uint64_t z = h + 0x9e3779b97f4a7c15ull;  // splitmix64 finalizer
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

dsgd_status dsgd_stream_create(uint64_t engine_seed, dsgd_stream** out) {
  if (!out) return dsgd::set_error(DSGD_EINVAL, "null output");
  *out = new dsgd_stream{std::mt19937_64(engine_seed)};
  return DSGD_OK;
}

dsgd_status dsgd_stream_make(uint64_t root_seed, const char* run_id, uint32_t node_id,
                             dsgd_purpose purpose, dsgd_stream** out) {
  return dsgd_stream_create(dsgd_derive_stream_seed(root_seed, run_id, node_id, purpose), out);
}

dsgd_status dsgd_stream_clone(const dsgd_stream* s, dsgd_stream** out) {
  if (!s || !out) return dsgd::set_error(DSGD_EINVAL, "null stream");
  *out = new dsgd_stream{s->engine};
  return DSGD_OK;
}

void dsgd_stream_destroy(dsgd_stream* s) { delete s; }

uint64_t dsgd_stream_next_u64(dsgd_stream* s) { return s->engine(); }

double dsgd_stream_uniform01(dsgd_stream* s) {
  const uint64_t bits = s->engine() >> 11;
  return (static_cast<double>(bits) + 0.5) * 0x1.0p-53;
}

double dsgd_stream_normal(dsgd_stream* s) {
  static constexpr double kPi = 3.141592653589793238462643383279502884;
  const double u1 = dsgd_stream_uniform01(s);
  const double u2 = dsgd_stream_uniform01(s);
  const double r = std::sqrt(-2.0 * std::log(u1));
  return r * std::cos(2.0 * kPi * u2);
}

dsgd_status dsgd_stream_uniform_index(dsgd_stream* s, uint32_t n, uint32_t* out) {
  if (n == 0) return dsgd::set_error(DSGD_EINVAL, "uniform_index over empty range");
  if (n == 1) {
    *out = 0;
    return DSGD_OK;
  }
  const uint64_t span = n;
  const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % span);
  uint64_t x = s->engine();
  while (x >= limit) x = s->engine();
  *out = static_cast<uint32_t>(x % span);
  return DSGD_OK;
}

dsgd_status dsgd_stream_exponential(dsgd_stream* s, double rate, double* out) {
  if (!(rate > 0.0)) return dsgd::set_error(DSGD_EINVAL, "exponential rate must be positive");
  *out = -std::log(dsgd_stream_uniform01(s)) / rate;
  return DSGD_OK;
}

void dsgd_stream_fill_normal(dsgd_stream* s, double sigma, double* out, uint64_t n) {
  for (uint64_t k = 0; k < n; ++k) out[k] = sigma * dsgd_stream_normal(s);
}

double dsgd_step_size_at(const dsgd_hyperparams* h, uint64_t t) {
  double alpha = h->alpha0;
  for (uint32_t i = 0; i < h->n_anneal; ++i) {
    if (h->anneal_at[i] <= t)
      alpha *= h->anneal_factor;
    else
      break;
  }
  return alpha;
}

dsgd_status dsgd_hyperparams_validate(const dsgd_hyperparams* h) {
  if (!h) return dsgd::set_error(DSGD_EINVAL, "null hyperparams");
  if (!(h->alpha0 > 0.0)) return dsgd::set_error(DSGD_EINVAL, "alpha0 must be positive");
  if (!(h->anneal_factor > 0.0 && h->anneal_factor <= 1.0))
    return dsgd::set_error(DSGD_EINVAL, "anneal_factor must be in (0, 1]");
  for (uint32_t i = 1; i < h->n_anneal; ++i)
    if (h->anneal_at[i] < h->anneal_at[i - 1])
      return dsgd::set_error(DSGD_EINVAL, "anneal_at must be sorted ascending");
  if (!(h->mu >= 0.0 && h->mu < 1.0)) return dsgd::set_error(DSGD_EINVAL, "mu must be in [0, 1)");
  if (!(h->weight_decay >= 0.0)) return dsgd::set_error(DSGD_EINVAL, "weight_decay must be >= 0");
  if (!(h->beta_gossip > 0.0 && h->beta_gossip < 1.0))
    return dsgd::set_error(DSGD_EINVAL, "beta_gossip must be in (0, 1)");
  if (!(h->beta_ea > 0.0 && h->beta_ea < 1.0))
    return dsgd::set_error(DSGD_EINVAL, "beta_ea must be in (0, 1)");
  if (h->tau < 1) return dsgd::set_error(DSGD_EINVAL, "tau must be >= 1");
  if (h->batch < 1) return dsgd::set_error(DSGD_EINVAL, "batch must be >= 1");
  return DSGD_OK;
}

dsgd_status dsgd_draw_pull_partners(dsgd_stream* const* partner_streams, uint32_t p,
                                    uint32_t* out) {
  if (!partner_streams || !out || p == 0) return dsgd::set_error(DSGD_EINVAL, "bad arguments");
  for (uint32_t i = 0; i < p; ++i) {
    const dsgd_status st = dsgd_stream_uniform_index(partner_streams[i], p, &out[i]);
    if (st != DSGD_OK) return st;
  }
  return DSGD_OK;
}

dsgd_status dsgd_draw_push_targets(dsgd_stream* const* partner_streams, uint32_t p,
                                   uint32_t* out) {
  if (!partner_streams || !out || p < 2)
    return dsgd::set_error(DSGD_EINVAL, "push targets need p >= 2");
  for (uint32_t i = 0; i < p; ++i) {
    uint32_t j = 0;
    const dsgd_status st = dsgd_stream_uniform_index(partner_streams[i], p - 1, &j);
    if (st != DSGD_OK) return st;
    if (j >= i) ++j;
    out[i] = j;
  }
  return DSGD_OK;
}

}  // extern "C"
