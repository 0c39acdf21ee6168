/*
 * dsgd_oracle.c -- TEST INFRASTRUCTURE ONLY (see dsgd_oracle.h).
 *
 * Plain-C restatement of the reference's deterministic RNG
 * (include/dsgd/rng.hpp:50-95, src/rng.cpp:24-112), step schedule
 * (src/core.cpp:82-92), partner draws (src/simulator.cpp:69-88) and, through
 * dsgd_oracle_impl.inc, the update rules of src/protocols.cpp and the run
 * drivers of src/simulator.cpp.  Build: oracle/Makefile (-O2
 * -ffp-contract=off, no -march / -ffast-math so rounding matches the
 * reference objects).
 */
#include "dsgd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- std::mt19937_64 (parameters fixed by the C++ standard) ---- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

void dsgdo_rng_seed(dsgdo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (uint32_t i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
  r->idx = MT_N;
}

static void mt_twist(dsgdo_rng* r) {
  for (uint32_t i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t dsgdo_rng_next(dsgdo_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:59-62: top 53 bits, centred in the cell, never 0 or 1 */
double dsgdo_uniform01(dsgdo_rng* r) {
  const uint64_t bits = dsgdo_rng_next(r) >> 11;
  return ((double)bits + 0.5) * 0x1.0p-53;
}

/* rng.hpp:65-70: Box-Muller, two raw draws, libm log/sqrt/cos */
double dsgdo_normal(dsgdo_rng* r) {
  static const double kPi = 3.141592653589793238462643383279502884;
  const double u1 = dsgdo_uniform01(r);
  const double u2 = dsgdo_uniform01(r);
  const double rad = sqrt(-2.0 * log(u1));
  return rad * cos(2.0 * kPi * u2);
}

/* NoiseModel::sample objectives.cpp:175-183: out[k] = sigma * normal(), k = 0..n-1 */
void dsgdo_fill_normal(dsgdo_rng* r, double sigma, double* out, uint64_t n) {
  for (uint64_t k = 0; k < n; ++k) out[k] = sigma * dsgdo_normal(r);
}

/* rng.cpp:64-70 */
double dsgdo_exponential(dsgdo_rng* r, double rate) { return -log(dsgdo_uniform01(r)) / rate; }

/* rng.cpp:72-91: n == 1 draws nothing; rejection at the top of the range */
uint32_t dsgdo_uniform_index(dsgdo_rng* r, uint32_t n) {
  if (n <= 1) return 0;
  const uint64_t span = n;
  const uint64_t limit = ~0ull - (~0ull % span);
  uint64_t x = dsgdo_rng_next(r);
  while (x >= limit) x = dsgdo_rng_next(r);
  return (uint32_t)(x % span);
}

/* ---- stream derivation rng.cpp:93-107 (FNV-1a + splitmix64 finalizer) */
static const char* purpose_name(int purpose) {
  switch (purpose) {
    case DSGDO_PURPOSE_NOISE: return "gradient-noise";
    case DSGDO_PURPOSE_SAMPLE: return "sample";
    case DSGDO_PURPOSE_PARTNER: return "partner-choice";
    case DSGDO_PURPOSE_CLOCK: return "clock";
    case DSGDO_PURPOSE_STRAGGLER: return "straggler";
    case DSGDO_PURPOSE_INIT: return "init";
  }
  return "unknown";
}

static uint64_t fnv_byte(uint64_t h, uint8_t b) { return (h ^ b) * 1099511628211ull; }

static uint64_t fnv_u64(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) h = fnv_byte(h, (uint8_t)(v >> (8 * i)));
  return h;
}

uint64_t dsgdo_derive_stream_seed(uint64_t root_seed, const char* run_id, uint32_t node_id,
                                  int purpose) {
  uint64_t h = 1469598103934665603ull;
  h = fnv_u64(h, root_seed);
  for (const char* c = run_id; *c; ++c) h = fnv_byte(h, (uint8_t)*c);
  h = fnv_byte(h, 0);
  for (const char* c = purpose_name(purpose); *c; ++c) h = fnv_byte(h, (uint8_t)*c);
  h = fnv_byte(h, 0);
  h = fnv_u64(h, node_id);
  uint64_t z = h + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void dsgdo_make_stream(dsgdo_rng* r, uint64_t root_seed, const char* run_id, uint32_t node_id,
                       int purpose) {
  dsgdo_rng_seed(r, dsgdo_derive_stream_seed(root_seed, run_id, node_id, purpose));
}

/* ---- core.cpp:82-92 */
double dsgdo_step_size_at(const dsgdo_hyper* h, uint64_t t) {
  double alpha = h->alpha0;
  for (uint32_t i = 0; i < h->n_anneal; ++i) {
    if (h->anneal_at[i] <= t)
      alpha *= h->anneal_factor;
    else
      break;
  }
  return alpha;
}

/* ---- simulator.cpp:69-88 */
void dsgdo_draw_pull_partners(dsgdo_rng* partner_streams, uint32_t p, uint32_t* out) {
  for (uint32_t i = 0; i < p; ++i) out[i] = dsgdo_uniform_index(&partner_streams[i], p);
}

void dsgdo_draw_push_targets(dsgdo_rng* partner_streams, uint32_t p, uint32_t* out) {
  for (uint32_t i = 0; i < p; ++i) {
    uint32_t j = dsgdo_uniform_index(&partner_streams[i], p - 1);
    if (j >= i) ++j;
    out[i] = j;
  }
}

void dsgdo_pull_schedule(uint64_t seed, const char* run_id, uint32_t p, uint32_t tau,
                         uint64_t rounds, uint32_t* out) {
  dsgdo_rng* s = (dsgdo_rng*)malloc(sizeof(dsgdo_rng) * p);
  for (uint32_t i = 0; i < p; ++i) dsgdo_make_stream(&s[i], seed, run_id, i, DSGDO_PURPOSE_PARTNER);
  for (uint64_t r = 0; r < rounds; ++r) {
    if (r > 0 && r % tau == 0)
      dsgdo_draw_pull_partners(s, p, out + r * p);
    else
      for (uint32_t i = 0; i < p; ++i) out[r * p + i] = 0xffffffffu;
  }
  free(s);
}

#define R double
#define SFX f64
#include "dsgd_oracle_impl.inc"
#undef R
#undef SFX

#define R float
#define SFX f32
#include "dsgd_oracle_impl.inc"
#undef R
#undef SFX

/* ---- LogisticObjective helpers (objectives.cpp:34-38, 147-162) ---- */
double dsgdo_sigmoid(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

void dsgdo_draw_rows(dsgdo_rng* sample, uint64_t begin, uint64_t end, uint32_t batch,
                     uint64_t* rows) {
  const uint32_t span = (uint32_t)(end - begin);
  for (uint32_t b = 0; b < batch; ++b) rows[b] = begin + dsgdo_uniform_index(sample, span);
}

static double log1pexp(double z) { /* objectives.cpp:29-32 */
  if (z > 0.0) return z + log1p(exp(-z));
  return log1p(exp(z));
}

double dsgdo_logistic_value(uint64_t n, uint64_t d, const double* X, const int32_t* y, double l2,
                            const double* theta) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double z = 0.0;
    for (uint64_t k = 0; k < d; ++k) z += X[i * d + k] * theta[k];
    s += log1pexp(z) - (double)y[i] * z;
  }
  double sq = 0.0; /* ParamVec::squared_norm: sequential sum of squares */
  for (uint64_t k = 0; k < d; ++k) sq += theta[k] * theta[k];
  return s / (double)n + 0.5 * l2 * sq;
}
