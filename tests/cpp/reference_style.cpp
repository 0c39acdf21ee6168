// Reference-style C++ caller of the drop-in ABI (include/dsgd_b200.hpp):
// the hand values of proj/tests/test_protocols.cpp, through the GPU kernels.
// Built by tests/test_cpp_caller.py; exit code 0 == all checks passed.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "dsgd_b200.hpp"

using namespace dsgd_b200;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static bool approx(double a, double b, double rel = 1e-15) {
  return std::fabs(a - b) <= rel * std::fmax(std::fabs(a), std::fabs(b));
}

static Hyperparams plain(double alpha, double mu = 0.0) {
  Hyperparams h;
  h.alpha0 = alpha;
  h.anneal_at.clear();
  h.mu = mu;
  h.weight_decay = 0.0;
  return h;
}

int main() {
  // local sgd step: scalar quadratic hand values (test_protocols.cpp:94-103)
  {
    Context ctx(1, 1, DSGD_F64, 0, DSGD_CTX_QUADRATIC);
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, {1.0});
    ctx.set_vector(0, DSGD_BUF_OPT, {0.0});
    ctx.set_state(0, {2.0}, {0.0}, 0);
    ctx.local_sgd_step(plain(0.1));
    std::vector<double> th(1), dp(1);
    std::uint64_t t = 0;
    ctx.get_state(0, &th, &dp, &t);
    CHECK(approx(th[0], 1.8) && approx(dp[0], -0.2) && t == 1);
  }
  // two momentum steps 1 -> 0.9 -> 0.729 (113-125)
  {
    Context ctx(1, 1, DSGD_F64, 0, DSGD_CTX_QUADRATIC);
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, {1.0});
    ctx.set_vector(0, DSGD_BUF_OPT, {0.0});
    ctx.set_state(0, {1.0}, {0.0}, 0);
    ctx.local_sgd_step(plain(0.1, 0.9));
    ctx.local_sgd_step(plain(0.1, 0.9));
    std::vector<double> th(1);
    ctx.get_state(0, &th, nullptr, nullptr);
    CHECK(approx(th[0], 0.729, 1e-14));
  }
  // all-reduce of equal deltas 4 -> 3.6 (146-155); pull round -> 1.8 (316-328)
  {
    Context ctx(1, 2, DSGD_F64, 0, DSGD_CTX_QUADRATIC);
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, {1.0});
    ctx.set_vector(0, DSGD_BUF_OPT, {0.0});
    ctx.set_state(0, {4.0}, {0.0}, 0);
    ctx.set_state(1, {4.0}, {0.0}, 0);
    ctx.allreduce_round(plain(0.1));
    std::vector<double> a(1), b(1);
    ctx.get_state(0, &a, nullptr, nullptr);
    ctx.get_state(1, &b, nullptr, nullptr);
    CHECK(approx(a[0], 3.6) && approx(b[0], 3.6));
    ctx.set_state(0, {1.0}, {0.0}, 0);
    ctx.set_state(1, {3.0}, {0.0}, 0);
    ctx.pull_gossip_round(plain(0.1), {1, 0});
    ctx.get_state(0, &a, nullptr, nullptr);
    ctx.get_state(1, &b, nullptr, nullptr);
    CHECK(approx(a[0], 1.8) && approx(b[0], 1.8));
    bool threw = false;
    try {
      ctx.pull_gossip_round(plain(0.1), {7, 0});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // EASGD client 1 -> 0.9, center 0 -> 0.1 (249-260)
  {
    Context ctx(1, 1, DSGD_F64, 0, DSGD_CTX_QUADRATIC | DSGD_CTX_CENTER);
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, {1.0});
    ctx.set_vector(0, DSGD_BUF_OPT, {0.0});
    ctx.set_vector(0, DSGD_BUF_CENTER, {0.0});
    ctx.set_state(0, {1.0}, {0.0}, 0);
    Hyperparams h = plain(0.0);
    h.beta_ea = 0.1;
    ctx.ea_round(h, true);
    std::vector<double> th(1);
    ctx.get_state(0, &th, nullptr, nullptr);
    const auto c = ctx.get_vector(0, DSGD_BUF_CENTER, 1);
    CHECK(approx(th[0], 0.9) && approx(c[0], 0.1));
  }
  // push mix (0,3,6) -> (3,1.5,4.5) via a round with alpha 0 (342-354)
  {
    Context ctx(1, 3, DSGD_F64, 0, DSGD_CTX_QUADRATIC);
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, {1.0});
    ctx.set_vector(0, DSGD_BUF_OPT, {0.0});
    const double x[3] = {0.0, 3.0, 6.0};
    for (int i = 0; i < 3; ++i) ctx.set_state(i, {x[i]}, {0.0}, 0);
    ctx.push_gossip_round(plain(0.0), {1, 2, 0});
    const double want[3] = {3.0, 1.5, 4.5};
    for (int i = 0; i < 3; ++i) {
      std::vector<double> th(1);
      ctx.get_state(i, &th, nullptr, nullptr);
      CHECK(approx(th[0], want[i]));
    }
  }
  // LogisticObjective (test_objectives.cpp tiny_logistic): at theta = 0 every
  // z = 0, sigmoid = 1/2, so the one-row minibatch gradient is (1/2 - y) x;
  // a plain step theta -= alpha * g
  {
    Context ctx(2, 1, DSGD_F64, 0, 0);
    ctx.set_logistic({{1.0, 0.0}, {0.0, 1.0}, {1.0, 1.0}, {-1.0, 0.5}}, {1, 0, 1, 0}, 0.1);
    const double y[4] = {1, 0, 1, 0};
    const double X[4][2] = {{1.0, 0.0}, {0.0, 1.0}, {1.0, 1.0}, {-1.0, 0.5}};
    for (uint64_t r = 0; r < 4; ++r) {
      ctx.set_state(0, {0.0, 0.0}, {0.0, 0.0}, 0);
      Gradient g;
      g.source = DSGD_GRAD_LOGISTIC;
      g.rows = {r};
      ctx.local_sgd_step(plain(0.5), g);
      std::vector<double> th(2);
      ctx.get_state(0, &th, nullptr, nullptr);
      for (int k = 0; k < 2; ++k) CHECK(approx(th[k], -0.5 * ((0.5 - y[r]) * X[r][k]), 1e-15));
    }
    // the constructor's checks surface as std::invalid_argument
    bool threw = false;
    try {
      ctx.set_logistic({{1.0, 0.0}}, {2}, 0.1);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  if (failures == 0) std::printf("reference-style C++ caller: all checks passed\n");
  return failures == 0 ? 0 : 1;
}
