// dsgd_worker.cpp -- a C++-only multi-GPU host for the drop-in ABI: the
// B200 counterpart of the reference's run_transport (transport.cpp:306-555,
// one worker per node), with one PROCESS per GPU instead of one thread per
// node and NVLink peer memory / NCCL instead of the mailbox network.
//
//   dsgd_worker --gpus N [--d 25000000] [--rounds 50] [--protocol all-reduce|pull-gossip|elastic-avg]
//
// The parent forks one worker per GPU before any CUDA call; the workers
// exchange their dsgd_ctx_export_handle blobs and the NCCL unique id through
// an anonymous shared mapping guarded by a process-shared barrier, connect,
// run the per-step loop (dsgd_run_rounds, synthetic quadratic gradients +
// device Philox noise) and report the device time measured by the library.
// No Python, no torch.
#include <pthread.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dsgd_b200.hpp"

namespace {

struct Shared {
  pthread_barrier_t barrier;
  char nccl_id[DSGD_NCCL_ID_BYTES];
  double ms[64];
  double wall_ms[64];
  uint64_t hash[64];
  int status[64];
  char backend[32];
  char note[256];
  char blobs[64][DSGD_HANDLE_BYTES];
};

// FNV-1a over the parameter bytes: ranks of an all-reduce must agree bit for bit
uint64_t fnv(const std::vector<double>& v) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* b = reinterpret_cast<const unsigned char*>(v.data());
  for (size_t i = 0; i < v.size() * sizeof(double); ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

int run_worker(int rank, int world, uint64_t d, uint64_t rounds, dsgd_protocol proto,
               Shared* sh) {
  using namespace dsgd_b200;
  try {
    const uint32_t flags =
        DSGD_CTX_QUADRATIC | (proto == DSGD_ELASTIC_AVG ? DSGD_CTX_CENTER : 0u);
    Context ctx(d, world, DSGD_F32, rank, flags, rank, 1);
    // quadratic objective s = 1, opt = 0; theta_0 = 1 (common start)
    ctx.set_vector(0, DSGD_BUF_SPECTRUM, std::vector<double>(d, 1.0));
    ctx.set_vector(0, DSGD_BUF_OPT, std::vector<double>(d, 0.0));
    ctx.set_state(0, std::vector<double>(d, 1.0), {}, 0);
    check(dsgd_ctx_export_handle(ctx.get(), sh->blobs[rank]));
    if (rank == 0) check(dsgd_nccl_unique_id(sh->nccl_id));
    pthread_barrier_wait(&sh->barrier);
    check(dsgd_ctx_connect_peers(ctx.get(), sh->blobs));
    check(dsgd_ctx_init_nccl(ctx.get(), sh->nccl_id, rank, world));
    if (rank == 0) {  // the library's own all-reduce choice (NVLS set up without torch)
      const char* name = nullptr;
      const char* note = nullptr;
      check(dsgd_ctx_allreduce_backend(ctx.get(), &name, &note));
      std::snprintf(sh->backend, sizeof(sh->backend), "%s", name);
      std::snprintf(sh->note, sizeof(sh->note), "%s", note);
    }
    if (proto == DSGD_ELASTIC_AVG) check(dsgd_ea_init_center(ctx.get()));
    check(dsgd_ctx_seed_streams(ctx.get(), 1, "run/trial0"));

    Hyperparams h;
    h.alpha0 = 0.05;
    h.anneal_at.clear();
    dsgd_run_desc run{};
    run.protocol = proto;
    run.hyper = h.c();
    run.scope = DSGD_SCOPE_AGGREGATE;
    run.grad = dsgd_grad_spec{DSGD_GRAD_QUADRATIC, nullptr, 2, nullptr, 0.01, 7};
    run.rounds = 3;  // warm-up
    check(dsgd_run_rounds(ctx.get(), &run));
    ctx.sync();
    pthread_barrier_wait(&sh->barrier);
    check(dsgd_profile_enable(ctx.get(), 1));
    run.rounds = rounds;
    const auto t0 = std::chrono::steady_clock::now();
    check(dsgd_run_rounds(ctx.get(), &run));
    ctx.sync();
    sh->wall_ms[rank] =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    double ms = 0.0;
    for (int k = 0; k < DSGD_K_COUNT; ++k) {
      double part = 0.0;
      uint64_t n = 0;
      check(dsgd_profile_read(ctx.get(), static_cast<dsgd_kernel_id>(k), &part, &n, 1));
      ms += part;
    }
    sh->ms[rank] = ms;
    std::vector<double> th(d);
    ctx.get_state(0, &th, nullptr, nullptr);
    sh->hash[rank] = fnv(th);
    sh->status[rank] = std::isfinite(th[0]) && std::isfinite(th[d - 1]) ? 0 : 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    sh->status[rank] = 1;
    return 1;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  int world = 2;
  uint64_t d = 25000000, rounds = 50;
  std::string proto_name = "all-reduce";
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    if (k == "--gpus") world = std::atoi(argv[i + 1]);
    if (k == "--d") d = std::strtoull(argv[i + 1], nullptr, 10);
    if (k == "--rounds") rounds = std::strtoull(argv[i + 1], nullptr, 10);
    if (k == "--protocol") proto_name = argv[i + 1];
  }
  const dsgd_protocol proto = proto_name == "pull-gossip"   ? DSGD_PULL_GOSSIP
                              : proto_name == "elastic-avg" ? DSGD_ELASTIC_AVG
                                                            : DSGD_ALLREDUCE;
  if (world < 2 || world > 64) {
    std::fprintf(stderr, "--gpus must be in [2, 64]\n");
    return 2;
  }
  auto* sh = static_cast<Shared*>(mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE,
                                       MAP_SHARED | MAP_ANONYMOUS, -1, 0));
  std::memset(sh, 0, sizeof(Shared));
  pthread_barrierattr_t attr;
  pthread_barrierattr_init(&attr);
  pthread_barrierattr_setpshared(&attr, PTHREAD_PROCESS_SHARED);
  pthread_barrier_init(&sh->barrier, &attr, world);
  std::vector<pid_t> kids;
  for (int r = 0; r < world; ++r) {
    const pid_t pid = fork();
    if (pid == 0) _exit(run_worker(r, world, d, rounds, proto, sh));
    kids.push_back(pid);
  }
  int bad = 0;
  for (pid_t pid : kids) {
    int st = 0;
    waitpid(pid, &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) bad = 1;
  }
  double worst = 0.0, wall = 0.0;
  bool same = true;
  for (int r = 0; r < world; ++r) {
    worst = std::max(worst, sh->ms[r]);
    wall = std::max(wall, sh->wall_ms[r]);
    bad |= sh->status[r];
    same = same && sh->hash[r] == sh->hash[0];
  }
  const double us_round = worst * 1e3 / static_cast<double>(rounds);
  const double us_wall = wall * 1e3 / static_cast<double>(rounds);
  std::printf("{\"tool\": \"dsgd_worker\", \"protocol\": \"%s\", \"gpus\": %d, \"d\": %llu, "
              "\"rounds\": %llu, \"allreduce_backend\": \"%s\", \"nvls_note\": \"%s\", "
              "\"us_per_round_kernels\": %.2f, \"us_per_round_wall\": %.2f, "
              "\"param_updates_per_s\": %.4e, \"ranks_identical\": %s, \"ok\": %s}\n",
              proto_name.c_str(), world, (unsigned long long)d, (unsigned long long)rounds,
              sh->backend, sh->note, us_round, us_wall, world * (double)d / (us_wall * 1e-6),
              same ? "true" : "false", bad ? "false" : "true");
  return bad;
}
