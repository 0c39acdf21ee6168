"""Repeat the resident run_sync (integration/run_sync_b200.cpp) cases many
times in one process, optionally after in-process multi-GPU groups (argv[1]
== 'inproc'), and report any run that is not byte-identical to the golden
fixture."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from tests.golden.make_golden import RUN_CASES  # noqa: E402

HARNESS = os.path.join(ROOT, "integration", "_build", "libdsgd_ref_b200_harness.so")
g = np.load(os.path.join(ROOT, "tests", "golden", "runs.npz"))


def inproc_round():
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams, run_rounds_inproc
    import torch
    n = torch.cuda.device_count()
    for proto in (N.ALLREDUCE, N.ELASTIC_AVG, N.PULL_GOSSIP):
        gs = Group.inproc(4_000_000, n, dtype="f32", devices=list(range(n)), quadratic=True,
                          center=proto == N.ELASTIC_AVG)
        for r, gg in enumerate(gs):
            gg.set_quadratic(np.ones(4_000_000))
            gg.set_state(0, np.random.default_rng(r).normal(size=4_000_000))
            gg.seed_streams(1, "run/trial0")
        if proto == N.ELASTIC_AVG:
            gs[0].ea_init_center()
        h = Hyperparams(alpha0=0.05, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
        run_rounds_inproc(gs, proto, h, 10, grad="quadratic", noise=("device", 0.01, 7))
        for gg in gs:
            gg.sync()
        for gg in gs:
            gg.close()


bad = 0
reps = int(os.environ.get("REPS", "20"))
for rep in range(reps):
    if len(sys.argv) > 1 and sys.argv[1] == "inproc":
        inproc_round()
    for name in ("pull8", "fresh4", "push5", "ea8", "c1_allreduce"):
        with O.ref_library(HARNESS):
            th, dp, t, c, gn = O.ref_run_resident(RUN_CASES[name])
        ok = np.asarray(th).tobytes() == g[f"{name}_theta"].tobytes()
        if not ok:
            bad += 1
            print(f"rep {rep} {name} DIFF max_abs "
                  f"{float(np.abs(th - g[f'{name}_theta']).max())}", flush=True)
print(f"done reps={reps} bad={bad}", flush=True)
sys.exit(1 if bad else 0)
