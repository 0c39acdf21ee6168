"""Single-process multi-GPU driver for profiling the NVLink kernels.

    python tools/nvlink_profile.py --gpus 2 --protocol all-reduce [--d 25000000] [--rounds 6]

One process drives an in-process group (dsgd_group_create_inproc) with rank
r on GPU r: the same kernels, peer mappings and (for p > 2) the library's
own NVSwitch multicast object as one process per GPU, but every launch is
issued from this thread in rank order, so each kernel's cross-GPU waits are
already satisfied when it starts.  That is what lets ncu -- which serialises
and replays every kernel -- profile the peer-read gossip kernel, the
one-shot / two-shot all-reduce and the EASGD chain with their NVLink
counters (nvlrx__bytes / nvltx__bytes) without a deadlock.

Prints one JSON line (backend, per-round wall time over the timed rounds).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1611_04581_b200 import _native as N  # noqa: E402
from paper_1611_04581_b200.engine import Group, Hyperparams, run_rounds_inproc  # noqa: E402

PROTO = {"all-reduce": N.ALLREDUCE, "pull-gossip": N.PULL_GOSSIP, "elastic-avg": N.ELASTIC_AVG,
         "push-gossip": N.PUSH_GOSSIP}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--protocol", default="all-reduce", choices=sorted(PROTO))
    ap.add_argument("--d", "--params", dest="d", type=int, default=25_000_000)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    proto = PROTO[a.protocol]
    gs = Group.inproc(a.d, a.gpus, dtype="f32", devices=list(range(a.gpus)), quadratic=True,
                      center=proto == N.ELASTIC_AVG)
    rng = np.random.default_rng(3)
    for r, g in enumerate(gs):
        g.set_quadratic(np.ones(a.d))
        g.set_state(0, rng.normal(size=a.d))
        g.seed_streams(1, "run/trial0")
    if proto == N.ELASTIC_AVG:
        gs[0].ea_init_center()
    h = Hyperparams(alpha0=0.05, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    kw = dict(grad="quadratic", noise=("device", 0.01, 7))
    run_rounds_inproc(gs, proto, h, a.warmup, **kw)
    for g in gs:
        g.sync()
    t0 = time.perf_counter()
    run_rounds_inproc(gs, proto, h, a.rounds, **kw)
    for g in gs:
        g.sync()
    dt = (time.perf_counter() - t0) / a.rounds
    backend, note = gs[0].allreduce_info()
    for g in gs:
        g.close()
    print(json.dumps({"tool": "nvlink_profile", "gpus": a.gpus, "protocol": a.protocol, "d": a.d,
                      "rounds": a.rounds, "allreduce_backend": backend, "nvls_note": note,
                      "us_per_round_wall": dt * 1e6}))


if __name__ == "__main__":
    main()
