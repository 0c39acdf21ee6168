"""Generates the committed golden fixtures in tests/golden/ from the COMPILED
REFERENCE (oracle/_ref/libdsgd_ref.so, built by oracle/Makefile from
/root/reference/proj/src).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement on machines without /root/reference
(tests/test_oracle_golden.py::test_golden_*)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

H = O.HyperParams
RUN_CASES = {
    # reference quadratic, all-reduce, p=2 (2000 rounds)
    "c1_allreduce": O.SimConfig(protocol=O.ALLREDUCE, p=2, hyper=H(alpha0=0.05, anneal_at=(), mu=0.9, weight_decay=1e-4),
                                sigma=float(np.sqrt(0.01 / 4)), rounds=2000, per_node_scope=False,
                                run_id="c1/trial0"),
    "c1_allreduce_mu0": O.SimConfig(protocol=O.ALLREDUCE, p=2, hyper=H(alpha0=0.05, anneal_at=(), mu=0.0, weight_decay=0.0),
                                    sigma=float(np.sqrt(0.01 / 4)), rounds=2000, run_id="c1/trial0"),
    "pull8": O.SimConfig(protocol=O.PULL, p=8, hyper=H(alpha0=0.05, anneal_at=(50,), mu=0.9),
                         sigma=0.05, rounds=120, init_kind=O.INIT_GAUSSIAN, run_id="run/trial0"),
    "push5": O.SimConfig(protocol=O.PUSH, p=5, hyper=H(alpha0=0.05, mu=0.9, tau=2),
                         sigma=0.05, rounds=60, init_kind=O.INIT_GAUSSIAN, run_id="push/trial1"),
    "ea8": O.SimConfig(protocol=O.ELASTIC, p=8, hyper=H(alpha0=0.05, mu=0.9, beta_ea=0.1),
                       sigma=0.05, rounds=80, init_kind=O.INIT_GAUSSIAN, run_id="ea/trial0"),
    "ea8_poisson": O.SimConfig(protocol=O.ELASTIC, p=8, hyper=H(alpha0=0.05, mu=0.9, beta_ea=0.1, tau=2),
                               sigma=0.05, events=300, poisson=True, init_kind=O.INIT_GAUSSIAN,
                               run_id="eap/trial0"),
    "stale4": O.SimConfig(protocol=O.STALE, p=4, hyper=H(alpha0=0.05, mu=0.9, beta_gossip=0.4),
                          sigma=0.05, rounds=50, init_kind=O.INIT_GAUSSIAN, run_id="st"),
    "fresh4": O.SimConfig(protocol=O.FRESH, p=4, hyper=H(alpha0=0.05, mu=0.5, beta_gossip=0.4, tau=3),
                          sigma=0.05, rounds=50, init_kind=O.INIT_GAUSSIAN, run_id="fr"),
    "async8": O.SimConfig(protocol=O.ASYNC_PULL, p=8, hyper=H(alpha0=0.05, mu=0.0, beta_gossip=0.5),
                          sigma=0.05, events=400, init_kind=O.INIT_OFFSET_ONES, seed=2, run_id="c4/trial0"),
}


def transport_case(p: int) -> "O.SimConfig":
    """The multi-GPU all-reduce case of tests/mgpu_worker.py, for the
    reference's threaded transport (run_transport, ring_allreduce)."""
    d = 1031
    hk = dict(alpha0=0.05, anneal_at=(20,), mu=0.9, weight_decay=1e-4, beta_gossip=0.4,
              beta_ea=0.15, tau=1)
    return O.SimConfig(protocol=O.ALLREDUCE, p=p, hyper=O.HyperParams(**hk), sigma=0.05,
                       spectrum=list(np.linspace(0.5, 2.0, d)), init_kind=O.INIT_OFFSET_ONES,
                       rounds=25, per_node_scope=False, run_id="mg/all-reduce")


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: needs /root/reference")
    seed = 0x5EED
    np.savez(os.path.join(HERE, "streams.npz"), seed=np.uint64(seed), n=np.uint64(7),
             u64=O.ref_stream(seed, 0, 1000), normal=O.ref_stream(seed, 2, 500),
             index=O.ref_stream(seed, 3, 500, 7))
    runs = {}
    for name, cfg in RUN_CASES.items():
        th, dp, t, c = O.ref_run(cfg)
        runs.update({f"{name}_theta": th, f"{name}_dprev": dp, f"{name}_t": t, f"{name}_center": c})
    np.savez(os.path.join(HERE, "runs.npz"), **runs)
    ring = {}
    for p, d in ((2, 5), (3, 7), (8, 21), (8, 4096)):
        x = np.array([O.Stream(1000 + r).normals(d) for r in range(p)])
        ring[f"in_{p}_{d}"] = x
        ring[f"out_{p}_{d}"] = O.ref_ring_allreduce(x, chaos_seed=1)
    np.savez(os.path.join(HERE, "ring.npz"), **ring)
    tr = {}
    for p in (2, 4, 8):
        th, dp, t, _ = O.ref_run(transport_case(p), transport=True, chaos_seed=p)
        tr.update({f"p{p}_theta": th, f"p{p}_dprev": dp, f"p{p}_t": t})
    np.savez(os.path.join(HERE, "transport.npz"), **tr)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
