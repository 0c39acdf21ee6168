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


def logistic_dataset():
    """A small LogisticObjective (F1 row of SURVEY §8(f)): n = 48 rows,
    d = 37 (not a multiple of any vector width), labels from a planted model,
    l2 = 0.05; node i of p = 4 samples rows [12 i, 12 i + 12) (sharded, the
    runner.cpp:100-115 shape)."""
    rng = np.random.default_rng(1611)
    n, d = 48, 37
    X = rng.standard_normal((n, d)) / np.sqrt(d)
    w = rng.standard_normal(d) * 3.0
    y = (X @ w + 0.3 * rng.standard_normal(n) > 0).astype(np.int32)
    ranges = np.array([[12 * i, 12 * i + 12] for i in range(4)], dtype=np.uint64)
    return X, y, 0.05, ranges


def _lg(protocol, **kw):
    hk = dict(alpha0=0.5, anneal_at=(25,), mu=0.9, weight_decay=1e-4, batch=3, beta_gossip=0.4,
              beta_ea=0.2, tau=1)
    hk.update(kw.pop("hyper", {}))
    base = dict(protocol=protocol, p=4, hyper=H(**hk), sigma=0.01, spectrum=[1.0] * 37,
                init_kind=O.INIT_GAUSSIAN, init_scale=0.5, rounds=40, run_id="lg/" + str(protocol))
    base.update(kw)
    return O.SimConfig(**base)


# The logistic trajectories (run_sync / run_async with sharded LogisticObjective
# node objectives; spectrum only carries d).
LOGISTIC_CASES = {
    "lg_allreduce": _lg(O.ALLREDUCE, per_node_scope=True),
    "lg_allreduce_agg": _lg(O.ALLREDUCE, per_node_scope=False, hyper=dict(batch=1)),
    "lg_pull": _lg(O.PULL),
    "lg_push": _lg(O.PUSH, hyper=dict(tau=2)),
    "lg_ea": _lg(O.ELASTIC, hyper=dict(batch=2)),
    "lg_stale": _lg(O.STALE),
    "lg_fresh": _lg(O.FRESH, hyper=dict(tau=2)),
    "lg_async": _lg(O.ASYNC_PULL, hyper=dict(mu=0.0), events=120, rounds=1),
    "lg_ea_poisson": _lg(O.ELASTIC, poisson=True, events=120, hyper=dict(tau=2)),
}


def make_logistic():
    X, y, l2, ranges = logistic_dataset()
    out = {"X": X, "y": y, "l2": np.float64(l2), "ranges": ranges}
    # stochastic_gradient known answers: theta, sample-stream seed, range, batch
    rng = np.random.default_rng(7)
    for k, (batch, b, e) in enumerate(((1, 0, 48), (3, 12, 24), (8, 0, 48))):
        theta = rng.standard_normal(X.shape[1])
        seed = O.derive_stream_seed(3, "lg/kat", k, "sample")
        O.ref_set_logistic(X, y, l2)
        out[f"kat{k}_theta"] = theta
        out[f"kat{k}_meta"] = np.array([batch, b, e, seed], dtype=np.uint64)
        out[f"kat{k}_grad"] = O.ref_logistic_grad(theta, batch, seed, b, e)
    for name, cfg in LOGISTIC_CASES.items():
        O.ref_set_logistic(X, y, l2, ranges)
        th, dp, t, c = O.ref_run(cfg)
        out.update({f"{name}_theta": th, f"{name}_dprev": dp, f"{name}_t": t,
                    f"{name}_center": c})
    O.ref_set_logistic(None, None, 0.0)
    np.savez(os.path.join(HERE, "logistic.npz"), **out)


# make_trace_record cadence cases: (RUN_CASES / LOGISTIC_CASES name, trace_every)
TRACE_CASES = {"c1_allreduce": 250, "pull8": 7, "push5": 9, "ea8": 10, "stale4": 10,
               "fresh4": 6, "async8": 50, "ea8_poisson": 40, "lg_pull": 8}


def make_traces():
    out = {}
    X, y, l2, ranges = logistic_dataset()
    for name, every in TRACE_CASES.items():
        if name.startswith("lg_"):
            O.ref_set_logistic(X, y, l2, ranges)
            cfg = LOGISTIC_CASES[name]
        else:
            O.ref_set_logistic(None, None, 0.0)
            cfg = RUN_CASES[name]
        rec, text = O.ref_run_traced(cfg, every)
        out[f"{name}_rec"] = rec
        out[f"{name}_jsonl"] = np.array(text)
    O.ref_set_logistic(None, None, 0.0)
    np.savez(os.path.join(HERE, "traces.npz"), **out)


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: needs /root/reference")
    if sys.argv[1:] in (["logistic"], ["traces"]):
        {"logistic": make_logistic, "traces": make_traces}[sys.argv[1]]()
        return
    make_logistic()
    make_traces()
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
