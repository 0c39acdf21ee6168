"""Multi-GPU parity worker (launched by tests/test_multigpu.py under
torchrun, one process per GPU).  Each rank hosts one node; after a run the
ranks all-gather their states and rank 0 compares with the oracle."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_1611_04581_b200 import driver as D
    from paper_1611_04581_b200 import protocols as P
    from paper_1611_04581_b200.engine import Group, Hyperparams

    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    results = {}
    names = {"all-reduce": O.ALLREDUCE, "all-reduce-pn": O.ALLREDUCE, "elastic-avg": O.ELASTIC,
             "pull-gossip": O.PULL, "push-gossip": O.PUSH, "gossip-stale": O.STALE,
             "gossip-fresh": O.FRESH}
    if len(sys.argv) > 2 and sys.argv[2] == "allreduce-only":
        names = {"all-reduce": O.ALLREDUCE, "all-reduce-pn": O.ALLREDUCE}
    if len(sys.argv) > 2 and sys.argv[2] == "logistic":
        logistic(rank, world, local, dtype, dist)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "timeout":
        timeout_case(rank, world, local, dtype, dist)
        return
    for proto, oid in names.items():
        # EASGD: a staged chain with several chunks per CTA and a ragged tail;
        # MGPU_AR_D / MGPU_ROUNDS: the all-reduce at a size that takes the
        # multi-pipeline two-shot path
        d = 1031 if proto != "elastic-avg" else 148 * 5 * 2048 + 1031
        rounds = 25
        if proto.startswith("all-reduce") and os.environ.get("MGPU_AR_D"):
            d = int(os.environ["MGPU_AR_D"])
            rounds = int(os.environ.get("MGPU_ROUNDS", "6"))
        hk = dict(alpha0=0.05, anneal_at=(20,), mu=0.9, weight_decay=1e-4, beta_gossip=0.4,
                  beta_ea=0.15, tau=1)
        ar = proto.startswith("all-reduce")
        pn = proto == "all-reduce-pn"
        cfg = O.SimConfig(protocol=oid, p=world, hyper=O.HyperParams(**hk), sigma=0.05,
                          spectrum=list(np.linspace(0.5, 2.0, d)),
                          init_kind=O.INIT_OFFSET_ONES if ar else O.INIT_GAUSSIAN,
                          rounds=rounds, per_node_scope=pn, run_id=f"mg/{proto}")
        obj = P.QuadraticObjective(cfg.spectrum)
        dcfg = D.SimConfig(protocol="all-reduce" if ar else proto, p=world, hyper=Hyperparams(**hk),
                           noise=P.NoiseModel.gaussian_per_coord(0.05, d),
                           init=D.InitSpec("offset-ones" if ar else "gaussian-spread"),
                           momentum_scope="per-node" if pn else "aggregate",
                           rounds=rounds, run_id=f"mg/{proto}")
        thetas = D.make_initial_nodes(dcfg, obj)
        g = Group.distributed(d, rank, world, local, dtype=dtype, quadratic=True, noise=True,
                              center=proto == "elastic-avg")
        g.set_timeout(20.0)
        g.set_quadratic(obj.spectrum)
        g.set_state(0, thetas[rank])
        if proto == "elastic-avg" and rank == 0:
            # the reference's pivot-form spatial mean of the initial thetas
            # in the context's precision, exactly as spatial_mean_f32/f64 does
            npd = np.float64 if dtype == "f64" else np.float32
            th = thetas.astype(npd)
            dev = np.zeros(d, dtype=npd)
            for i in range(1, world):
                dev = dev + (th[i] - th[0])
            c = th[0] + dev * (npd(1) / npd(world))
            g.set_center(c.astype(np.float64))
        dist.barrier()
        g.seed_streams(1, f"mg/{proto}")
        g.run_rounds(D.PROTOCOLS[dcfg.protocol], Hyperparams(**hk), rounds,
                     scope="per-node" if pn else "aggregate",
                     grad="quadratic", host_noise_sigma=0.05)
        g.sync()
        th, dp, t = g.get_state(0)
        center = g.get_center() if proto == "elastic-avg" and rank == 0 else None
        allst = [None] * world
        dist.all_gather_object(allst, (th, dp, t))
        if rank == 0:
            npd = np.float64 if dtype == "f64" else np.float32
            if ar:
                # multi-GPU all-reduce = the reference's threaded transport
                # (ring_allreduce order), not the simulator's pivot mean
                on = O.run_transport_allreduce(cfg, dtype=npd)
                oth, odp, ot, oc = on.theta, on.dprev, on.t, None
                if dtype == "f64" and not pn:
                    from tests.golden.make_golden import transport_case
                    gp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                      "transport.npz")
                    if world in (2, 4, 8) and os.path.exists(gp):
                        gold = np.load(gp)[f"p{world}_theta"]
                        assert np.array_equal(oth, gold)
            else:
                oth, odp, ot, oc = O.run(cfg, dtype=npd)
            dev_th = np.array([s[0] for s in allst]).astype(npd)
            exact = dev_th.tobytes() == oth.tobytes()
            if ar:  # delta_prev too (aggregate: the average; per-node: own delta)
                dev_dp = np.array([s_[1] for s_ in allst]).astype(npd)
                exact = exact and dev_dp.tobytes() == odp.tobytes()
            rel = float(np.abs(dev_th.astype(float) - oth.astype(float)).max() /
                        np.abs(oth).max())
            same_ranks = all(np.array_equal(allst[0][0], s[0]) for s in allst)
            cexact = None
            if center is not None:
                cexact = center.astype(npd).tobytes() == oc.tobytes()
            results[proto] = {"bit_exact": exact, "max_rel": rel, "ranks_identical": same_ranks,
                              "center_exact": cexact,
                              "nvls": getattr(g, "allreduce_backend", "") == "nvls",
                              "backend": getattr(g, "allreduce_backend", "")}
        dist.barrier()
        g.close()
    if rank == 0:
        print("RESULT " + json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def timeout_case(rank, world, local, dtype, dist):
    """A peer that never arrives: rank 0 keeps stepping, the others stop
    after construction.  Rank 0's second pull round (RAW wait on its partner's
    round counter) and its second all-reduce round must end with
    TransportError after the configured timeout, not hang the GPU
    (transport.cpp:123-133, test_transport.cpp:148-155)."""
    import time

    import numpy as np

    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=0.0)
    res = {}
    for proto in ("pull-gossip", "all-reduce", "elastic-avg"):
        # elastic-avg: rank 0's second gated round waits for the ring closure
        # from rank p-1 inside the staged chain kernel's producer warp
        g = Group.distributed(4096, rank, world, local, dtype=dtype, quadratic=True,
                              center=proto == "elastic-avg")
        g.set_timeout(0.5)
        g.set_quadratic(np.ones(4096))
        g.set_state(0, np.full(4096, float(rank)))
        dist.barrier()
        if rank == 0:
            t0 = time.time()
            err = None
            try:
                for _ in range(2):
                    if proto == "pull-gossip":
                        g.pull_gossip_round(h, [1] + [0] * (world - 1), grad="quadratic")
                    elif proto == "elastic-avg":
                        g.ea_round(h, gated=True, grad="quadratic")
                    else:
                        g.allreduce_round(h, grad="quadratic")
                g.sync()
            except N.TransportError as e:
                err = str(e)
            res[proto] = {"timed_out": err is not None, "seconds": time.time() - t0,
                          "message": err}
        dist.barrier()
        g.close()
    if rank == 0:
        print("RESULT " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def logistic(rank, world, local, dtype, dist):
    """F1 on one node per GPU: the sharded LogisticObjective (rows from each
    rank's sample stream) through every protocol; rank 0 compares with the
    single-context run of the same configuration (itself pinned to the
    reference's trajectories by tests/test_gpu_logistic.py).  Gossip and
    EASGD run the same kernels in the same order -> bit-exact; the
    all-reduce sums in ring order vs the pivot mean -> tolerance."""
    from paper_1611_04581_b200 import driver as D
    from paper_1611_04581_b200 import protocols as P
    from paper_1611_04581_b200.engine import Group, Hyperparams
    from tests.golden.make_golden import logistic_dataset
    X, y, l2, _ = logistic_dataset()
    n, d = X.shape
    obj = P.LogisticObjective(X, y, l2)
    shards = [obj.shard(n * i // world, n * (i + 1) // world) for i in range(world)]
    hk = dict(alpha0=0.5, anneal_at=(10,), mu=0.9, weight_decay=1e-4, beta_gossip=0.4,
              beta_ea=0.15, tau=1, batch=3)
    results = {}
    for proto in ("all-reduce", "elastic-avg", "pull-gossip", "push-gossip", "gossip-stale",
                  "gossip-fresh"):
        dcfg = D.SimConfig(protocol=proto, p=world, hyper=Hyperparams(**hk),
                           noise=P.NoiseModel.gaussian_per_coord(0.01, d),
                           init=D.InitSpec("gaussian-spread", scale=0.5),
                           momentum_scope="aggregate", rounds=20, run_id=f"mgl/{proto}")
        thetas = D.make_initial_nodes(dcfg, obj)
        g = Group.distributed(d, rank, world, local, dtype=dtype, noise=True,
                              center=proto == "elastic-avg")
        g.set_timeout(20.0)
        g.set_logistic(X, y, l2)
        g.logistic_set_sample_range(0, *shards[rank].range)
        g.set_state(0, thetas[rank])
        if proto == "elastic-avg" and rank == 0:
            npd = np.float64 if dtype == "f64" else np.float32
            th = thetas.astype(npd)
            dev = np.zeros(d, dtype=npd)
            for i in range(1, world):
                dev = dev + (th[i] - th[0])
            g.set_center((th[0] + dev * (npd(1) / npd(world))).astype(np.float64))
        dist.barrier()
        g.seed_streams(1, f"mgl/{proto}")
        g.run_rounds(D.PROTOCOLS[proto], Hyperparams(**hk), 20, scope="aggregate",
                     grad="logistic", host_noise_sigma=0.01)
        g.sync()
        th, dp, t = g.get_state(0)
        center = g.get_center() if proto == "elastic-avg" and rank == 0 else None
        allst = [None] * world
        dist.all_gather_object(allst, (th, dp, t))
        dist.barrier()
        g.close()
        if rank == 0:
            r = D.run_sync(dcfg, obj, dtype=dtype, device=local, node_objs=shards)
            dev_th = np.array([s_[0] for s_ in allst])
            rel = float(np.abs(dev_th - r.theta).max() / np.abs(r.theta).max())
            res = {"bit_exact": dev_th.tobytes() == r.theta.tobytes(), "max_rel": rel,
                   "t_ok": [int(s_[2]) for s_ in allst] == r.t.tolist()}
            if center is not None:
                res["center_exact"] = center.tobytes() == r.center.tobytes()
            results[proto] = res
        dist.barrier()
    if rank == 0:
        print("RESULT " + json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
