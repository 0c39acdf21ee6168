"""The multi-GPU kernels on ONE GPU: p one-node contexts of an in-process
group (dsgd_group_create_inproc) share the device and one stream; every
round is issued rank by rank, so each cross-rank flag wait is already
satisfied when its kernel starts (no kernel ever waits on another running
kernel).  This runs the exact code the one-process-per-GPU path runs --
the peer-memory all-reduce in the reference ring order (one-shot for p <= 4,
two-shot ring reduce for any p), the EASGD chain (p - 1 hops + the ring
closure), the peer-read gossip / push / stale / fresh kernels with their
RAW / WAR round counters, the device trace over peers and the pivot-form
center init -- on the driver's single-GPU box, at p = 2, 3, 4 and 8.

Bars: the all-reduce is bit-exact with the reference's threaded transport
(ring_allreduce transport.cpp:183-248; the p = 2/4/8 fp64 runs also against
the compiled reference's fixture tests/golden/transport.npz); every other
rule bit-exact with the oracle's run_sync (simulator.cpp:234-369)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1611_04581_b200 import driver as D
from paper_1611_04581_b200 import protocols as P
from paper_1611_04581_b200.engine import Group, Hyperparams, run_rounds_inproc

pytestmark = pytest.mark.gpu

OID = {"all-reduce": O.ALLREDUCE, "all-reduce-pn": O.ALLREDUCE, "elastic-avg": O.ELASTIC,
       "pull-gossip": O.PULL, "push-gossip": O.PUSH, "gossip-stale": O.STALE,
       "gossip-fresh": O.FRESH}
HK = dict(alpha0=0.05, anneal_at=(20,), mu=0.9, weight_decay=1e-4, beta_gossip=0.4,
          beta_ea=0.15, tau=1)
NPD = {"f64": np.float64, "f32": np.float32}


def run_group(proto, world, dtype, d, rounds, monkeypatch, backend=None, sigma=0.05,
              run_id=None, devices=None):
    if backend:
        monkeypatch.setenv("DSGD_ALLREDUCE", backend)
    else:
        monkeypatch.delenv("DSGD_ALLREDUCE", raising=False)
    ar = proto.startswith("all-reduce")
    pn = proto == "all-reduce-pn"
    run_id = run_id or f"ip/{proto}/{world}"
    cfg = O.SimConfig(protocol=OID[proto], p=world, hyper=O.HyperParams(**HK), sigma=sigma,
                      spectrum=list(np.linspace(0.5, 2.0, d)),
                      init_kind=O.INIT_OFFSET_ONES if ar else O.INIT_GAUSSIAN,
                      rounds=rounds, per_node_scope=pn, run_id=run_id)
    obj = P.QuadraticObjective(cfg.spectrum)
    dcfg = D.SimConfig(protocol="all-reduce" if ar else proto, p=world, hyper=Hyperparams(**HK),
                       noise=None if sigma is None else P.NoiseModel.gaussian_per_coord(sigma, d),
                       init=D.InitSpec("offset-ones" if ar else "gaussian-spread"),
                       momentum_scope="per-node" if pn else "aggregate", rounds=rounds,
                       run_id=run_id)
    thetas = D.make_initial_nodes(dcfg, obj)
    gs = Group.inproc(d, world, dtype=dtype, quadratic=True, noise=True,
                      center=proto == "elastic-avg", devices=devices)
    try:
        for r, g in enumerate(gs):
            g.set_quadratic(obj.spectrum)
            g.set_state(0, thetas[r])
            g.seed_streams(1, run_id)
        if proto == "elastic-avg":
            gs[0].ea_init_center()  # rank 0 reads every rank's theta (pivot-form mean)
        run_rounds_inproc(gs, D.PROTOCOLS[dcfg.protocol], Hyperparams(**HK), rounds,
                          scope="per-node" if pn else "aggregate", grad="quadratic",
                          host_noise_sigma=sigma or 0.0)
        st = [g.get_state(0) for g in gs]
        center = gs[0].get_center() if proto == "elastic-avg" else None
        tr = gs[0].trace()  # the distributed trace: peer reads after every peer's last round
        kernels = sum(g.launch_count()[0] for g in gs)
    finally:
        for g in gs:
            g.close()
    npd = NPD[dtype]
    th = np.array([s[0] for s in st]).astype(npd)
    dp = np.array([s[1] for s in st]).astype(npd)
    t = np.array([s[2] for s in st], dtype=np.uint64)
    if ar:
        on = O.run_transport_allreduce(cfg, dtype=npd)
        oth, odp, ot, oc = on.theta, on.dprev, on.t, None
    else:
        oth, odp, ot, oc = O.run(cfg, dtype=npd)
    return dict(th=th, dp=dp, t=t, center=center, oth=oth, odp=odp, ot=ot, oc=oc, cfg=cfg,
                trace=tr, kernels=kernels)


def same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


def check(res, proto):
    assert res["t"].tolist() == res["ot"].tolist()
    assert same(res["th"], res["oth"]), float(np.abs(res["th"].astype(float) -
                                                     res["oth"].astype(float)).max())
    assert same(res["dp"], res["odp"])
    if res["center"] is not None:
        assert same(res["center"].astype(res["oc"].dtype), res["oc"])
    ref = O.trace(res["oth"], res["cfg"].spectrum)
    for k in ("sq_err_consensus", "sq_err_opt"):
        assert res["trace"][k] == pytest.approx(ref[k], rel=1e-9), k


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("proto", sorted(OID))
def test_inproc_group_matches_oracle(world, dtype, proto, monkeypatch):
    """d = 1031 (ragged vector tails, uneven ring chunks), 25 rounds, noise."""
    res = run_group(proto, world, dtype, 1031, 25, monkeypatch)
    check(res, proto)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_inproc_ring_allreduce_matches_reference_fixture(world, monkeypatch):
    """A5 ring_allreduce at p = 2/4/8: the oracle transport restatement this
    test compares with is itself the compiled reference's output
    (tests/golden/transport.npz, made by tests/golden/make_golden.py)."""
    from tests.golden.make_golden import transport_case
    cfg = transport_case(world)
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "transport.npz"))
    on = O.run_transport_allreduce(cfg)
    assert same(on.theta, gold[f"p{world}_theta"])
    res = run_group("all-reduce", world, "f64", cfg.d, cfg.rounds, monkeypatch,
                    backend="oneshot" if world <= 4 else "p2p", run_id=cfg.run_id)
    assert same(res["th"], gold[f"p{world}_theta"])


@pytest.mark.parametrize("world,backend", [(2, "p2p"), (3, "p2p"), (4, "p2p"), (3, "oneshot"),
                                           (4, "oneshot"), (8, "p2p")])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_inproc_allreduce_backends_staged_sizes(world, backend, dtype, monkeypatch):
    """Sizes that take the staged (cp.async.bulk) one-shot / two-shot delta
    kernels and the ring reduce with vector bodies + scalar heads/tails."""
    res = run_group("all-reduce", world, dtype, 3 * 2048 * 4 + 13, 6, monkeypatch, backend=backend)
    check(res, "all-reduce")


@pytest.mark.parametrize("pipes", [2, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_inproc_two_shot_pipelines(dtype, pipes, monkeypatch):
    """d >= 8M per rank: the two-shot round splits d into 2 (default) or 4
    (the >= 700M-per-worker default) pipelines with own counters; all four
    ranks' exchanges, then the reduces."""
    monkeypatch.setenv("DSGD_AR_PIPES", str(pipes))
    res = run_group("all-reduce", 4, dtype, (8 << 20) + 1031, 3, monkeypatch, backend="p2p",
                    sigma=None)
    check(res, "all-reduce")


@pytest.mark.parametrize("proto", ["pull-gossip", "elastic-avg", "push-gossip", "gossip-stale",
                                   "gossip-fresh"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_inproc_p8_staged_sizes(proto, dtype, monkeypatch):
    """p = 8 at a size that takes the staged peer-read gossip kernel
    (k_step_tma2) and a multi-chunk EASGD chain (7 hops + ring closure)."""
    res = run_group(proto, 8, dtype, 5 * 4096 + 7, 8, monkeypatch)
    check(res, proto)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_inproc_ea_chain_staged_ring_wraps(dtype, monkeypatch):
    """The staged EASGD chain (k_ea_chain_tma) with every CTA cycling its
    4-stage shared-memory ring several times (> 4 chunks per CTA on a
    148-SM grid) and a ragged last chunk: 3 ranks (2 hops + ring closure),
    4 rounds, bit-exact with the oracle."""
    res = run_group("elastic-avg", 3, dtype, 148 * 6 * 2048 + 13, 4, monkeypatch)
    check(res, "elastic-avg")



def n_gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("n_gpus() < 2")
@pytest.mark.parametrize("proto", sorted(OID))
def test_inproc_p8_across_gpus(proto, monkeypatch):
    """p = 8 ranks spread over every visible GPU (rank r on GPU r mod n):
    the 8-rank kernels -- the 7-hop EASGD chain + ring closure, 8-way
    gossip flags, the two-shot ring reduce at p = 8 -- with real NVLink
    traffic between the GPUs (the shape of an 8-GPU box the pool cannot
    provide), bit-exact with the oracle / the reference's ring order."""
    n = n_gpus()
    res = run_group(proto, 8, "f32", 5 * 4096 + 7, 6, monkeypatch,
                    devices=[r % n for r in range(8)], run_id=f"ipx/{proto}")
    check(res, proto)
