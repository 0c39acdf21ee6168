"""Parity of the B200 kernels (through the C ABI) with the CPU oracle.

Bars (BASELINE.md "Parity bars"):
  * fp64 contexts: bit-exact with the reference operation order (oracle
    fp64, itself pinned bit-exact to the compiled reference);
  * fp32 contexts: bit-exact with the same operation order in binary32
    (oracle fp32), and within 1e-5 max relative error of the fp64 oracle
    per step (teacher-forced);
  * peer / index selection: bit-exact (host streams, tests/test_abi.py).
"""
import numpy as np
import pytest

import oracle as O
from paper_1611_04581_b200 import _native as N
from paper_1611_04581_b200 import driver as D
from paper_1611_04581_b200 import protocols as P
from paper_1611_04581_b200.engine import Group, Hyperparams

pytestmark = pytest.mark.gpu

NP = {"f64": np.float64, "f32": np.float32}


def H(**kw):
    base = dict(alpha0=0.07, anneal_at=(3,), anneal_factor=0.5, mu=0.9, weight_decay=1e-3,
                beta_gossip=0.3, beta_ea=0.2, tau=1)
    base.update(kw)
    return base


def make_case(p, d, dtype, seed=0, fixed=False, noise=True, t0=3):
    rng = np.random.default_rng(seed)
    f = NP[dtype]
    c = dict(theta=rng.normal(size=(p, d)).astype(f), dprev=(0.1 * rng.normal(size=(p, d))).astype(f),
             t=np.full(p, t0, dtype=np.uint64), spec=rng.uniform(0.5, 2.0, d).astype(f),
             opt=rng.normal(size=d).astype(f),
             gfixed=rng.normal(size=(p, d)).astype(f) if fixed else None,
             noise=(0.05 * rng.normal(size=(p, d))).astype(f) if noise else None,
             center=rng.normal(size=d).astype(f))
    return c


def load_group(c, dtype):
    p, d = c["theta"].shape
    g = Group(d, p, dtype=dtype, quadratic=True, grad=True, noise=c["noise"] is not None,
              center=True)
    g.set_quadratic(c["spec"].astype(np.float64), c["opt"].astype(np.float64))
    for i in range(p):
        g.set_state(i, c["theta"][i].astype(np.float64), c["dprev"][i].astype(np.float64),
                    int(c["t"][i]))
        if c["gfixed"] is not None:
            g.set_vector(i, N.BUF_GRAD, c["gfixed"][i].astype(np.float64))
        if c["noise"] is not None:
            g.set_vector(i, N.BUF_NOISE, c["noise"][i].astype(np.float64))
    g.set_center(c["center"].astype(np.float64))
    return g


def read_group(g, p, dtype):
    f = NP[dtype]
    th, dp, t = zip(*[g.get_state(i) for i in range(p)])
    return np.array(th).astype(f), np.array(dp).astype(f), np.array(t, dtype=np.uint64)


def oracle_nodes(c):
    return O.Nodes(c["theta"], c["dprev"], c["t"], dtype=c["theta"].dtype)


def okw(c):
    return dict(spec=c["spec"], opt=c["opt"], gfixed=c["gfixed"], noise=c["noise"])


def same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


RULES = ["local", "allreduce", "allreduce_pn", "ea", "ea_ungated", "pull", "push", "stale",
         "fresh", "async"]


def run_rule(rule, g, n, c, h_kw, partner, target):
    h = Hyperparams(**h_kw)
    hc = O.HyperParams(**{k: v for k, v in h_kw.items()})
    grad = "buffer" if c["gfixed"] is not None else "quadratic"
    nz = c["noise"] is not None
    center = c["center"].copy()
    if rule == "local":
        g.local_sgd_step(h, grad=grad, noise=nz)
        O.local_sgd_step(n, hc, **okw(c))
    elif rule in ("allreduce", "allreduce_pn"):
        scope = "per-node" if rule == "allreduce_pn" else "aggregate"
        g.allreduce_round(h, scope=scope, grad=grad, noise=nz)
        O.allreduce_round(n, hc, per_node=rule == "allreduce_pn", **okw(c))
    elif rule in ("ea", "ea_ungated"):
        g.ea_round(h, gated=rule == "ea", grad=grad, noise=nz)
        O.ea_round(n, center, rule == "ea", hc, **okw(c))
    elif rule == "pull":
        g.pull_gossip_round(h, partner, grad=grad, noise=nz)
        O.pull_gossip_round(n, partner, hc, **okw(c))
    elif rule == "push":
        g.push_gossip_round(h, target, grad=grad, noise=nz)
        O.push_gossip_round(n, target, hc, **okw(c))
    elif rule == "stale":
        g.gossip_stale_round(h, partner, grad=grad, noise=nz)
        O.stale_round(n, partner, hc, **okw(c))
    elif rule == "fresh":
        g.gossip_fresh_round(h, partner, grad=grad, noise=nz)
        O.fresh_round(n, partner, hc, **okw(c))
    elif rule == "async":
        i, j = 0, n.p - 1
        g.async_pull_event(h, i, j, grad=grad, noise=nz)
        O.async_pull_event(n, i, j, hc, **okw(c))
    return center


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("p,d,fixed,noise,mu,wd", [
    (1, 1, False, False, 0.9, 1e-3),
    (2, 7, True, True, 0.0, 0.0),
    (5, 33, False, True, 0.9, 1e-3),
    (8, 1027, True, False, 0.5, 0.0),
    (3, 4099, False, True, 0.9, 1e-4),
])
def test_rule_bit_exact(dtype, rule, p, d, fixed, noise, mu, wd):
    if rule == "push" and p < 2:
        pytest.skip("push targets need p >= 2")
    c = make_case(p, d, dtype, seed=p * 1000 + d, fixed=fixed, noise=noise)
    rng = np.random.default_rng(d)
    partner = rng.integers(0, p, size=p).astype(np.uint32)
    target = np.array([(i + 1 + int(rng.integers(0, max(1, p - 1)))) % p for i in range(p)],
                      dtype=np.uint32)
    h_kw = H(mu=mu, weight_decay=wd)
    g = load_group(c, dtype)
    n = oracle_nodes(c)
    center = run_rule(rule, g, n, c, h_kw, partner, target)
    th, dp, t = read_group(g, p, dtype)
    assert same(th, n.theta), np.abs(th.astype(float) - n.theta.astype(float)).max()
    if rule != "async":
        assert same(dp, n.dprev)
    assert t.tolist() == n.t.tolist()
    if rule in ("ea", "ea_ungated"):
        assert same(g.get_center().astype(NP[dtype]), center)
    g.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_multi_round_state_machine(dtype):
    """Several rounds of mixed rules in one context (ping-pong buffers,
    momentum memory, clocks) stay bit-exact."""
    p, d = 6, 515
    c = make_case(p, d, dtype, seed=7, noise=False, t0=0)
    g = load_group(c, dtype)
    n = oracle_nodes(c)
    center = c["center"].copy()
    hk = H()
    h, hc = Hyperparams(**hk), O.HyperParams(**hk)
    rng = np.random.default_rng(1)
    for r in range(12):
        kind = r % 4
        partner = rng.integers(0, p, size=p).astype(np.uint32)
        if kind == 0:
            g.allreduce_round(h, grad="quadratic")
            O.allreduce_round(n, hc, spec=c["spec"], opt=c["opt"])
        elif kind == 1:
            g.pull_gossip_round(h, partner, grad="quadratic")
            O.pull_gossip_round(n, partner, hc, spec=c["spec"], opt=c["opt"])
        elif kind == 2:
            g.ea_round(h, gated=True, grad="quadratic")
            O.ea_round(n, center, True, hc, spec=c["spec"], opt=c["opt"])
        else:
            g.local_sgd_step(h, grad="quadratic")
            O.local_sgd_step(n, hc, spec=c["spec"], opt=c["opt"])
    th, dp, t = read_group(g, p, dtype)
    assert same(th, n.theta) and same(dp, n.dprev) and t.tolist() == n.t.tolist()
    g.close()


def test_misaligned_external_gradient_scalar_path():
    import torch
    p, d = 2, 1001
    c = make_case(p, d, "f32", seed=3, fixed=True, noise=False)
    g = load_group(c, "f32")
    buf = torch.zeros(p * d + 8, dtype=torch.float32, device="cuda")
    ptrs = []
    for i in range(p):
        off = 1 + i * (d + 3)  # 4-byte aligned, not 16-byte aligned
        buf[off:off + d] = torch.from_numpy(c["gfixed"][i]).cuda()
        ptrs.append(buf.data_ptr() + 4 * off)
    torch.cuda.synchronize()
    h_kw = H()
    g.local_sgd_step(Hyperparams(**h_kw), grad=ptrs)
    n = oracle_nodes(c)
    O.local_sgd_step(n, O.HyperParams(**h_kw), **okw(c))
    th, dp, _ = read_group(g, p, "f32")
    assert same(th, n.theta) and same(dp, n.dprev)
    g.close()


def test_grad_norm_out_matches_reference_norm():
    p, d = 3, 2000
    c = make_case(p, d, "f64", seed=11, noise=True)
    g = load_group(c, "f64")
    hk = H()
    v = g.allreduce_round(Hyperparams(**hk), grad="quadratic", noise=True, grad_norm=True)
    # model gradient (pre-noise) at the lookahead, max over nodes
    la = c["theta"] + hk["mu"] * c["dprev"]
    gm = c["spec"] * (la - c["opt"]) + hk["weight_decay"] * la
    assert v == pytest.approx(np.sqrt((gm ** 2).sum(axis=1)).max(), rel=1e-12)
    g.close()


# ------------------------------------------------------------ full size
@pytest.mark.parametrize("rule", ["local", "pull", "ea"])
def test_full_size_fp32_bit_exact(rule):
    """BASELINE sizes (25M / 10M params, fp32) against the fp32 oracle."""
    d, p = (25_000_000, 1) if rule == "local" else (10_000_000, 2)
    c = make_case(p, d, "f32", seed=5, fixed=True, noise=True)
    g = load_group(c, "f32")
    n = oracle_nodes(c)
    run_rule(rule, g, n, c, H(), np.array([1, 0][:p], dtype=np.uint32), None)
    th, dp, _ = read_group(g, p, "f32")
    assert same(th, n.theta) and same(dp, n.dprev)
    g.close()


# --------------------------------------------------- reference-mirror API
quad1 = P.QuadraticObjective([1.0], [0.0])


def plain(alpha, mu=0.0):
    return Hyperparams(alpha0=alpha, anneal_at=(), mu=mu, weight_decay=0.0)


def test_mirror_hand_values():
    """test_protocols.cpp golden values through the device kernels."""
    z = P.NoiseModel.zero(1)
    n = P.local_sgd_step(P.make_node(0, [2.0]), quad1, z, plain(0.1))
    assert n.theta[0] == pytest.approx(1.8, rel=1e-15) and n.t == 1
    assert n.delta_prev[0] == pytest.approx(-0.2, rel=1e-15)
    n = P.make_node(0, [1.0])
    n = P.local_sgd_step(n, quad1, z, plain(0.1, 0.9))
    n = P.local_sgd_step(n, quad1, z, plain(0.1, 0.9))
    assert n.theta[0] == pytest.approx(0.729, rel=1e-14)
    h = plain(0.1)
    h.weight_decay = 0.5
    assert P.local_sgd_step(P.make_node(0, [2.0]), quad1, z, h).theta[0] == pytest.approx(1.7)
    nodes = P.allreduce_round([P.make_node(0, [4.0]), P.make_node(1, [4.0])], quad1, z, plain(0.1))
    assert [x.theta[0] for x in nodes] == [pytest.approx(3.6, rel=1e-15)] * 2
    he = plain(0.0)
    he.beta_ea = 0.1
    node, upd = P.ea_client_step(P.make_node(0, [1.0]), [0.0], quad1, z, he)
    assert upd[0] == pytest.approx(0.1, rel=1e-15) and node.theta[0] == pytest.approx(0.9)
    s = P.ea_server_apply(P.ServerState(np.array([0.0])), [0.1])
    assert s.theta_center[0] == pytest.approx(0.1) and s.applied_updates == 1
    with pytest.raises(P.InvalidArgument):
        P.ea_server_apply(s, [1.0, 2.0])
    mixed = P.pull_mix([P.make_node(0, [1.0]), P.make_node(1, [3.0])], [1, 0])
    assert [x.theta[0] for x in mixed] == [2.0, 2.0]
    out = P.pull_gossip_round([P.make_node(0, [1.0]), P.make_node(1, [3.0])], [1, 0], quad1, z,
                              plain(0.1))
    assert [x.theta[0] for x in out] == [pytest.approx(1.8, rel=1e-15)] * 2
    out = P.push_mix([P.make_node(i, [v]) for i, v in enumerate([0.0, 3.0, 6.0])], [1, 2, 0])
    assert [x.theta[0] for x in out] == [pytest.approx(3.0), pytest.approx(1.5), pytest.approx(4.5)]
    with pytest.raises(P.InvalidArgument):
        P.push_mix([P.make_node(0, [1.0]), P.make_node(1, [2.0])], [0, 0])
    hs = plain(0.1)
    hs.beta_gossip = 0.5
    assert P.gossip_stale_step(P.make_node(0, [2.0]), [0.0], quad1, z, hs).theta[0] == \
        pytest.approx(0.8, rel=1e-15)
    assert P.gossip_fresh_step(P.make_node(0, [2.0]), [0.0], quad1, z, hs).theta[0] == \
        pytest.approx(0.9, rel=1e-15)
    ha = plain(0.1)
    ha.beta_gossip = 0.5
    out = P.async_pull_event([P.make_node(0, [2.0])], 0, 0, quad1, z, ha)
    assert out[0].theta[0] == pytest.approx(1.9, rel=1e-15)


def test_mirror_errors():
    z = P.NoiseModel.zero(1)
    a, b = P.make_node(0, [1.0]), P.make_node(1, [1.0])
    b.t = 3
    with pytest.raises(P.InvalidArgument):
        P.allreduce_round([a, b], quad1, z, plain(0.1))
    with pytest.raises(P.InvalidArgument):
        P.pull_mix([P.make_node(0, [1.0])], [7])
    with pytest.raises(P.InvalidArgument):
        P.ea_client_step(P.make_node(0, [1.0]), [0.0, 1.0], quad1, z, plain(0.1))


def test_mirror_equal_starts_stay_equal_under_noise():
    """test_protocols.cpp:174-187: exact equality under noise, 10 rounds."""
    obj = P.QuadraticObjective([1.0, 10.0])
    noise = P.NoiseModel.gaussian_per_coord(0.3, 2)
    nodes = [P.make_node(i, [1.0, -1.0], 1, "test") for i in range(4)]
    for _ in range(10):
        nodes = P.allreduce_round(nodes, obj, noise, plain(0.05))
        for x in nodes[1:]:
            assert same(x.theta, nodes[0].theta)


def test_mirror_consensus_at_optimum_every_protocol():
    obj = P.QuadraticObjective([1.0, 3.0], [0.5, -0.5])
    star = obj.opt
    z = P.NoiseModel.zero(2)
    h = plain(0.1, 0.9)
    h.beta_gossip, h.beta_ea = 0.5, 0.1
    mk = lambda: [P.make_node(i, star) for i in range(3)]  # noqa: E731
    outs = [P.allreduce_round(mk(), obj, z, h), P.pull_gossip_round(mk(), [1, 2, 0], obj, z, h),
            P.push_gossip_round(mk(), [1, 2, 0], obj, z, h),
            P.async_pull_event(mk(), 0, 2, obj, z, h)]
    for nodes in outs:
        for x in nodes:
            assert same(x.theta, star)
    assert same(P.gossip_stale_step(P.make_node(0, star), star, obj, z, h).theta, star)
    assert same(P.gossip_fresh_step(P.make_node(0, star), star, obj, z, h).theta, star)
    node, upd = P.ea_client_step(P.make_node(0, star), star, obj, z, h)
    assert same(node.theta, star) and same(upd, np.zeros(2))


def test_spatial_mean_exact_on_identical_inputs():
    for v in (0.1, 1.0 / 3.0, 2.2250738585072014e-308, 12345.6789):
        m = P.spatial_mean([np.array([v, -v])] * 3)
        assert m[0] == v and m[1] == -v


# --------------------------------------------------- whole trajectories
def to_driver(cfg: O.SimConfig) -> D.SimConfig:
    names = {O.ALLREDUCE: "all-reduce", O.ELASTIC: "elastic-avg", O.PULL: "pull-gossip",
             O.PUSH: "push-gossip", O.STALE: "gossip-stale", O.FRESH: "gossip-fresh",
             O.ASYNC_PULL: "async-pull"}
    kinds = {O.INIT_ZEROS: "zeros", O.INIT_OFFSET_ONES: "offset-ones",
             O.INIT_GAUSSIAN: "gaussian-spread", O.INIT_EXPLICIT: "explicit"}
    hp = cfg.hyper
    h = Hyperparams(alpha0=hp.alpha0, anneal_factor=hp.anneal_factor, anneal_at=tuple(hp.anneal_at),
                    mu=hp.mu, weight_decay=hp.weight_decay, beta_gossip=hp.beta_gossip,
                    beta_ea=hp.beta_ea, tau=hp.tau)
    noise = None if cfg.sigma is None else P.NoiseModel.gaussian_per_coord(cfg.sigma, cfg.d)
    return D.SimConfig(protocol=names[cfg.protocol], p=cfg.p, hyper=h, noise=noise,
                       init=D.InitSpec(kinds[cfg.init_kind], cfg.target_sq_err, cfg.init_scale,
                                       cfg.init_values),
                       momentum_scope="per-node" if cfg.per_node_scope else "aggregate",
                       rounds=cfg.rounds, events=cfg.events, rate_per_node=cfg.rate_per_node,
                       seed=cfg.seed, run_id=cfg.run_id)


def run_device(cfg: O.SimConfig, dtype: str):
    obj = P.QuadraticObjective(cfg.spectrum, cfg.opt)
    dc = to_driver(cfg)
    if cfg.protocol == O.ASYNC_PULL:
        return D.run_async_pull(dc, obj, dtype=dtype)
    return D.run_sync(dc, obj, dtype=dtype)


def golden_cases():
    from tests.golden.make_golden import RUN_CASES
    return {k: v for k, v in RUN_CASES.items() if not v.poisson}


@pytest.mark.parametrize("name", sorted(golden_cases()))
def test_trajectory_fp64_matches_golden_reference(name):
    """Whole run_sync / run_async trajectories (incl. the C1 config: 2000
    rounds, p=2, reference quadratic, noise) bit-exact with the compiled
    reference's output committed in tests/golden/runs.npz."""
    cfg = golden_cases()[name]
    g = np.load("tests/golden/runs.npz")
    r = run_device(cfg, "f64")
    assert same(r.theta, g[f"{name}_theta"])
    assert same(r.delta_prev, g[f"{name}_dprev"])
    assert r.t.tolist() == g[f"{name}_t"].tolist()
    if cfg.protocol == O.ELASTIC:
        assert same(r.center, g[f"{name}_center"])


@pytest.mark.parametrize("name", sorted(golden_cases()))
def test_trajectory_fp32_matches_fp32_restatement(name):
    cfg = golden_cases()[name]
    r = run_device(cfg, "f32")
    th, dp, t, c = O.run(cfg, dtype=np.float32)
    assert same(r.theta.astype(np.float32), th)
    assert same(r.delta_prev.astype(np.float32), dp)


def test_fp32_teacher_forced_within_1e5_of_fp64():
    """C1 (SPEC reference quadratic, all-reduce, p=2): each fp32 GPU step
    from the fp64 oracle state lands within 1e-5 max relative error
    (norm-wise, denominator clamped at 1e-3*||theta_0||) of the fp64 step."""
    spec, d, p = [1.0, 2.0, 5.0, 10.0], 4, 2
    hk = dict(alpha0=0.05, anneal_at=(), mu=0.9, weight_decay=1e-4)
    h, hc = Hyperparams(**hk), O.HyperParams(**hk)
    sigma = float(np.sqrt(0.01 / 4))
    n = O.Nodes(np.full((p, d), np.sqrt(8.0 / (p * d))))
    streams = [O.Stream.make(1, "c1/trial0", i, "gradient-noise") for i in range(p)]
    g = Group(d, p, dtype="f32", quadratic=True, noise=True)
    g.set_quadratic(spec)
    floor = 1e-3 * np.linalg.norm(n.theta)
    worst = 0.0
    for r in range(300):
        noise = np.array([[sigma * s.normal() for _ in range(d)] for s in streams])
        for i in range(p):
            g.set_state(i, n.theta[i].astype(np.float32).astype(np.float64),
                        n.dprev[i].astype(np.float32).astype(np.float64), int(n.t[i]))
            g.set_vector(i, N.BUF_NOISE, noise[i].astype(np.float32).astype(np.float64))
        g.allreduce_round(h, grad="quadratic", noise=True)
        O.allreduce_round(n, hc, spec=spec, noise=noise)
        th = np.array([g.get_state(i)[0] for i in range(p)])
        err = np.abs(th - n.theta).max() / max(np.abs(n.theta).max(), floor)
        worst = max(worst, err)
    assert worst <= 1e-5, worst
    g.close()


# ---------------------------------------------------------- SURVEY §8(f)
def test_async_elastic_fp64_matches_golden_reference():
    """F4: asynchronous EASGD under the Poisson clock (run_async
    simulator.cpp:380-449), one fused client-event kernel per tick,
    bit-exact with the compiled reference (golden ea8_poisson)."""
    from tests.golden.make_golden import RUN_CASES
    cfg = RUN_CASES["ea8_poisson"]
    g = np.load("tests/golden/runs.npz")
    obj = P.QuadraticObjective(cfg.spectrum, cfg.opt)
    r = D.run_async_elastic(to_driver(cfg), obj, dtype="f64")
    assert same(r.theta, g["ea8_poisson_theta"])
    assert same(r.delta_prev, g["ea8_poisson_dprev"])
    assert r.t.tolist() == g["ea8_poisson_t"].tolist()
    assert same(r.center, g["ea8_poisson_center"])
    r32 = D.run_async_elastic(to_driver(cfg), obj, dtype="f32")
    th, dp, t, c = O.run(cfg, dtype=np.float32)
    assert same(r32.theta.astype(np.float32), th) and same(r32.center.astype(np.float32), c)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_trace_metrics_match_oracle(dtype):
    """F3: make_trace_record on the device (fp64 accumulation; the summation
    order differs from the reference's, so relative 1e-12)."""
    p, d = 5, 3001
    c = make_case(p, d, dtype, seed=21)
    g = load_group(c, dtype)
    tr = g.trace()
    ref = O.trace(c["theta"], c["spec"], c["opt"])
    for k in ("sq_err_consensus", "loss_mean", "sq_err_opt"):
        assert tr[k] == pytest.approx(ref[k], rel=1e-12), k
    th = c["theta"].astype(np.float64).copy()
    th[2, 17] = np.nan
    g.set_state(2, th[2])
    with pytest.raises(N.DsgdError, match="non-finite"):
        g.trace()
    g.close()


def _device_noise(d, sigma, seed, t, grad_ptrs=None):
    """Extract the in-kernel noise: alpha = 1, mu = wd = 0, zero gradient
    -> delta' = -xi."""
    g = Group(d, 1, dtype="f32", grad=True)
    g.set_state(0, np.zeros(d), np.zeros(d), t)
    h = Hyperparams(alpha0=1.0, anneal_at=(), mu=0.0, weight_decay=0.0)
    g.local_sgd_step(h, grad=grad_ptrs or "buffer", noise=("device", sigma, seed))
    xi = -g.get_state(0)[1]
    g.close()
    return xi


def test_device_noise_statistics_and_determinism():
    """F1: Philox noise inside the fused kernel: N(0, sigma^2), a function of
    (seed, node, t, k) only -- identical on the vector and scalar paths."""
    import torch
    d, sigma = 1_000_003, 0.3
    a = _device_noise(d, sigma, 7, 5)
    b = _device_noise(d, sigma, 7, 5)
    assert same(a, b)
    assert abs(a.mean()) < 5 * sigma / np.sqrt(d)
    assert a.std() == pytest.approx(sigma, rel=5e-3)
    c = _device_noise(d, sigma, 7, 6)
    assert abs(np.corrcoef(a, c)[0, 1]) < 0.01
    z = torch.zeros(d + 8, device="cuda")  # misaligned zero gradient -> scalar path
    torch.cuda.synchronize()
    s = _device_noise(d, sigma, 7, 5, grad_ptrs=[z.data_ptr() + 4])
    assert same(s, a)


# ------------------------------------------- the headline kernel (N = 1)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("d,fixed,noise,mu,wd,scope", [
    (5000, True, False, 0.9, 1e-4, "aggregate"),    # 2 full fp32 tiles + ragged tail
    (2048 * 7 + 3, False, True, 0.9, 1e-3, "per-node"),
    (4096, True, True, 0.0, 0.0, "aggregate"),       # exact tiles, no tail
    (1_000_003, True, True, 0.9, 1e-4, "aggregate"),
])
def test_single_node_allreduce_staged_kernel_bit_exact(dtype, d, fixed, noise, mu, wd, scope):
    """p = 1 all-reduce rounds run k_local_tma (every input stream staged
    through smem by cp.async.bulk); bit-exact with the oracle over 3 rounds."""
    c = make_case(1, d, dtype, seed=d, fixed=fixed, noise=noise)
    g = load_group(c, dtype)
    n = oracle_nodes(c)
    hk = H(mu=mu, weight_decay=wd)
    h, hc = Hyperparams(**hk), O.HyperParams(**hk)
    for _ in range(3):
        g.allreduce_round(h, scope=scope, grad="buffer" if fixed else "quadratic", noise=noise)
        O.allreduce_round(n, hc, per_node=scope == "per-node", **okw(c))
    th, dp, t = read_group(g, 1, dtype)
    assert same(th, n.theta) and same(dp, n.dprev) and t.tolist() == n.t.tolist()
    g.close()


def test_device_noise_same_on_ldg_and_staged_kernels():
    """In-kernel Philox noise depends only on (seed, node, t, k): the LDG
    local-step kernel and the staged p = 1 all-reduce kernel draw the same."""
    d = 300_001
    rng = np.random.default_rng(4)
    theta = rng.normal(size=d)
    hk = dict(alpha0=0.1, anneal_at=(), mu=0.5, weight_decay=0.0)
    out = []
    for kind in ("local", "allreduce"):
        g = Group(d, 1, dtype="f32", quadratic=True)
        g.set_quadratic(np.ones(d), np.zeros(d))
        g.set_state(0, theta, np.zeros(d), 4)
        fn = g.local_sgd_step if kind == "local" else g.allreduce_round
        fn(Hyperparams(**hk), grad="quadratic", noise=("device", 0.2, 99))
        out.append(g.get_state(0)[0])
        g.close()
    assert same(out[0], out[1])


@pytest.mark.parametrize("p", [16, 32])
@pytest.mark.parametrize("rule", ["allreduce", "ea", "pull", "push"])
def test_many_nodes_one_gpu_bit_exact(p, rule):
    """Up to DSGD_MAX_LOCAL_NODES = 32 workers in one context."""
    d = 777
    c = make_case(p, d, "f64", seed=p, fixed=True, noise=True)
    rng = np.random.default_rng(p)
    partner = rng.integers(0, p, size=p).astype(np.uint32)
    target = np.array([(i + 1 + int(rng.integers(0, p - 1))) % p for i in range(p)], dtype=np.uint32)
    g = load_group(c, "f64")
    n = oracle_nodes(c)
    center = run_rule(rule, g, n, c, H(), partner, target)
    th, dp, t = read_group(g, p, "f64")
    assert same(th, n.theta) and same(dp, n.dprev)
    if rule == "ea":
        assert same(g.get_center(), center)
    g.close()


def test_device_tracer_records_launches():
    """DSGD_TRACE: every traced launch stamps entry <= after-wait <= done."""
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "from paper_1611_04581_b200.engine import Group, Hyperparams\n"
        "g = Group(100_000, 2, quadratic=True)\n"
        "g.set_quadratic(np.ones(100_000))\n"
        "h = Hyperparams(alpha0=0.1, anneal_at=())\n"
        "for _ in range(3): g.pull_gossip_round(h, [1, 0], grad='quadratic')\n"
        "tr = g.trace_dump()\n"
        "assert tr.shape == (3, 5), tr.shape\n"
        "assert (tr[:, 2] <= tr[:, 3]).all() and (tr[:, 3] <= tr[:, 4]).all() and (tr[:, 4] > 0).all()\n"
        "assert tr[:, 1].tolist() == [0, 1, 2]\n"
        "print('ok')\n")
    env = dict(__import__("os").environ, DSGD_TRACE="64")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=120, cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr


@pytest.mark.parametrize("name", ["c1_allreduce", "pull8", "push5", "ea8", "stale4", "fresh4",
                                  "async8", "ea8_poisson"])
def test_trace_records_match_reference(name):
    """F3: run_sync / run_async trace records (make_trace_record every
    trace_every rounds/events, simulator.cpp:356-361 / 431-434) against the
    compiled reference's: t, sim_time and alpha exact; the metrics are fp64
    reductions in another order (relative 1e-11)."""
    from tests.golden.make_golden import RUN_CASES, TRACE_CASES
    cfg = RUN_CASES[name]
    gold = np.load("tests/golden/traces.npz")[f"{name}_rec"]
    obj = P.QuadraticObjective(cfg.spectrum, cfg.opt)
    dc = to_driver(cfg)
    dc.trace_every = TRACE_CASES[name]
    if cfg.protocol == O.ASYNC_PULL:
        r = D.run_async_pull(dc, obj, dtype="f64")
    elif cfg.poisson:
        r = D.run_async_elastic(dc, obj, dtype="f64")
    else:
        r = D.run_sync(dc, obj, dtype="f64")
    assert len(r.trace) == len(gold)
    for rec, g in zip(r.trace, gold):
        assert rec.t == int(g[0])
        assert rec.sim_time == g[1]
        assert rec.alpha == g[5]
        assert rec.sq_err_opt == pytest.approx(g[2], rel=1e-11, abs=1e-300)
        assert rec.sq_err_consensus == pytest.approx(g[3], rel=1e-11, abs=1e-300)
        assert rec.loss_mean == pytest.approx(g[4], rel=1e-11, abs=1e-300)
        assert rec.protocol == dc.protocol and rec.run_id == cfg.run_id
