"""Pins the CPU oracle (oracle/dsgd_oracle.c) before it is trusted as the
checker: against the reference tests' own hand values
(proj/tests/test_protocols.cpp, test_core.cpp, acceptance_main.cpp C6/C7),
the survey KATs, the committed golden fixtures (tests/golden/, made from the
compiled reference by tests/golden/make_golden.py) and -- where this
container has /root/reference -- the compiled reference itself
(oracle/_ref), bit for bit in fp64."""
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
quad1 = dict(spec=[1.0], opt=[0.0])  # scalar_quadratic() test_protocols.cpp:38-40


def one(theta, dtype=np.float64, t=0):
    return O.Nodes([theta] if np.ndim(theta) == 1 else [[theta]], dtype=dtype, t=[t])


# ---------------------------------------------------------------- KATs
def test_stream_seed_kats():
    # SURVEY.md §8(c) KATs measured from the compiled reference
    assert O.derive_stream_seed(1, "run", 0, "partner-choice") == 0x3636A58102FD6E9E
    assert O.derive_stream_seed(1, "run", 0xFFFFFFFF, "clock") == 0x618266BF79EAA43B


def test_pull_partner_schedule_kat():
    sched = O.pull_schedule(1, "run/trial0", 8, 1, 5)
    assert (sched[0] == 0xFFFFFFFF).all()  # t = 0 is never gated (simulator.cpp:25)
    assert sched[1:].tolist() == [[1, 2, 4, 3, 4, 1, 2, 7], [0, 6, 6, 0, 0, 7, 6, 4],
                                  [7, 4, 2, 6, 7, 0, 2, 5], [1, 2, 6, 4, 1, 6, 7, 3]]


def test_uniform_index_one_draws_nothing():
    # test_core.cpp:195-200
    a, b = O.Stream(99), O.Stream(99)
    assert a.uniform_index(1) == 0
    assert a.next_u64() == b.next_u64()


def test_mt19937_64_standard_value():
    # C++ standard [rand.predef]: 10000th draw of default-seeded mt19937_64
    s = O.Stream(5489)
    for _ in range(9999):
        s.next_u64()
    assert s.next_u64() == 9981545732273789042


def test_streams_purpose_separated():
    # test_core.cpp:167-193
    base = O.Stream.make(42, "run", 3, "gradient-noise")
    same = O.Stream.make(42, "run", 3, "gradient-noise")
    others = [O.Stream.make(42, "run", 3, "partner-choice"), O.Stream.make(42, "run", 4, "gradient-noise"),
              O.Stream.make(43, "run", 3, "gradient-noise"), O.Stream.make(42, "other", 3, "gradient-noise")]
    a = [base.next_u64() for _ in range(64)]
    assert a == [same.next_u64() for _ in range(64)]
    for o in others:
        assert a != [o.next_u64() for _ in range(64)]


def test_step_schedule():
    h = O.HyperParams()
    assert O.step_size_at(h, 0) == 0.1
    assert O.step_size_at(h, 149999) == 0.1
    assert O.step_size_at(h, 150000) == pytest.approx(0.01, rel=1e-15)
    assert O.step_size_at(h, 300000) == pytest.approx(0.001, rel=1e-15)


# ------------------------------------------------- hand values (protocols)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_local_step_hand_values(dtype):
    tol = 1e-15 if dtype == np.float64 else 1e-6
    n = O.local_sgd_step(one(2.0, dtype), O.plain(0.1), **quad1)  # test_protocols.cpp:94-103
    assert n.theta[0, 0] == pytest.approx(1.8, rel=tol) and n.t[0] == 1
    assert n.dprev[0, 0] == pytest.approx(-0.2, rel=tol)
    n = O.local_sgd_step(one(2.0, dtype), O.plain(0.0), **quad1)  # 105-111
    assert n.theta[0, 0] == 2.0
    n = one(1.0, dtype)  # two Nesterov steps 113-125
    O.local_sgd_step(n, O.plain(0.1, 0.9), **quad1)
    assert n.theta[0, 0] == pytest.approx(0.9, rel=tol)
    O.local_sgd_step(n, O.plain(0.1, 0.9), **quad1)
    assert n.theta[0, 0] == pytest.approx(0.729, rel=10 * tol)
    h = O.plain(0.1)
    h.weight_decay = 0.5  # 136-144
    n = O.local_sgd_step(one(2.0, dtype), h, **quad1)
    assert n.theta[0, 0] == pytest.approx(1.7, rel=tol)


def test_allreduce_hand_values_and_exactness():
    n = O.allreduce_round(O.Nodes([[4.0], [4.0]]), O.plain(0.1), **quad1)  # 146-155
    assert n.theta[:, 0] == pytest.approx([3.6, 3.6], rel=1e-15)
    # p = 1 all-reduce == local step, bit-exact (157-172)
    seq, par = one(2.0), one(2.0)
    for _ in range(5):
        O.local_sgd_step(seq, O.plain(0.1, 0.9), **quad1)
        O.allreduce_round(par, O.plain(0.1, 0.9), **quad1)
    assert par.theta.tobytes() == seq.theta.tobytes()
    assert par.dprev.tobytes() == seq.dprev.tobytes()
    # exact spatial mean on identical inputs (test_core.cpp:106-114)
    for v in (0.1, 1.0 / 3.0, 2.2250738585072014e-308, 12345.6789):
        m = O.spatial_mean(np.array([[v, -v]] * 3))
        assert m[0] == v and m[1] == -v


def test_allreduce_equal_starts_stay_equal_under_noise():
    # test_protocols.cpp:174-187
    spec, opt = [1.0, 10.0], [0.0, 0.0]
    n = O.Nodes([[1.0, -1.0]] * 4)
    streams = [O.Stream.make(1, "test", i, "gradient-noise") for i in range(4)]
    for _ in range(10):
        noise = np.array([[0.3 * s.normal() for _ in range(2)] for s in streams])
        O.allreduce_round(n, O.plain(0.05), spec=spec, opt=opt, noise=noise)
        for i in range(1, 4):
            assert n.theta[i].tobytes() == n.theta[0].tobytes()


def test_ea_hand_values():
    h = O.plain(0.0)
    h.beta_ea = 0.1  # test_protocols.cpp:249-260
    n, c = one(1.0), np.zeros(1)
    O.ea_round(n, c, True, h, **quad1)
    assert c[0] == pytest.approx(0.1, rel=1e-15)
    assert n.theta[0, 0] == pytest.approx(0.9, rel=1e-15) and n.t[0] == 1
    h.beta_ea = 0.25  # 262-270
    n, c = one(0.7), np.array([0.7])
    O.ea_round(n, c, True, h, **quad1)
    assert c[0] == 0.7 and n.theta[0, 0] == 0.7


def test_pull_push_hand_values():
    assert O.pull_mix(np.array([[1.0], [3.0]]), [1, 0])[:, 0].tolist() == [2.0, 2.0]
    x = np.array([[1.0, 2.0], [-3.0, 4.0]])
    assert O.pull_mix(x, [0, 1]).tobytes() == x.tobytes()  # self-pull identity (297-307)
    n = O.pull_gossip_round(O.Nodes([[1.0], [3.0]]), [1, 0], O.plain(0.1), **quad1)
    assert n.theta[:, 0] == pytest.approx([1.8, 1.8], rel=1e-15)  # 316-328
    out = O.push_mix(np.array([[0.0], [3.0], [6.0]]), [1, 2, 0])  # 342-354
    assert out[:, 0] == pytest.approx([3.0, 1.5, 4.5], rel=1e-15)
    out = O.push_mix(np.array([[0.5], [3.0], [6.0]]), [1, 2, 1])  # 356-367
    assert out[0, 0] == 0.5 and out[1, 0] == pytest.approx((3.0 + 0.5 + 6.0) / 3.0)
    with pytest.raises(ValueError):
        O.push_mix(np.array([[1.0], [2.0]]), [0, 0])


def test_stale_fresh_async_hand_values():
    h = O.plain(0.1)
    h.beta_gossip = 0.5
    # stale: node 0 at 2 with partner value 0 -> 0.8 (402-412)
    n = O.Nodes([[2.0], [0.0]])
    O.stale_round(n, [1, 1], h, **quad1)
    assert n.theta[0, 0] == pytest.approx(0.8, rel=1e-15)
    # fresh: own step 2 -> 1.8, partner post-step 0 (at optimum) -> 0.9 (434-442)
    n = O.Nodes([[2.0], [0.0]])
    O.fresh_round(n, [1, 1], h, **quad1)
    assert n.theta[0, 0] == pytest.approx(0.9, rel=1e-15)
    # async (481-517)
    h0 = O.plain(0.0)
    h0.beta_gossip = 0.5
    n = O.async_pull_event(O.Nodes([[2.0], [0.0]]), 0, 1, h0, **quad1)
    assert n.theta[:, 0].tolist() == [pytest.approx(1.0, rel=1e-15), 0.0]
    assert n.t.tolist() == [1, 0]
    h1 = O.plain(0.1)
    h1.beta_gossip = 0.0
    n = O.async_pull_event(O.Nodes([[2.0], [5.0]]), 0, 1, h1, **quad1)
    assert n.theta[0, 0] == pytest.approx(1.8, rel=1e-15)
    n = O.async_pull_event(O.Nodes([[2.0]]), 0, 0, h, **quad1)
    assert n.theta[0, 0] == pytest.approx(1.9, rel=1e-15)
    h2 = O.plain(0.1)
    h2.anneal_at, h2.anneal_factor, h2.beta_gossip = (5,), 0.1, 0.0  # 519-531
    n = O.async_pull_event(O.Nodes([[2.0], [2.0]], t=[5, 0]), 0, 1, h2, **quad1)
    assert n.theta[0, 0] == pytest.approx(2.0 - 0.01 * 2.0, rel=1e-15)


def test_consensus_at_optimum_invariant_every_protocol():
    # test_protocols.cpp:533-563
    spec, opt = [1.0, 3.0], [0.5, -0.5]
    h = O.plain(0.1, 0.9)
    h.beta_gossip, h.beta_ea = 0.5, 0.1
    star = np.array(opt)
    mk = lambda: O.Nodes([opt] * 3)  # noqa: E731
    outs = [O.allreduce_round(mk(), h, spec=spec, opt=opt),
            O.pull_gossip_round(mk(), [1, 2, 0], h, spec=spec, opt=opt),
            O.push_gossip_round(mk(), [1, 2, 0], h, spec=spec, opt=opt),
            O.async_pull_event(mk(), 0, 2, h, spec=spec, opt=opt),
            O.stale_round(mk(), [1, 2, 0], h, spec=spec, opt=opt),
            O.fresh_round(mk(), [1, 2, 0], h, spec=spec, opt=opt)]
    c = star.copy()
    outs.append(O.ea_round(mk(), c, True, h, spec=spec, opt=opt))
    for n in outs:
        for i in range(3):
            assert n.theta[i].tobytes() == star.tobytes()
    assert c.tobytes() == star.tobytes()


# ----------------------------------------------- acceptance C6 / C7 shapes
def test_c6_degenerations_bit_exact():
    """acceptance_main.cpp:377-498 (a): p = 1, every sync protocol == the
    sequential SGD chain, momentum/wd/annealing/noise included."""
    base = O.SimConfig(p=1, hyper=O.HyperParams(alpha0=0.1, anneal_at=(20,), mu=0.9,
                                                weight_decay=1e-4, beta_ea=0.0),
                       sigma=float(np.sqrt(0.02 / 4)), init_kind=O.INIT_EXPLICIT,
                       init_values=[1.0, -1.0, 0.5, 2.0], rounds=40, run_id="c6a")
    chain = O.Nodes([base.init_values])
    s = O.Stream.make(1, "c6a", 0, "gradient-noise")
    for _ in range(40):
        O.local_sgd_step(chain, base.hyper, spec=base.spectrum,
                         noise=[[base.sigma * s.normal() for _ in range(4)]])
    for proto in (O.PULL, O.PUSH, O.STALE, O.FRESH, O.ELASTIC):
        base.protocol = proto
        th, _, _, _ = O.run(base)
        assert th.tobytes() == chain.theta.tobytes(), proto


def test_c7_ring_exactness():
    """acceptance_main.cpp:503-540: p = 8, d = 4096, inputs N(0,1) from
    RngStream(1000 + r); ring within 1e-12*p of the direct mean, identical on
    every node."""
    p, d = 8, 4096
    x = np.array([O.Stream(1000 + r).normals(d) for r in range(p)])
    out = O.ring_allreduce(x)
    assert all(out[r].tobytes() == out[0].tobytes() for r in range(p))
    direct = x.sum(axis=0) / p
    assert np.abs(out[0] - direct).max() <= 1e-12 * p


# ------------------------------------------ committed golden fixtures
def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} missing (run tests/golden/make_golden.py)")
    return np.load(path, allow_pickle=False)


def test_golden_streams():
    g = _golden("streams.npz")
    s = O.Stream(int(g["seed"]))
    assert [s.next_u64() for _ in range(len(g["u64"]))] == g["u64"].tolist()
    s = O.Stream(int(g["seed"]))
    assert np.array([s.normal() for _ in range(len(g["normal"]))]).tobytes() == g["normal"].tobytes()
    s = O.Stream(int(g["seed"]))
    assert [s.uniform_index(int(g["n"])) for _ in range(len(g["index"]))] == g["index"].tolist()


def test_golden_runs():
    from tests.golden.make_golden import RUN_CASES
    g = _golden("runs.npz")
    for name, cfg in RUN_CASES.items():
        th, dp, t, c = O.run(cfg)
        assert th.tobytes() == g[f"{name}_theta"].tobytes(), name
        assert dp.tobytes() == g[f"{name}_dprev"].tobytes(), name
        assert t.tolist() == g[f"{name}_t"].tolist(), name
        if cfg.protocol == O.ELASTIC:
            assert c.tobytes() == g[f"{name}_center"].tobytes(), name


def test_golden_ring():
    g = _golden("ring.npz")
    for key in [k for k in g.files if k.startswith("in_")]:
        out = O.ring_allreduce(g[key])
        assert out.tobytes() == g["out_" + key[3:]].tobytes(), key


# ------------------------------------ live reference (this container only)
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_ref_streams_bit_exact():
    for seed in (0, 1, 99, 2**63 + 5):
        s = O.Stream(seed)
        assert O.ref_stream(seed, 0, 700).tolist() == [s.next_u64() for _ in range(700)]
        s = O.Stream(seed)
        assert O.ref_stream(seed, 2, 300).tobytes() == np.array([s.normal() for _ in range(300)]).tobytes()
        for n in (1, 2, 3, 7, 8, 1000, 2**31 + 11):
            s = O.Stream(seed)
            assert O.ref_stream(seed, 3, 200, n).tolist() == [s.uniform_index(n) for _ in range(200)]
        s = O.Stream(seed)
        assert O.ref_stream(seed, 4, 100, 3).tobytes() == np.array([s.exponential(3.0) for _ in range(100)]).tobytes()
    for node in (0, 1, 7, 0xFFFFFFFF):
        for purpose, pid in O.PURPOSE.items():
            assert O.ref().ref_derive_stream_seed(7, b"x/trial3", node, pid) == \
                O.derive_stream_seed(7, "x/trial3", node, purpose)


def _rand_cases():
    rng = np.random.default_rng(0)
    cases = []
    for proto in (O.ALLREDUCE, O.ELASTIC, O.PULL, O.PUSH, O.STALE, O.FRESH, O.ASYNC_PULL):
        for k in range(3):
            p = int(rng.integers(1, 7))
            d = int(rng.integers(1, 9))
            h = O.HyperParams(alpha0=float(rng.uniform(0.01, 0.2)), anneal_at=(7, 15),
                              anneal_factor=0.5, mu=[0.0, 0.9, 0.5][k],
                              weight_decay=[0.0, 1e-4, 0.01][k], beta_gossip=0.3,
                              beta_ea=float(rng.uniform(0.05, 0.5)), tau=[1, 2, 3][k])
            cfg = O.SimConfig(protocol=proto, p=p, hyper=h,
                              sigma=[None, 0.1, 0.0][k],
                              spectrum=list(rng.uniform(0.5, 3.0, d)),
                              opt=list(rng.normal(size=d)),
                              init_kind=[O.INIT_GAUSSIAN, O.INIT_OFFSET_ONES, O.INIT_GAUSSIAN][k],
                              per_node_scope=bool(k % 2), poisson=(proto == O.ELASTIC and k == 2),
                              rounds=25, events=60, seed=int(rng.integers(1, 100)),
                              run_id=f"case{proto}/trial{k}")
            cases.append(cfg)
    return cases


@needs_ref
@pytest.mark.parametrize("cfg", _rand_cases(), ids=lambda c: f"proto{c.protocol}-p{c.p}-{c.run_id}")
def test_ref_runs_bit_exact(cfg):
    if cfg.protocol == O.PUSH and cfg.p == 1:
        cfg.p = 2
    a = O.run(cfg)
    b = O.ref_run(cfg)
    n = 4 if cfg.protocol == O.ELASTIC else 3  # the center exists for elastic-avg only
    for x, y in list(zip(a, b))[:n]:
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()


@needs_ref
@pytest.mark.parametrize("kind", ["local", "allreduce", "ea", "pull", "push", "stale", "fresh", "async"])
@pytest.mark.parametrize("fixed", [False, True])
def test_ref_round_primitives_bit_exact(kind, fixed):
    rng = np.random.default_rng(hash((kind, fixed)) % 2**32)
    p, d = 5, 33
    h = O.HyperParams(alpha0=0.07, anneal_at=(3,), mu=0.9, weight_decay=1e-3, beta_gossip=0.3,
                      beta_ea=0.2)
    theta, dprev = rng.normal(size=(p, d)), rng.normal(size=(p, d)) * 0.1
    t = np.full(p, 3 if kind != "async" else 2, dtype=np.uint64)
    if kind == "async":
        t = rng.integers(0, 6, size=p).astype(np.uint64)
    spec, opt = rng.uniform(0.5, 2, d), rng.normal(size=d)
    gfixed = rng.normal(size=(p, d)) if fixed else None
    sigma = 0.05
    partner = (rng.integers(0, p, size=p) if kind not in ("push",) else
               np.array([(i + 1 + int(rng.integers(0, p - 1))) % p for i in range(p)]))
    noise = np.array([O.noise_for_step(11, "prim", i, sigma, d) for i in range(p)])
    center = rng.normal(size=d)
    a = O.Nodes(theta, dprev, t)
    b = O.Nodes(theta, dprev, t)
    ca, cb = center.copy(), center.copy()
    kw = dict(spec=spec, opt=opt, gfixed=gfixed, noise=noise)
    if kind == "local":
        O.local_sgd_step(a, h, **kw)
    elif kind == "allreduce":
        O.allreduce_round(a, h, per_node=True, **kw)
    elif kind == "ea":
        O.ea_round(a, ca, True, h, **kw)
    elif kind == "pull":
        O.pull_gossip_round(a, partner, h, **kw)
    elif kind == "push":
        O.push_gossip_round(a, partner, h, **kw)
    elif kind == "stale":
        O.stale_round(a, partner, h, **kw)
    elif kind == "fresh":
        O.fresh_round(a, partner, h, **kw)
    elif kind == "async":
        O.async_pull_event(a, 2, 4, h, **kw)
    O.ref_round(kind, b, h, partner=partner, spec=spec, opt=opt, gfixed=gfixed, sigma=sigma,
                seed=11, run_id="prim", per_node=True, center=cb, i=2, j=4)
    assert a.theta.tobytes() == b.theta.tobytes()
    if kind != "async":
        assert a.dprev.tobytes() == b.dprev.tobytes()
    assert a.t.tolist() == b.t.tolist()
    assert ca.tobytes() == cb.tobytes()


@needs_ref
def test_ref_ring_allreduce_bit_exact():
    rng = np.random.default_rng(3)
    for p, d in ((2, 5), (3, 7), (8, 21), (8, 4096), (5, 3)):
        x = rng.normal(size=(p, d))
        assert O.ring_allreduce(x).tobytes() == O.ref_ring_allreduce(x, chaos_seed=p).tobytes()


@needs_ref
def test_ref_transport_allreduce_matches_ring_restatement():
    """run_transport all-reduce uses ring_allreduce: its final theta equals a
    restated loop of (local delta -> ring mean -> theta += avg)."""
    cfg = O.SimConfig(protocol=O.ALLREDUCE, p=4, hyper=O.HyperParams(alpha0=0.05, mu=0.9),
                      sigma=0.05, rounds=12, per_node_scope=False, run_id="tr")
    th_ref, dp_ref, _, _ = O.ref_run(cfg, transport=True)
    p, d = cfg.p, cfg.d
    n = O.Nodes(np.tile(np.array(cfg.spectrum) * 0 + np.sqrt(8.0 / (p * d)), (p, 1)))
    streams = [O.Stream.make(1, "tr", i, "gradient-noise") for i in range(p)]
    for r in range(cfg.rounds):
        noise = np.array([[cfg.sigma * s.normal() for _ in range(d)] for s in streams])
        deltas = np.zeros((p, d))
        for i in range(p):
            m = O.Nodes(n.theta[i:i + 1], n.dprev[i:i + 1], n.t[i:i + 1])
            O.local_sgd_step(m, cfg.hyper, spec=cfg.spectrum, noise=noise[i:i + 1])
            deltas[i] = m.dprev[0]
        avg = O.ring_allreduce(deltas)
        n.theta = n.theta + avg
        n.dprev = avg.copy()
        n.t += 1
    assert n.theta.tobytes() == th_ref.tobytes()


def test_golden_transport_allreduce_restatement():
    """The restated run_transport all-reduce loop equals the compiled
    reference's threaded transport (fixture) bit for bit, p = 2, 4, 8."""
    from tests.golden.make_golden import transport_case
    g = _golden("transport.npz")
    for p in (2, 4, 8):
        n = O.run_transport_allreduce(transport_case(p))
        assert n.theta.tobytes() == g[f"p{p}_theta"].tobytes()
        assert n.dprev.tobytes() == g[f"p{p}_dprev"].tobytes()


# ------------------------------------------ LogisticObjective (F1)
def test_golden_logistic_gradient_kats():
    """The restated stochastic_gradient (rows from the node's sample stream,
    objectives.cpp:147-162) equals the compiled reference's bit for bit."""
    g = _golden("logistic.npz")
    X, y, l2 = g["X"], g["y"], float(g["l2"])
    for k in range(3):
        batch, b, e, seed = (int(v) for v in g[f"kat{k}_meta"])
        rows = O.Stream(seed).draw_rows(b, e, batch)
        assert all(b <= r < e for r in rows)
        got = O.logistic_grad(X, y, l2, g[f"kat{k}_theta"], rows)
        assert got.tobytes() == g[f"kat{k}_grad"].tobytes(), k


def test_logistic_tiny_hand_values():
    """test_objectives.cpp tiny_logistic: at theta = 0 every z = 0, so
    sigmoid = 1/2 and the single-row gradient is (1/2 - y) x + l2 * 0."""
    X = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [-1.0, 0.5]])
    y = np.array([1, 0, 1, 0], dtype=np.int32)
    assert O.sigmoid(0.0) == 0.5
    for r in range(4):
        g = O.logistic_grad(X, y, 0.1, np.zeros(2), [r])
        assert g.tolist() == ((0.5 - y[r]) * X[r]).tolist()
    # batch mean then l2 * theta, in that order
    th = np.array([0.3, -0.2])
    g = O.logistic_grad(X, y, 0.1, th, [0, 3, 3])
    acc = np.zeros(2)
    for r in (0, 3, 3):
        acc = acc + (O.sigmoid(float(X[r] @ th)) - y[r]) * X[r]
    assert np.allclose(g, acc * (1.0 / 3) + 0.1 * th, rtol=0, atol=1e-15)


def test_logistic_fp32_policy_close_to_fp64():
    g = _golden("logistic.npz")
    X, y, l2 = g["X"], g["y"], float(g["l2"])
    th = g["kat2_theta"]
    rows = np.arange(0, 48, 5)
    g64 = O.logistic_grad(X, y, l2, th, rows)
    g32 = O.logistic_grad(X.astype(np.float32), y, l2, th.astype(np.float32), rows)
    assert np.abs(g32 - g64).max() <= 1e-6 * np.abs(g64).max()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ref_logistic_gradient_random_bit_exact():
    rng = np.random.default_rng(3)
    for n, d, batch in ((5, 3, 1), (17, 64, 4), (40, 129, 9)):
        X = rng.standard_normal((n, d))
        y = rng.integers(0, 2, n).astype(np.int32)
        O.ref_set_logistic(X, y, 0.01)
        th = rng.standard_normal(d)
        seed = O.derive_stream_seed(9, "lg", n, "sample")
        want = O.ref_logistic_grad(th, batch, seed, 1, n)
        got = O.logistic_grad(X, y, 0.01, th, O.Stream(seed).draw_rows(1, n, batch))
        assert got.tobytes() == want.tobytes()
    O.ref_set_logistic(None, None, 0.0)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ref_logistic_constructor_errors():
    with pytest.raises(ValueError, match="l2 must be positive"):
        O.ref_set_logistic(np.ones((2, 2)), [0, 1], 0.0)
    with pytest.raises(ValueError, match="labels must be 0 or 1"):
        O.ref_set_logistic(np.ones((2, 2)), [0, 2], 0.1)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ref_logistic_value_bit_exact():
    rng = np.random.default_rng(12)
    X = rng.standard_normal((30, 17)) * 3
    y = rng.integers(0, 2, 30).astype(np.int32)
    O.ref_set_logistic(X, y, 0.2)
    for _ in range(3):
        th = rng.standard_normal(17) * 4
        assert O.logistic_value(X, y, 0.2, th) == O.ref_logistic_value(th)
    O.ref_set_logistic(None, None, 0.0)


def test_golden_trace_jsonl_schema_round_trips():
    """trace_record_to_json_line / _from_json_line (trace_io.cpp:40-77):
    the driver's TraceRecord re-emits the reference's own JSONL lines byte
    for byte (sorted keys, compact, shortest round-trip doubles, null for an
    absent sim_time / sq_err_opt)."""
    from paper_1611_04581_b200.driver import TraceRecord
    g = _golden("traces.npz")
    n = 0
    for key in [k for k in g.files if k.endswith("_jsonl")]:
        text = str(g[key])
        if not text:
            pytest.skip("fixture made without trace_io")
        for line in text.splitlines():
            assert TraceRecord.from_json_line(line).to_json_line() == line
            n += 1
    assert n > 50
    with pytest.raises(RuntimeError, match="not valid JSON"):
        TraceRecord.from_json_line("{")
    with pytest.raises(RuntimeError, match="unknown protocol name"):
        TraceRecord.from_json_line('{"alpha":1,"loss_mean":0,"protocol":"x","run_id":"r",'
                                   '"sim_time":null,"sq_err_consensus":0,"sq_err_opt":null,"t":0}')
    with pytest.raises(RuntimeError, match="missing or mistyped"):
        TraceRecord.from_json_line('{"alpha":1}')


def test_golden_trace_metrics_restatement():
    """make_trace_record (simulator.cpp:92-123) restated (dsgdo_trace, the
    GPU trace test's checker) on the oracle's final state equals the
    reference's last trace record for the golden runs."""
    from tests.golden.make_golden import RUN_CASES, TRACE_CASES
    g = _golden("traces.npz")
    for name in ("c1_allreduce", "pull8", "push5", "ea8", "stale4", "fresh4"):
        cfg = RUN_CASES[name]
        th, _, _, _ = O.run(cfg)
        last = g[f"{name}_rec"][-1]
        assert int(last[0]) == cfg.rounds
        opt = np.zeros(cfg.d) if cfg.opt is None else np.asarray(cfg.opt)
        m = O.trace(th, cfg.spectrum, opt)
        assert m["sq_err_opt"] == pytest.approx(last[2], rel=1e-12), name
        assert m["sq_err_consensus"] == pytest.approx(last[3], rel=1e-12, abs=1e-300), name
        assert m["loss_mean"] == pytest.approx(last[4], rel=1e-12), name


def test_golden_logistic_value_restatement():
    """LogisticObjective::value restated (the GPU logistic trace test's
    checker) on the reference's final lg_pull state equals the loss of the
    reference's last trace record of the same run."""
    from tests.golden.make_golden import LOGISTIC_CASES
    lg = _golden("logistic.npz")
    tr = _golden("traces.npz")
    th = lg["lg_pull_theta"]
    want = tr["lg_pull_rec"][-1]
    assert int(want[0]) == LOGISTIC_CASES["lg_pull"].rounds
    got = np.mean([O.logistic_value(lg["X"], lg["y"], float(lg["l2"]), th[i])
                   for i in range(th.shape[0])])
    assert got == pytest.approx(want[4], rel=1e-13)


@pytest.mark.parametrize("name", ["lg_pull", "lg_allreduce", "lg_allreduce_agg"])
def test_golden_logistic_trajectories_restated_bit_exact(name):
    """The oracle's LogisticObjective run_sync (rows from the sample streams,
    host noise, pull mix / ring-free pivot mean) reproduces the reference's
    40-round trajectories byte for byte."""
    from tests.golden.make_golden import LOGISTIC_CASES
    g = _golden("logistic.npz")
    th, dp, t = O.logistic_run(LOGISTIC_CASES[name], g["X"], g["y"], float(g["l2"]),
                               g["ranges"])
    assert th.tobytes() == g[f"{name}_theta"].tobytes()
    assert dp.tobytes() == g[f"{name}_dprev"].tobytes()
    assert t.tolist() == g[f"{name}_t"].tolist()
