"""GPU parity of the logistic gradient source (the device
LogisticObjective::stochastic_gradient, objectives.cpp:147-162) against the
oracle restatement (pinned bit-exactly to the compiled reference by
tests/test_oracle_golden.py) and the reference's own trajectories committed
in tests/golden/logistic.npz.

Tolerance: the minibatch dot product z = x . theta is a tree sum over the
device (the reference sums k sequentially), so z -- and only z -- agrees to
rounding, not bitwise.  Everything after z runs in the reference order.
fp64: 1e-12 relative (per-step), 1e-9 relative (40-round trajectories).
fp32 (fp64 z, fp32 accumulation; the oracle's fp32 policy): 1e-5 relative."""
import numpy as np
import pytest

import oracle as O
from paper_1611_04581_b200 import _native as N
from paper_1611_04581_b200 import driver as D
from paper_1611_04581_b200 import protocols as P
from paper_1611_04581_b200.engine import Group, Hyperparams

pytestmark = pytest.mark.gpu

NP = {"f64": np.float64, "f32": np.float32}
TOL = {"f64": 1e-12, "f32": 1e-5}


def close(a, b, rel):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(1.0, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) <= rel * scale


def dataset(n=40, d=1003, seed=5):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) / np.sqrt(d)
    y = (rng.standard_normal(n) > 0).astype(np.int32)
    return X, y, 0.03


def HK(**kw):
    base = dict(alpha0=0.3, anneal_at=(), mu=0.9, weight_decay=1e-3, beta_gossip=0.4,
                beta_ea=0.2, tau=1, batch=3)
    base.update(kw)
    return base


def lookahead(theta, dprev, mu, f):
    """compute_local_delta's evaluation point in the context dtype (protocols.cpp:92-93)."""
    if mu == 0.0:
        return theta.copy()
    return (theta + (f(mu) * dprev).astype(f)).astype(f)


def grads_at(points, X, y, l2, rows):
    return np.stack([O.logistic_grad(X, y, l2, points[i], rows[i]) for i in range(len(points))])


def setup(p, dtype, X, y, l2, seed=1, center=False):
    f = NP[dtype]
    rng = np.random.default_rng(seed)
    d = X.shape[1]
    theta = rng.standard_normal((p, d)).astype(f)
    dprev = (0.1 * rng.standard_normal((p, d))).astype(f)
    t = np.full(p, 2, dtype=np.uint64)
    c = rng.standard_normal(d).astype(f)
    g = Group(d, p, dtype=dtype, center=center)
    g.set_logistic(X, y, l2)
    for i in range(p):
        g.set_state(i, theta[i].astype(np.float64), dprev[i].astype(np.float64), int(t[i]))
    if center:
        g.set_center(c.astype(np.float64))
    return g, theta, dprev, t, c


def read(g, p, dtype):
    f = NP[dtype]
    th, dp, t = zip(*[g.get_state(i) for i in range(p)])
    return np.array(th).astype(f), np.array(dp).astype(f), np.array(t, dtype=np.uint64)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("d", [37, 1003, 300007])
def test_logistic_gradient_buffer_matches_oracle(dtype, d):
    """The produced minibatch gradient (DSGD_BUF_GRAD after a local step)
    equals stochastic_gradient at the lookahead point."""
    f = NP[dtype]
    X, y, l2 = dataset(n=24, d=d)
    Xf = X.astype(f)
    p = 3
    g, theta, dprev, t, _ = setup(p, dtype, X, y, l2)
    h = HK(batch=4)
    rows = np.array([[0, 5, 5, 23], [7, 1, 2, 3], [11, 11, 11, 11]], dtype=np.uint64)
    g.local_sgd_step(Hyperparams(**h), grad="logistic", rows=rows)
    got = np.array([g.get_vector(i, N.BUF_GRAD) for i in range(p)]).astype(f)
    want = grads_at(lookahead(theta, dprev, h["mu"], f), Xf, y, l2, rows)
    assert close(got, want, TOL[dtype])
    g.close()


def oracle_round(kind, dtype, X, y, l2, theta, dprev, t, c, rows, hk, partner=None, i=0, j=0,
                 gated=True, per_node=False):
    """The reference rule with the logistic gradient at the rule's evaluation
    point, composed from oracle primitives (the same decomposition the
    reference performs: mix, then compute_local_delta at the mixed theta)."""
    f = NP[dtype]
    Xf = X.astype(f)
    h = O.HyperParams(**hk)
    n = O.Nodes(theta.copy(), dprev.copy(), t.copy(), dtype=f)
    center = c.copy()
    mu = hk["mu"]
    if kind in ("local", "allreduce", "stale", "fresh"):
        G = grads_at(lookahead(theta, dprev, mu, f), Xf, y, l2, rows)
        if kind == "local":
            O.local_sgd_step(n, h, gfixed=G)
        elif kind == "allreduce":
            O.allreduce_round(n, h, gfixed=G, per_node=per_node)
        elif kind == "stale":
            O.stale_round(n, partner, h, gfixed=G)
        else:
            O.fresh_round(n, partner, h, gfixed=G)
    elif kind in ("pull", "push"):
        mixed = O.pull_mix(theta, partner) if kind == "pull" else O.push_mix(theta, partner)
        G = grads_at(lookahead(mixed, dprev, mu, f), Xf, y, l2, rows)
        n = O.Nodes(mixed, dprev.copy(), t.copy(), dtype=f)
        O.local_sgd_step(n, h, gfixed=G)
    elif kind == "ea":
        moved = theta.copy()
        if gated:
            cc = c.copy()
            beta = f(hk["beta_ea"])
            for k in range(len(theta)):
                u = (beta * (moved[k] - cc).astype(f)).astype(f)
                moved[k] = (moved[k] - u).astype(f)
                cc = (cc + u).astype(f)
        G = grads_at(lookahead(moved, dprev, mu, f), Xf, y, l2, rows)
        O.ea_round(n, center, gated, h, gfixed=G)
    elif kind == "async":
        G = np.zeros_like(theta)
        G[i] = O.logistic_grad(Xf, y, l2, theta[i], rows[i])
        O.async_pull_event(n, i, j, h, gfixed=G)
    return n.theta, n.dprev, n.t, center


CASES = [("local", {}), ("allreduce", {}), ("allreduce", {"per_node": True}),
         ("pull", {"partner": [2, 0, 0, 3]}), ("push", {"partner": [1, 2, 3, 0]}),
         ("ea", {"gated": True}), ("ea", {"gated": False}),
         ("stale", {"partner": [3, 3, 1, 0]}), ("fresh", {"partner": [1, 1, 0, 2]}),
         ("async", {"i": 2, "j": 0})]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind,extra", CASES, ids=[f"{k}-{i}" for i, (k, _) in enumerate(CASES)])
def test_logistic_rules_match_oracle(kind, extra, dtype):
    X, y, l2 = dataset()
    p = 4
    g, theta, dprev, t, c = setup(p, dtype, X, y, l2, seed=3, center=True)
    hk = HK()
    h = Hyperparams(**hk)
    rows = np.random.default_rng(9).integers(0, X.shape[0], (p, hk["batch"])).astype(np.uint64)
    kw = dict(grad="logistic", rows=rows)
    if kind == "local":
        g.local_sgd_step(h, **kw)
    elif kind == "allreduce":
        g.allreduce_round(h, scope="per-node" if extra.get("per_node") else "aggregate", **kw)
    elif kind == "pull":
        g.pull_gossip_round(h, extra["partner"], **kw)
    elif kind == "push":
        g.push_gossip_round(h, extra["partner"], **kw)
    elif kind == "ea":
        g.ea_round(h, gated=extra["gated"], **kw)
    elif kind == "stale":
        g.gossip_stale_round(h, extra["partner"], **kw)
    elif kind == "fresh":
        g.gossip_fresh_round(h, extra["partner"], **kw)
    elif kind == "async":
        g.async_pull_event(h, extra["i"], extra["j"], **kw)
    th, dp, tt = read(g, p, dtype)
    want = oracle_round(kind, dtype, X, y, l2, theta, dprev, t, c, rows, hk, **extra)
    assert close(th, want[0], TOL[dtype])
    if kind != "async":
        assert close(dp, want[1], TOL[dtype])
    assert tt.tolist() == want[2].tolist()
    if kind == "ea":
        assert close(g.get_center().astype(NP[dtype]), want[3], TOL[dtype])
    g.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_logistic_ea_client_event_matches_oracle(dtype):
    """Asynchronous EASGD tick (simulator.cpp:419-428) with the logistic source."""
    X, y, l2 = dataset()
    p, i = 4, 1
    g, theta, dprev, t, c = setup(p, dtype, X, y, l2, seed=4, center=True)
    hk = HK(batch=2)
    rows = np.array([[0, 0], [3, 9], [0, 0], [0, 0]], dtype=np.uint64)
    g.ea_client_event(Hyperparams(**hk), i, True, grad="logistic", rows=rows)
    th, dp, tt = read(g, p, dtype)
    f = NP[dtype]
    # node i alone against the center: the single-client EA sweep
    want = oracle_round("ea", dtype, X, y, l2, theta[i:i + 1], dprev[i:i + 1], t[i:i + 1], c,
                        rows[i:i + 1], hk)
    assert close(th[i], want[0][0], TOL[dtype]) and close(dp[i], want[1][0], TOL[dtype])
    assert close(g.get_center().astype(f), want[3], TOL[dtype])
    others = [k for k in range(p) if k != i]
    assert np.array_equal(th[others], theta[others])
    g.close()


def golden():
    return np.load("tests/golden/logistic.npz")


def _driver_case(name):
    from tests.golden.make_golden import LOGISTIC_CASES
    from tests.test_gpu_parity import to_driver
    cfg = LOGISTIC_CASES[name]
    dc = to_driver(cfg)
    dc.hyper.batch = cfg.hyper.batch
    gd = golden()
    obj = P.LogisticObjective(gd["X"], gd["y"], float(gd["l2"]))
    shards = [obj.shard(int(b), int(e)) for b, e in gd["ranges"]]
    return cfg, dc, obj, shards


@pytest.mark.parametrize("name", ["lg_allreduce", "lg_allreduce_agg", "lg_pull", "lg_push",
                                  "lg_ea", "lg_stale", "lg_fresh", "lg_async", "lg_ea_poisson"])
def test_logistic_trajectory_matches_golden_reference(name):
    """Whole run_sync / run_async trajectories with sharded LogisticObjective
    node objectives (rows from every node's sample stream, host noise from
    its noise stream) against the compiled reference's output."""
    cfg, dc, obj, shards = _driver_case(name)
    if cfg.protocol == O.ASYNC_PULL:
        r = D.run_async_pull(dc, obj, dtype="f64", node_objs=shards)
    elif cfg.poisson:
        r = D.run_async_elastic(dc, obj, dtype="f64", node_objs=shards)
    else:
        r = D.run_sync(dc, obj, dtype="f64", node_objs=shards)
    gd = golden()
    assert r.t.tolist() == gd[f"{name}_t"].tolist()
    assert close(r.theta, gd[f"{name}_theta"], 1e-9)
    if cfg.protocol != O.ASYNC_PULL:
        assert close(r.delta_prev, gd[f"{name}_dprev"], 1e-9)
    if cfg.protocol == O.ELASTIC:
        assert close(r.center, gd[f"{name}_center"], 1e-9)


def test_logistic_value_semantic_mirror_consumes_sample_stream():
    """protocols.local_sgd_step with a LogisticObjective draws its rows from
    node.rng.sample like stochastic_gradient (objectives.cpp:154-157)."""
    X, y, l2 = dataset(n=16, d=64)
    obj = P.LogisticObjective(X, y, l2).shard(4, 12)
    node = P.make_node(0, np.linspace(-1, 1, 64), seed=3, run_id="mirror")
    h = Hyperparams(**HK(batch=5))
    out = P.local_sgd_step(node, obj, P.NoiseModel.zero(64), h)
    s = O.Stream.make(3, "mirror", 0, "sample")
    rows = s.draw_rows(4, 12, 5)
    la = lookahead(node.theta, node.delta_prev, 0.9, np.float64)
    G = O.logistic_grad(X, y, l2, la, rows)
    n = O.Nodes(node.theta[None], node.delta_prev[None], np.zeros(1, np.uint64))
    O.local_sgd_step(n, O.HyperParams(**HK(batch=5)), gfixed=G[None])
    assert close(out.theta, n.theta[0], 1e-12)
    # the mirror's stream advanced by exactly `batch` draws
    assert out.rng.sample.uniform_index(8) == s.uniform_index(8)


def test_logistic_errors():
    g = Group(8, 2, dtype="f64")
    with pytest.raises(N.DsgdError, match="no logistic dataset"):
        g.local_sgd_step(Hyperparams(**HK()), grad="logistic")
    with pytest.raises(N.InvalidArgument, match="logistic dataset is empty"):
        g.set_logistic(np.zeros((0, 8)), [], 0.1)
    with pytest.raises(N.InvalidArgument, match="l2 must be positive"):
        g.set_logistic(np.ones((2, 8)), [0, 1], 0.0)
    with pytest.raises(N.InvalidArgument, match="labels must be 0 or 1"):
        g.set_logistic(np.ones((2, 8)), [0, 3], 0.1)
    g.set_logistic(np.ones((4, 8)), [0, 1, 1, 0], 0.1)
    with pytest.raises(N.InvalidArgument, match="invalid sample range"):
        g.logistic_set_sample_range(0, 3, 3)
    with pytest.raises(N.InvalidArgument, match="invalid sample range"):
        g.logistic_set_sample_range(1, 0, 5)
    with pytest.raises(N.InvalidArgument, match="batch must be >= 1"):
        g.local_sgd_step(Hyperparams(**HK(batch=0)), grad="logistic",
                         rows=np.zeros((2, 1), np.uint64))
    with pytest.raises(N.InvalidArgument, match="row out of range"):
        g.local_sgd_step(Hyperparams(**HK(batch=1)), grad="logistic",
                         rows=np.array([[0], [4]], np.uint64))
    with pytest.raises(N.DsgdError, match="seed_streams"):
        g.local_sgd_step(Hyperparams(**HK(batch=1)), grad="logistic")
    g.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_logistic_trace_loss_matches_oracle(dtype):
    """make_trace_record's loss_mean (simulator.cpp:101-110) with the
    logistic objective: mean over nodes of LogisticObjective::value."""
    X, y, l2 = dataset(n=30, d=2001)
    p = 5
    g, theta, _, _, _ = setup(p, dtype, X, y, l2, seed=8)
    th = theta.astype(np.float64)
    want = np.mean([O.logistic_value(X.astype(NP[dtype]).astype(np.float64), y, l2, th[i])
                    for i in range(p)])
    tr = g.trace()
    assert tr["loss_mean"] == pytest.approx(want, rel=1e-12)
    g.close()


def test_logistic_trace_records_match_reference():
    """The logistic run's trace (no optimum: sq_err_opt null; loss =
    LogisticObjective::value) against the reference's records."""
    from tests.golden.make_golden import TRACE_CASES
    cfg, dc, obj, shards = _driver_case("lg_pull")
    dc.trace_every = TRACE_CASES["lg_pull"]
    r = D.run_sync(dc, obj, dtype="f64", node_objs=shards)
    gold = np.load("tests/golden/traces.npz")["lg_pull_rec"]
    assert len(r.trace) == len(gold)
    for rec, g in zip(r.trace, gold):
        assert rec.t == int(g[0]) and rec.sim_time == g[1] and rec.alpha == g[5]
        assert rec.sq_err_opt is None and np.isnan(g[2])
        assert rec.sq_err_consensus == pytest.approx(g[3], rel=1e-8)
        assert rec.loss_mean == pytest.approx(g[4], rel=1e-9)


def test_p_nodes_batch_b_match_one_node_batch_pb():
    """test_protocols.cpp:221-247 through the value-semantic mirror: two
    all-reduce nodes with batch 2 (rows from their own sample streams,
    gradient on the device) track one node stepping with the mean of the
    two shards' minibatch gradients (MeanOfStreamsObjective, 51-79) drawn
    from copies of the same streams, within 1e-10; both nodes stay equal."""
    X = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [-1.0, 0.5], [0.5, -0.5], [2.0, 0.0]])
    y = np.array([1, 0, 1, 0, 1, 0], dtype=np.int32)
    data = P.LogisticObjective(X, y, 0.05)
    noise = P.NoiseModel.zero(2)
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.0, weight_decay=0.0, batch=2)
    theta0 = np.array([0.3, -0.2])
    nodes = [P.make_node(i, theta0, 9, "eq") for i in range(2)]
    copies = [O.Stream.make(9, "eq", i, "sample") for i in range(2)]  # the merged objective's
    single = O.Nodes(theta0[None].copy())
    hs = O.HyperParams(alpha0=0.1, anneal_at=(), mu=0.0, weight_decay=0.0, batch=4)
    for _ in range(20):
        nodes = P.allreduce_round(nodes, data, noise, h)
        th = single.theta[0]
        acc = np.zeros(2)
        for s in copies:
            acc = acc + O.logistic_grad(X, y, 0.05, th, s.draw_rows(0, 6, 2))
        acc = acc * (1.0 / 2)
        O.local_sgd_step(single, hs, gfixed=acc[None])
        assert np.abs(nodes[0].theta - single.theta[0]).max() <= 1e-10
        assert nodes[0].theta.tobytes() == nodes[1].theta.tobytes()


@pytest.mark.parametrize("name", ["lg_pull", "lg_allreduce"])
def test_logistic_trajectory_fp32_matches_fp32_restatement(name):
    """fp32 contexts over 40 rounds against the oracle's fp32 logistic run
    (same rows, noise and partners; the device's tree-summed dot product is
    the only difference): within 1e-5."""
    cfg, dc, obj, shards = _driver_case(name)
    r = D.run_sync(dc, obj, dtype="f32", node_objs=shards)
    gd = golden()
    th, dp, t = O.logistic_run(cfg, gd["X"], gd["y"], float(gd["l2"]), gd["ranges"],
                               dtype=np.float32)
    assert r.t.tolist() == t.tolist()
    assert close(r.theta.astype(np.float32), th, 1e-5)
