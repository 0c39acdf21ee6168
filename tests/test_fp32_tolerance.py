"""The north star's fp32 bar, for every rule, at the configs' shapes:
"per-step parameters must match within a stated fp32 tolerance (max rel err
1e-5)" against the reference's fp64 arithmetic (protocols.cpp:85-297).

* Teacher-forced: each fp32 GPU step starts from the fp64 oracle state
  (rounded to fp32 on upload, like every input) and is compared with the
  fp64 oracle step from the same state.  Error metric (norm-wise, max
  norm): max_k |x32 - x64| / max(max_k |x64|, 1e-3 * max_k |x64_0|) over
  every node's theta and delta_prev (and the EASGD center); bar 1e-5.
  Shapes: all-reduce p = 1 x 25M (configs[3] at N = 1), EASGD p = 8 x 25M
  (configs[2]), pull-gossip p = 8 x 10M (configs[1], partners from the
  reference partner streams), push / stale / fresh / async at p = 8 x 10M,
  per-node all-reduce p = 4 x 4M, local step p = 1 x 25M.
* Free-running: whole fp32 trajectories of every golden run_sync / run_async
  configuration, extended to >= 200 rounds (C1: 2000), against the fp64
  oracle (itself pinned to the compiled reference): same metric, bar 1e-5.
"""
import dataclasses

import numpy as np
import pytest

import oracle as O
from paper_1611_04581_b200 import _native as N
from paper_1611_04581_b200 import driver as D
from paper_1611_04581_b200 import protocols as P
from paper_1611_04581_b200.engine import (Group, Hyperparams, Stream, draw_pull_partners,
                                          draw_push_targets)

pytestmark = pytest.mark.gpu

TOL = 1e-5
HK = dict(alpha0=0.05, anneal_at=(2,), anneal_factor=0.5, mu=0.9, weight_decay=1e-4,
          beta_gossip=0.4, beta_ea=0.1, tau=1)

# rule -> (p, d, teacher-forced steps)
SHAPES = {
    "allreduce": (1, 25_000_000, 3),
    "local": (1, 25_000_000, 2),
    "allreduce_pn": (4, 4_000_000, 2),
    "ea": (8, 25_000_000, 2),
    "ea_ungated": (8, 10_000_000, 1),
    "pull": (8, 10_000_000, 3),
    "push": (8, 10_000_000, 2),
    "stale": (8, 10_000_000, 2),
    "fresh": (8, 10_000_000, 2),
    "async": (8, 10_000_000, 4),
}


def rel_err(x32, x64, floor):
    return float(np.abs(x32 - x64).max() / max(float(np.abs(x64).max()), floor))


def schedules(p, rounds, run_id="run/trial0"):
    """Partner / target maps from the reference partner streams (seed 1)."""
    pull = [Stream.make(1, run_id, i, "partner-choice") for i in range(p)]
    push = [Stream.make(1, run_id + "/push", i, "partner-choice") for i in range(p)]
    clock = Stream.make(1, run_id, 0xFFFFFFFF, "clock")
    maps = []
    for _ in range(rounds):
        i = clock.uniform_index(p)
        maps.append((draw_pull_partners(pull), draw_push_targets(push) if p > 1 else None,
                     (i, pull[i].uniform_index(p))))
    return maps


@pytest.mark.parametrize("rule", sorted(SHAPES))
def test_teacher_forced_fp32_step_within_1e5_of_fp64(rule):
    p, d, steps = SHAPES[rule]
    rng = np.random.default_rng(sum(map(ord, rule)))
    spec = rng.uniform(0.5, 2.0, d)
    opt = rng.normal(size=d)
    theta = rng.normal(size=(p, d))
    dprev = 0.1 * rng.normal(size=(p, d))
    center = rng.normal(size=d)
    use_noise = not rule.startswith("ea")  # keep the 8 x 25M case within host memory
    n64 = O.Nodes(theta, dprev, np.full(p, 1, dtype=np.uint64))
    del theta, dprev
    floor_th = 1e-3 * float(np.abs(n64.theta).max())
    floor_dp = 1e-3 * float(np.abs(n64.dprev).max())
    h, hc = Hyperparams(**HK), O.HyperParams(**HK)
    maps = schedules(p, steps)
    g = Group(d, p, dtype="f32", quadratic=True, noise=use_noise, center=rule.startswith("ea"))
    g.set_quadratic(spec, opt)
    worst = {"theta": 0.0, "delta": 0.0, "center": 0.0}
    try:
        for step in range(steps):
            noise = 0.01 * rng.normal(size=(p, d)) if use_noise else None
            for i in range(p):
                g.set_state(i, n64.theta[i], n64.dprev[i], int(n64.t[i]))
                if use_noise:
                    g.set_vector(i, N.BUF_NOISE, noise[i])
            if rule.startswith("ea"):
                g.set_center(center)
            partner, target, (ai, aj) = maps[step]
            kw = dict(grad="quadratic", noise=use_noise)
            okw = dict(spec=spec, opt=opt, noise=noise)
            if rule == "allreduce":
                g.allreduce_round(h, **kw)
                O.allreduce_round(n64, hc, per_node=False, **okw)
            elif rule == "allreduce_pn":
                g.allreduce_round(h, scope="per-node", **kw)
                O.allreduce_round(n64, hc, per_node=True, **okw)
            elif rule == "local":
                g.local_sgd_step(h, **kw)
                O.local_sgd_step(n64, hc, **okw)
            elif rule in ("ea", "ea_ungated"):
                gated = rule == "ea"
                g.ea_round(h, gated=gated, **kw)
                O.ea_round(n64, center, gated, hc, **okw)
                c32 = g.get_center()
                worst["center"] = max(worst["center"], rel_err(c32, center, floor_th))
            elif rule == "pull":
                g.pull_gossip_round(h, partner, **kw)
                O.pull_gossip_round(n64, partner, hc, **okw)
            elif rule == "push":
                g.push_gossip_round(h, target, **kw)
                O.push_gossip_round(n64, target, hc, **okw)
            elif rule == "stale":
                g.gossip_stale_round(h, partner, **kw)
                O.stale_round(n64, partner, hc, **okw)
            elif rule == "fresh":
                g.gossip_fresh_round(h, partner, **kw)
                O.fresh_round(n64, partner, hc, **okw)
            elif rule == "async":
                g.async_pull_event(h, ai, aj, **kw)
                O.async_pull_event(n64, ai, aj, hc, **okw)
            for i in range(p):
                th32, dp32, t32 = g.get_state(i)
                assert t32 == int(n64.t[i])
                worst["theta"] = max(worst["theta"], rel_err(th32, n64.theta[i], floor_th))
                if rule != "async":  # async_pull_event leaves delta_prev untouched
                    worst["delta"] = max(worst["delta"], rel_err(dp32, n64.dprev[i], floor_dp))
    finally:
        g.close()
    print(f"{rule} p={p} d={d}: worst rel err {worst}")
    assert max(worst.values()) <= TOL, worst
    assert worst["theta"] > 0.0  # fp32 really differs from fp64 (the test is not vacuous)


def golden_sync():
    from tests.golden.make_golden import RUN_CASES
    return {k: v for k, v in RUN_CASES.items() if not v.poisson}


def to_driver(cfg):
    from tests.test_gpu_parity import to_driver as td
    return td(cfg)


@pytest.mark.parametrize("name", sorted(golden_sync()))
def test_free_running_fp32_trajectory_within_1e5_of_fp64(name):
    """>= 200 rounds (C1: its own 2000) of the fp32 device run vs the fp64
    oracle run of the same configuration: noise streams, partner streams,
    gating and annealing identical; only the arithmetic width differs."""
    cfg = golden_sync()[name]
    if cfg.protocol == O.ASYNC_PULL:
        cfg = dataclasses.replace(cfg, events=max(cfg.events, 1600))
    else:
        cfg = dataclasses.replace(cfg, rounds=max(cfg.rounds, 300))
    obj = P.QuadraticObjective(cfg.spectrum, cfg.opt)
    dc = to_driver(cfg)
    r = D.run_async_pull(dc, obj, dtype="f32") if cfg.protocol == O.ASYNC_PULL else \
        D.run_sync(dc, obj, dtype="f32")
    th64, dp64, t64, c64 = O.run(cfg, dtype=np.float64)
    assert r.t.tolist() == t64.tolist()
    floor = 1e-3 * float(np.abs(th64).max())
    err = rel_err(r.theta, th64, floor)
    print(f"{name}: {cfg.rounds} rounds, fp32 vs fp64 rel err {err:.3e}")
    assert err <= TOL
    if cfg.protocol == O.ELASTIC:
        assert rel_err(r.center, c64, floor) <= TOL
