"""Per-step worker loop: run_sync (simulator.cpp:214-374) and the async-pull
driver (run_async 380-449) on the device.

The round loop itself runs in C++ inside the library (dsgd_run_rounds:
gating, step sizes, partner draws from the reference streams, host noise
draws, fused kernels); this module builds the initial nodes exactly as
make_initial_nodes (simulator.cpp:162-208) and collects the result.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .engine import Group, Hyperparams, Stream
from .protocols import InvalidArgument, LogisticObjective, NoiseModel, QuadraticObjective

PROTOCOLS = {"all-reduce": N.ALLREDUCE, "elastic-avg": N.ELASTIC_AVG,
             "pull-gossip": N.PULL_GOSSIP, "push-gossip": N.PUSH_GOSSIP,
             "gossip-stale": N.GOSSIP_STALE, "gossip-fresh": N.GOSSIP_FRESH,
             "async-pull": N.ASYNC_PULL}


@dataclass
class InitSpec:
    """simulator.hpp:57-70"""
    kind: str = "offset-ones"   # zeros | offset-ones | gaussian-spread | explicit
    target_sq_err: float = 8.0
    scale: float = 1.0
    values: Optional[Sequence[float]] = None


@dataclass
class SimConfig:
    """simulator.hpp:72-90 (the parameter-relevant fields)."""
    protocol: str = "all-reduce"
    p: int = 8
    hyper: Hyperparams = field(default_factory=Hyperparams)
    noise: Optional[NoiseModel] = None
    init: InitSpec = field(default_factory=InitSpec)
    momentum_scope: str = "per-node"   # SimConfig default (simulator.hpp:80)
    rounds: int = 1000
    events: int = 10000
    rate_per_node: float = 1.0
    seed: int = 1
    run_id: str = "run"


@dataclass
class RunResult:
    theta: np.ndarray          # [p, d]
    delta_prev: np.ndarray     # [p, d]
    t: np.ndarray              # [p]
    center: Optional[np.ndarray] = None


def make_initial_nodes(cfg: SimConfig, obj: QuadraticObjective) -> np.ndarray:
    d = obj.dim()
    opt = obj.optimum()
    kind = cfg.init.kind
    if kind == "zeros":
        base = np.zeros(d)
    elif kind == "offset-ones":
        if opt is None:
            raise InvalidArgument("offset-ones init requires an objective with a known optimum")
        if not cfg.init.target_sq_err > 0:
            raise InvalidArgument("init target_sq_err must be positive")
        c = math.sqrt(cfg.init.target_sq_err / (float(cfg.p) * float(d)))
        base = opt + c
    elif kind == "gaussian-spread":
        base = np.zeros(d) if opt is None else opt.copy()
    elif kind == "explicit":
        if cfg.init.values is None or len(cfg.init.values) != d:
            raise InvalidArgument("explicit init size must match objective dimension")
        base = np.asarray(cfg.init.values, dtype=np.float64)
    else:
        raise InvalidArgument(f"unknown init kind {kind}")
    thetas = np.tile(base, (cfg.p, 1))
    if kind == "gaussian-spread":
        for i in range(cfg.p):
            s = Stream.make(cfg.seed, cfg.run_id, i, "init")
            thetas[i] = base + cfg.init.scale * s.fill_normal(1.0, d)
    return thetas


def _group_for(cfg: SimConfig, d: int, dtype: str, center: bool = False,
               obj=None, node_objs=None, device: int = 0) -> Group:
    noise = cfg.noise is not None and cfg.noise.kind != "zero"
    logistic = isinstance(obj, LogisticObjective)
    g = Group(d, cfg.p, dtype=dtype, quadratic=not logistic, noise=noise, center=center,
              device=device)
    try:
        _set_objective(g, cfg, obj, node_objs)
    except Exception:
        g.close()
        raise
    return g


def _set_objective(g: Group, cfg: SimConfig, obj, node_objs):
    """Quadratic: spectrum/optimum buffers.  Logistic: the dataset, and each
    node's sample range from node_objs (run_sync(cfg, eval_obj, node_objs),
    simulator.hpp:134-140; the sharded runs of runner.cpp:100-115)."""
    if isinstance(obj, LogisticObjective):
        g.set_logistic(obj.features, obj.labels, obj.l2)
        objs = node_objs if node_objs is not None else [obj] * cfg.p
        if len(objs) != cfg.p:
            raise InvalidArgument("node objective count must equal p")
        for i, o in enumerate(objs):
            if not isinstance(o, LogisticObjective) or o.dim() != obj.dim():
                raise InvalidArgument("node objectives must share the evaluation dimension")
            if not np.array_equal(o.features, obj.features) or o.l2 != obj.l2:
                raise InvalidArgument("node objectives must share the device dataset")
            g.logistic_set_sample_range(i, *o.range)
        g.seed_streams(cfg.seed, cfg.run_id)
    else:
        g.set_quadratic(obj.spectrum, obj.opt)


def _grad_kind(obj) -> str:
    return "logistic" if isinstance(obj, LogisticObjective) else "quadratic"


def run_sync(cfg: SimConfig, obj: QuadraticObjective, dtype: str = "f64",
             device: int = 0, node_objs=None) -> RunResult:
    """run_sync for all-reduce, elastic-avg, pull/push gossip, gossip-stale
    and gossip-fresh -- every round one fused kernel (two for fresh).  With
    a LogisticObjective the minibatch gradient of each node is computed on
    the device first (rows from the node's sample stream)."""
    if cfg.protocol not in PROTOCOLS or cfg.protocol == "async-pull":
        raise InvalidArgument("async-pull requires the asynchronous driver")
    if cfg.rounds == 0:
        raise InvalidArgument("rounds must be >= 1")
    d = obj.dim()
    if cfg.noise is not None and cfg.noise.dim != d:
        raise InvalidArgument("noise dimension must match objective dimension")
    thetas = make_initial_nodes(cfg, obj)
    g = _group_for(cfg, d, dtype, cfg.protocol == "elastic-avg", obj, node_objs, device)
    try:
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        if cfg.protocol == "elastic-avg":
            g.ea_init_center()   # spatial_mean(theta_0)  simulator.cpp:62-67
        g.seed_streams(cfg.seed, cfg.run_id)
        sigma = cfg.noise.sigma if cfg.noise is not None and cfg.noise.kind != "zero" else 0.0
        g.run_rounds(PROTOCOLS[cfg.protocol], cfg.hyper, cfg.rounds,
                     scope=cfg.momentum_scope, grad=_grad_kind(obj), host_noise_sigma=sigma)
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        t = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], t[i] = g.get_state(i)
        center = g.get_center() if cfg.protocol == "elastic-avg" else None
        return RunResult(th, dp, t, center)
    finally:
        g.close()


def run_async_elastic(cfg: SimConfig, obj: QuadraticObjective, dtype: str = "f64",
                      device: int = 0, node_objs=None) -> RunResult:
    """run_async for elastic-avg under the Poisson clock (simulator.cpp:
    380-449): master clock (gap, then node); the ticking client runs
    ea_client_step + ea_server_apply when gated on its own t, else a local
    step -- one fused event kernel per tick."""
    if cfg.events == 0:
        raise InvalidArgument("events must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = _group_for(cfg, d, dtype, True, obj, node_objs, device)
    try:
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        g.ea_init_center()
        clock = Stream.make(cfg.seed, cfg.run_id, 0xFFFFFFFF, "clock")
        noise = [Stream.make(cfg.seed, cfg.run_id, i, "gradient-noise") for i in range(cfg.p)]
        t = [0] * cfg.p
        tau = cfg.hyper.tau
        for _ in range(cfg.events):
            clock.exponential(cfg.p * cfg.rate_per_node)
            i = clock.uniform_index(cfg.p)
            if use_noise:
                g.set_vector(i, N.BUF_NOISE, noise[i].fill_normal(cfg.noise.sigma, d))
            gated = t[i] > 0 and t[i] % tau == 0
            g.ea_client_event(cfg.hyper, i, gated, grad=_grad_kind(obj), noise=use_noise)
            t[i] += 1
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        tt = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], tt[i] = g.get_state(i)
        return RunResult(th, dp, tt, g.get_center())
    finally:
        g.close()


def run_async_pull(cfg: SimConfig, obj: QuadraticObjective, dtype: str = "f64",
                   device: int = 0, node_objs=None) -> RunResult:
    """run_async for async-pull (simulator.cpp:380-449): master Poisson clock
    (gap, then node), partner from the ticking node's stream, one fused
    event kernel per tick."""
    if cfg.events == 0:
        raise InvalidArgument("events must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = _group_for(cfg, d, dtype, False, obj, node_objs, device)
    try:
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        clock = Stream.make(cfg.seed, cfg.run_id, 0xFFFFFFFF, "clock")
        partner = [Stream.make(cfg.seed, cfg.run_id, i, "partner-choice") for i in range(cfg.p)]
        noise = [Stream.make(cfg.seed, cfg.run_id, i, "gradient-noise") for i in range(cfg.p)]
        for _ in range(cfg.events):
            clock.exponential(cfg.p * cfg.rate_per_node)
            i = clock.uniform_index(cfg.p)
            j = partner[i].uniform_index(cfg.p)
            if use_noise:
                g.set_vector(i, N.BUF_NOISE, noise[i].fill_normal(cfg.noise.sigma, d))
            g.async_pull_event(cfg.hyper, i, j, grad=_grad_kind(obj), noise=use_noise)
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        t = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], t[i] = g.get_state(i)
        return RunResult(th, dp, t)
    finally:
        g.close()
