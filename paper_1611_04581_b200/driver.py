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
from .protocols import InvalidArgument, NoiseModel, QuadraticObjective

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
        if not cfg.init.target_sq_err > 0:
            raise InvalidArgument("init target_sq_err must be positive")
        c = math.sqrt(cfg.init.target_sq_err / (float(cfg.p) * float(d)))
        base = opt + c
    elif kind == "gaussian-spread":
        base = opt.copy()
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


def _group_for(cfg: SimConfig, d: int, dtype: str) -> Group:
    noise = cfg.noise is not None and cfg.noise.kind != "zero"
    return Group(d, cfg.p, dtype=dtype, quadratic=True, noise=noise,
                 center=cfg.protocol == "elastic-avg")


def run_sync(cfg: SimConfig, obj: QuadraticObjective, dtype: str = "f64",
             device: int = 0) -> RunResult:
    """run_sync for all-reduce, elastic-avg, pull/push gossip, gossip-stale
    and gossip-fresh -- every round one fused kernel (two for fresh)."""
    if cfg.protocol not in PROTOCOLS or cfg.protocol == "async-pull":
        raise InvalidArgument("async-pull requires the asynchronous driver")
    if cfg.rounds == 0:
        raise InvalidArgument("rounds must be >= 1")
    d = obj.dim()
    if cfg.noise is not None and cfg.noise.dim != d:
        raise InvalidArgument("noise dimension must match objective dimension")
    thetas = make_initial_nodes(cfg, obj)
    g = _group_for(cfg, d, dtype)
    try:
        g.set_quadratic(obj.spectrum, obj.opt)
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        if cfg.protocol == "elastic-avg":
            g.ea_init_center()   # spatial_mean(theta_0)  simulator.cpp:62-67
        g.seed_streams(cfg.seed, cfg.run_id)
        sigma = cfg.noise.sigma if cfg.noise is not None and cfg.noise.kind != "zero" else 0.0
        g.run_rounds(PROTOCOLS[cfg.protocol], cfg.hyper, cfg.rounds,
                     scope=cfg.momentum_scope, grad="quadratic", host_noise_sigma=sigma)
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
                      device: int = 0) -> RunResult:
    """run_async for elastic-avg under the Poisson clock (simulator.cpp:
    380-449): master clock (gap, then node); the ticking client runs
    ea_client_step + ea_server_apply when gated on its own t, else a local
    step -- one fused event kernel per tick."""
    if cfg.events == 0:
        raise InvalidArgument("events must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = Group(d, cfg.p, dtype=dtype, quadratic=True, noise=use_noise, center=True,
              device=device)
    try:
        g.set_quadratic(obj.spectrum, obj.opt)
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
            g.ea_client_event(cfg.hyper, i, gated, grad="quadratic", noise=use_noise)
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
                   device: int = 0) -> RunResult:
    """run_async for async-pull (simulator.cpp:380-449): master Poisson clock
    (gap, then node), partner from the ticking node's stream, one fused
    event kernel per tick."""
    if cfg.events == 0:
        raise InvalidArgument("events must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = Group(d, cfg.p, dtype=dtype, quadratic=True, noise=use_noise)
    try:
        g.set_quadratic(obj.spectrum, obj.opt)
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
            g.async_pull_event(cfg.hyper, i, j, grad="quadratic", noise=use_noise)
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        t = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], t[i] = g.get_state(i)
        return RunResult(th, dp, t)
    finally:
        g.close()
