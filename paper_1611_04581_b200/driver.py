"""Per-step worker loop: run_sync (simulator.cpp:214-374) and the async-pull
driver (run_async 380-449) on the device.

The round loop itself runs in C++ inside the library (dsgd_run_rounds:
gating, step sizes, partner draws from the reference streams, host noise
draws, fused kernels); this module builds the initial nodes exactly as
make_initial_nodes (simulator.cpp:162-208) and collects the result.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .engine import Group, Hyperparams, Stream, step_size_at
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
    trace_every: int = 10             # simulator.hpp:86
    exchange_latency: float = 0.0     # added to gated gossip rounds (virtual time)
    straggler_constant: float = 1.0   # StragglerModel kConstant (the default model)


@dataclass
class TraceRecord:
    """dsgd::TraceRecord (core.hpp:105-116)."""
    run_id: str
    protocol: str
    t: int
    sim_time: Optional[float]
    sq_err_opt: Optional[float]
    sq_err_consensus: float
    loss_mean: float
    alpha: float

    def to_json_line(self) -> str:
        """trace_record_to_json_line (trace_io.cpp:40-51): nlohmann's
        default object is a std::map, so keys come out sorted; compact."""
        j = {"run_id": self.run_id, "protocol": self.protocol, "t": int(self.t),
             "sim_time": self.sim_time, "sq_err_opt": self.sq_err_opt,
             "sq_err_consensus": self.sq_err_consensus, "loss_mean": self.loss_mean,
             "alpha": self.alpha}
        return json.dumps(j, sort_keys=True, separators=(",", ":"))

    @staticmethod
    def from_json_line(line: str) -> "TraceRecord":
        """trace_record_from_json_line (trace_io.cpp:53-77)."""
        try:
            j = json.loads(line)
        except ValueError as e:
            raise RuntimeError(f"trace line is not valid JSON: {e}")
        try:
            proto = j["protocol"]
            if proto not in PROTOCOLS:
                raise RuntimeError("unknown protocol name: " + str(proto))
            opt = lambda k: None if j[k] is None else float(j[k])  # noqa: E731
            return TraceRecord(str(j["run_id"]), proto, int(j["t"]), opt("sim_time"),
                               opt("sq_err_opt"), float(j["sq_err_consensus"]),
                               float(j["loss_mean"]), float(j["alpha"]))
        except (KeyError, TypeError) as e:
            raise RuntimeError(f"trace line missing or mistyped field: {e}")


def write_trace_jsonl(trace: Sequence[TraceRecord]) -> str:
    return "".join(r.to_json_line() + "\n" for r in trace)


@dataclass
class RunResult:
    theta: np.ndarray          # [p, d]
    delta_prev: np.ndarray     # [p, d]
    t: np.ndarray              # [p]
    center: Optional[np.ndarray] = None
    trace: List[TraceRecord] = field(default_factory=list)
    sim_time: float = 0.0


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


def _record(g: Group, cfg: SimConfig, obj, t: int, sim_time: float, alpha: float) -> TraceRecord:
    """make_trace_record (simulator.cpp:92-123) on the device: one fused
    reduction over every node's theta (fp64 accumulation)."""
    m = g.trace()
    return TraceRecord(cfg.run_id, cfg.protocol, t, sim_time,
                       m["sq_err_opt"] if obj.optimum() is not None else None,
                       m["sq_err_consensus"], m["loss_mean"], alpha)


def _run_events(g: Group, cfg: SimConfig, obj, protocol: int, use_noise: bool):
    """The run_async event loop in the library (dsgd_run_events: clock,
    partner and noise streams, one fused event kernel per tick), cut at the
    trace points (simulator.cpp:431-434)."""
    g.seed_streams(cfg.seed, cfg.run_id)
    sigma = cfg.noise.sigma if use_noise else 0.0
    trace = [_record(g, cfg, obj, 0, 0.0, step_size_at(cfg.hyper, 0))]
    done, sim_time, alpha = 0, 0.0, 0.0
    while done < cfg.events:
        k = min(cfg.trace_every - done % cfg.trace_every, cfg.events - done)
        sim_time, alpha = g.run_events(protocol, cfg.hyper, k, cfg.rate_per_node,
                                       grad=_grad_kind(obj), host_noise_sigma=sigma,
                                       sim_time=sim_time, alpha=alpha)
        done += k
        trace.append(_record(g, cfg, obj, done, sim_time, alpha))
    return trace, sim_time


def _round_time(cfg: SimConfig, gated: bool) -> float:
    """Virtual time of one synchronous round under the constant straggler
    model (simulator.cpp:240-349): every node takes `constant`, gated gossip
    rounds add the exchange latency (push only when p > 1)."""
    lat = 0.0
    if gated and cfg.protocol in ("pull-gossip", "gossip-stale", "gossip-fresh"):
        lat = cfg.exchange_latency
    if gated and cfg.protocol == "push-gossip" and cfg.p > 1:
        lat = cfg.exchange_latency
    return cfg.straggler_constant + lat


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
    if cfg.trace_every == 0:
        raise InvalidArgument("trace_every must be >= 1")
    if not cfg.straggler_constant > 0:
        raise InvalidArgument("straggler constant must be positive")
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
        h = cfg.hyper
        trace = [_record(g, cfg, obj, 0, 0.0, step_size_at(h, 0))]
        done, sim_time = 0, 0.0
        while done < cfg.rounds:
            # run up to the next trace point in one library call (the round
            # loop itself runs in C++)
            k = min(cfg.trace_every - done % cfg.trace_every, cfg.rounds - done)
            g.run_rounds(PROTOCOLS[cfg.protocol], h, k,
                         scope=cfg.momentum_scope, grad=_grad_kind(obj), host_noise_sigma=sigma)
            for r in range(done, done + k):
                sim_time += _round_time(cfg, r > 0 and r % h.tau == 0)
            done += k
            trace.append(_record(g, cfg, obj, done, sim_time, step_size_at(h, done)))
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        t = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], t[i] = g.get_state(i)
        center = g.get_center() if cfg.protocol == "elastic-avg" else None
        return RunResult(th, dp, t, center, trace, sim_time)
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
    if cfg.trace_every == 0:
        raise InvalidArgument("trace_every must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = _group_for(cfg, d, dtype, True, obj, node_objs, device)
    try:
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        g.ea_init_center()
        trace, sim_time = _run_events(g, cfg, obj, N.ELASTIC_AVG, use_noise)
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        tt = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], tt[i] = g.get_state(i)
        return RunResult(th, dp, tt, g.get_center(), trace, sim_time)
    finally:
        g.close()


def run_async_pull(cfg: SimConfig, obj: QuadraticObjective, dtype: str = "f64",
                   device: int = 0, node_objs=None) -> RunResult:
    """run_async for async-pull (simulator.cpp:380-449): master Poisson clock
    (gap, then node), partner from the ticking node's stream, one fused
    event kernel per tick."""
    if cfg.events == 0:
        raise InvalidArgument("events must be >= 1")
    if cfg.trace_every == 0:
        raise InvalidArgument("trace_every must be >= 1")
    d = obj.dim()
    thetas = make_initial_nodes(cfg, obj)
    use_noise = cfg.noise is not None and cfg.noise.kind != "zero"
    g = _group_for(cfg, d, dtype, False, obj, node_objs, device)
    try:
        for i in range(cfg.p):
            g.set_state(i, thetas[i])
        trace, sim_time = _run_events(g, cfg, obj, N.ASYNC_PULL, use_noise)
        th = np.zeros((cfg.p, d))
        dp = np.zeros((cfg.p, d))
        t = np.zeros(cfg.p, dtype=np.uint64)
        for i in range(cfg.p):
            th[i], dp[i], t[i] = g.get_state(i)
        return RunResult(th, dp, t, None, trace, sim_time)
    finally:
        g.close()
