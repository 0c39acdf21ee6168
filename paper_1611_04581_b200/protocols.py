"""The reference's update-rule interface, value semantics included
(/root/reference/proj/include/dsgd/protocols.hpp:45-152),
executed by the B200 kernels.

Every function here has the reference signature: it takes NodeStates (host
fp64 vectors + streams) by value and returns new ones.  Internally it
uploads the states to a cached device ``Group``, runs the fused CUDA kernel
of that rule through the C ABI and downloads the result -- there is no host
arithmetic on parameters and no CPU fallback.  Noise draws come from each
node's own reference stream on the host (NoiseModel::sample,
objectives.cpp:175-183) so trajectories are bit-identical with the reference
in ``dtype="f64"`` and the same operation order in ``"f32"``.

This mirror exists so callers and parity tests read like the reference's own
(proj/tests/test_protocols.cpp); the performance path is ``engine.Group``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _native as N
from .engine import (Group, Hyperparams, Stream, derive_stream_seed, draw_pull_partners,
                     draw_push_targets, step_size_at)

InvalidArgument = N.InvalidArgument
TransportError = N.TransportError

AGGREGATE, PER_NODE = "aggregate", "per-node"


# ------------------------------------------------------------ objectives
class QuadraticObjective:
    """f = 1/2 sum_k a_k (theta_k - opt_k)^2 (objectives.hpp:57-73)."""

    def __init__(self, spectrum: Sequence[float], opt: Optional[Sequence[float]] = None):
        self.spectrum = np.asarray(spectrum, dtype=np.float64)
        if self.spectrum.size == 0:
            raise InvalidArgument("quadratic spectrum must be non-empty")
        if not (self.spectrum > 0).all():
            raise InvalidArgument("quadratic spectrum entries must be positive")
        self.opt = (np.zeros_like(self.spectrum) if opt is None
                    else np.asarray(opt, dtype=np.float64))
        if self.opt.shape != self.spectrum.shape:
            raise InvalidArgument("quadratic optimum dimension must match spectrum")

    def dim(self) -> int:
        return self.spectrum.size

    def optimum(self) -> np.ndarray:
        return self.opt

    def convexity_params(self):
        return float(self.spectrum.min()), float(self.spectrum.max())


class GradientObjective:
    """The Objective plugin slot (objectives.hpp:33-53) filled with a given
    minibatch gradient -- the GPU path's external gradient buffer."""

    def __init__(self, gradient: Sequence[float]):
        self.gradient = np.asarray(gradient, dtype=np.float64)

    def dim(self) -> int:
        return self.gradient.size


class LogisticObjective:
    """l2-regularised logistic regression on a fixed design matrix
    (objectives.hpp:75-107, objectives.cpp:80-162): the dataset lives on the
    device and the minibatch gradient is computed there (DSGD_GRAD_LOGISTIC)."""

    def __init__(self, features, labels: Sequence[int], l2: float):
        rows = [np.asarray(r, dtype=np.float64) for r in features]
        if not rows:
            raise InvalidArgument("logistic dataset is empty")
        if len(rows) != len(labels):
            raise InvalidArgument("logistic features/labels size mismatch")
        if not l2 > 0.0:
            raise InvalidArgument("logistic l2 must be positive (strong convexity)")
        d = rows[0].size
        if any(r.size != d for r in rows):
            raise InvalidArgument("logistic feature rows have inconsistent width")
        if any(int(y) not in (0, 1) for y in labels):
            raise InvalidArgument("logistic labels must be 0 or 1")
        self.features = np.stack(rows)
        self.labels = np.asarray(labels, dtype=np.int32)
        self.l2 = float(l2)
        self.range = (0, len(rows))
        self.lipschitz = self.l2 + 0.25 * float((self.features ** 2).sum(axis=1).max())

    def dim(self) -> int:
        return self.features.shape[1]

    def num_samples(self) -> int:
        return self.features.shape[0]

    def optimum(self):
        return None

    def set_sample_range(self, begin: int, end: int) -> None:
        """objectives.cpp:108-114"""
        if begin >= end or end > self.num_samples():
            raise InvalidArgument("invalid sample range")
        self.range = (begin, end)

    def shard(self, begin: int, end: int) -> "LogisticObjective":
        o = LogisticObjective.__new__(LogisticObjective)
        o.__dict__.update(self.__dict__)
        o.set_sample_range(begin, end)
        return o

    def convexity_params(self):
        return self.l2, self.lipschitz


Objective = Union[QuadraticObjective, GradientObjective, LogisticObjective]


@dataclass
class NoiseModel:
    """Additive gradient noise (objectives.hpp:109-127)."""
    kind: str = "zero"
    sigma: float = 0.0
    dim: int = 0

    @staticmethod
    def zero(dim: int) -> "NoiseModel":
        return NoiseModel("zero", 0.0, dim)

    @staticmethod
    def gaussian_per_coord(sigma: float, dim: int) -> "NoiseModel":
        if sigma < 0:
            raise InvalidArgument("noise sigma must be >= 0")
        return NoiseModel("gaussian", sigma, dim)

    @staticmethod
    def gaussian_total(total_variance: float, dim: int) -> "NoiseModel":
        if total_variance < 0:
            raise InvalidArgument("total variance must be >= 0")
        if dim == 0:
            raise InvalidArgument("noise dim must be >= 1")
        return NoiseModel("gaussian", math.sqrt(total_variance / dim), dim)

    def sample(self, rng: Stream) -> Optional[np.ndarray]:
        """None for the zero kind (no draws; the kernel adds +0.0)."""
        if self.kind == "zero":
            return None
        return rng.fill_normal(self.sigma, self.dim)


# --------------------------------------------------------------- state
@dataclass
class NodeRng:
    noise: Stream
    sample: Stream
    partner: Stream
    straggler: Stream

    def clone(self) -> "NodeRng":
        return NodeRng(self.noise.clone(), self.sample.clone(), self.partner.clone(),
                       self.straggler.clone())


@dataclass
class NodeState:
    """dsgd::NodeState (core.hpp:92-98)."""
    id: int
    theta: np.ndarray
    delta_prev: np.ndarray
    t: int
    rng: NodeRng

    def copy(self) -> "NodeState":
        return NodeState(self.id, self.theta.copy(), self.delta_prev.copy(), self.t,
                         self.rng.clone())


def make_node_rng(seed: int, run_id: str, node: int) -> NodeRng:
    return NodeRng(Stream.make(seed, run_id, node, "gradient-noise"),
                   Stream.make(seed, run_id, node, "sample"),
                   Stream.make(seed, run_id, node, "partner-choice"),
                   Stream.make(seed, run_id, node, "straggler"))


def make_node(node_id: int, theta0, seed: int = 1, run_id: str = "run") -> NodeState:
    th = np.array(theta0, dtype=np.float64, copy=True).reshape(-1)
    return NodeState(node_id, th, np.zeros_like(th), 0, make_node_rng(seed, run_id, node_id))


@dataclass
class ServerState:
    """EASGD server (protocols.hpp:30-33)."""
    theta_center: np.ndarray
    applied_updates: int = 0


# ------------------------------------------------------ device plumbing
_GROUPS = {}


def _group(p: int, d: int, dtype: str) -> Group:
    key = (p, d, dtype)
    g = _GROUPS.get(key)
    if g is None:
        g = Group(d, p, dtype=dtype, quadratic=True, grad=True, noise=True, center=True)
        _GROUPS[key] = g
    return g


def _objs(obj, p: int) -> List[Objective]:
    objs = list(obj) if isinstance(obj, (list, tuple)) else [obj] * p
    if len(objs) != p:
        raise InvalidArgument("objective list size must equal node count")
    if any(o is None for o in objs):
        raise InvalidArgument("null objective")
    return objs


def _load(g: Group, nodes: Sequence[NodeState], objs: Sequence[Objective],
          noise: Optional[NoiseModel], draw: Sequence[bool], h: Optional[Hyperparams] = None):
    """Upload states, objective and this step's noise; returns the gradient
    keyword arguments of the Group rule call."""
    d = g.d
    for i, n in enumerate(nodes):
        if n.theta.size != d or n.delta_prev.size != d:
            raise InvalidArgument("ParamVec dimension mismatch")
        g.set_state(i, n.theta, n.delta_prev, n.t)
    quad = isinstance(objs[0], QuadraticObjective)
    rows = None
    if isinstance(objs[0], LogisticObjective):
        # the dataset on the device; each drawing node's minibatch rows from its
        # own sample stream (objectives.cpp:154-157), consumed here on the host
        base = objs[0]
        if any(not isinstance(o, LogisticObjective) or o.dim() != d for o in objs):
            raise InvalidArgument("stochastic_gradient: dimension mismatch")
        if any(not np.array_equal(o.features, base.features) or o.l2 != base.l2 for o in objs):
            raise InvalidArgument("per-node logistic objectives must share one dataset")
        g.set_logistic(base.features, base.labels, base.l2)
        batch = h.batch if h is not None else 1
        if batch == 0:
            raise InvalidArgument("batch must be >= 1")
        rows = np.zeros((len(nodes), batch), dtype=np.uint64)
        for i, (n, o) in enumerate(zip(nodes, objs)):
            b, e = o.range
            rows[i] = [b + n.rng.sample.uniform_index(e - b) for _ in range(batch)] \
                if draw[i] else b
    elif quad:
        for o in objs:
            if not isinstance(o, QuadraticObjective) or not (
                    o.spectrum is objs[0].spectrum or np.array_equal(o.spectrum, objs[0].spectrum)) \
                    or not np.array_equal(o.opt, objs[0].opt):
                raise InvalidArgument("per-node objectives must share one quadratic")
            if o.dim() != d:
                raise InvalidArgument("gradient: dimension mismatch")
        g.set_quadratic(objs[0].spectrum, objs[0].opt)
    else:
        for i, o in enumerate(objs):
            if o.dim() != d:
                raise InvalidArgument("gradient: dimension mismatch")
            g.set_vector(i, N.BUF_GRAD, o.gradient)
    use_noise = noise is not None and noise.kind != "zero"
    if use_noise:
        if noise.dim != d:
            raise InvalidArgument("noise dimension must match objective")
        for i, n in enumerate(nodes):
            xi = noise.sample(n.rng.noise) if draw[i] else np.zeros(d)
            g.set_vector(i, N.BUF_NOISE, xi)
    if rows is not None:
        return dict(grad="logistic", noise=use_noise, rows=rows)
    return dict(grad="quadratic" if quad else "buffer", noise=use_noise)


def _store(g: Group, nodes: Sequence[NodeState]) -> List[NodeState]:
    out = []
    for i, n in enumerate(nodes):
        th, dp, t = g.get_state(i)
        out.append(NodeState(n.id, th, dp, t, n.rng))
    return out


def _by_value(nodes: Sequence[NodeState]) -> List[NodeState]:
    return [n.copy() for n in nodes]


def _norm_update(grad_norm_out, v):
    if grad_norm_out is not None and v is not None:
        grad_norm_out[0] = max(grad_norm_out[0], v)


# --------------------------------------------------------- update rules
def local_sgd_step(node: NodeState, obj: Objective, noise: NoiseModel, h: Hyperparams,
                   grad_norm_out: Optional[list] = None, dtype: str = "f64") -> NodeState:
    """protocols.cpp:102-108 (fused kernel k_step, mode step)."""
    node = node.copy()
    g = _group(1, node.theta.size, dtype)
    kw = _load(g, [node], _objs(obj, 1), noise, [True], h)
    _norm_update(grad_norm_out, g.local_sgd_step(h, **kw,
                                                 grad_norm=grad_norm_out is not None))
    return _store(g, [node])[0]


def compute_local_delta(node: NodeState, obj: Objective, noise: NoiseModel, h: Hyperparams,
                        grad_norm_out: Optional[list] = None, dtype: str = "f64") -> np.ndarray:
    """protocols.cpp:85-100: the step's delta; consumes node's noise stream
    (node is taken by reference), leaves theta and t untouched."""
    g = _group(1, node.theta.size, dtype)
    kw = _load(g, [node], _objs(obj, 1), noise, [True], h)
    _norm_update(grad_norm_out, g.local_sgd_step(h, **kw,
                                                 grad_norm=grad_norm_out is not None))
    return g.get_state(0)[1]


def allreduce_round(nodes: Sequence[NodeState], obj, noise: NoiseModel, h: Hyperparams,
                    scope: str = AGGREGATE, grad_norm_out: Optional[list] = None,
                    dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:110-131 (fused kernel k_allreduce_local)."""
    if not nodes:
        raise InvalidArgument("allreduce_round on empty node set")
    if any(n.t != nodes[0].t for n in nodes):
        raise InvalidArgument("synchronous round requires equal node clocks")
    nodes = _by_value(nodes)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    kw = _load(g, nodes, _objs(obj, len(nodes)), noise, [True] * len(nodes), h)
    _norm_update(grad_norm_out, g.allreduce_round(h, scope=scope, **kw,
                                                  grad_norm=grad_norm_out is not None))
    return _store(g, nodes)


def ea_client_step(node: NodeState, center, obj: Objective, noise: NoiseModel,
                   h: Hyperparams, grad_norm_out: Optional[list] = None,
                   dtype: str = "f64") -> Tuple[NodeState, np.ndarray]:
    """protocols.cpp:140-153 (fused kernel k_ea_local with the update output)."""
    import torch
    center = np.asarray(center, dtype=np.float64)
    if center.size != node.theta.size:
        raise InvalidArgument("ea_client_step center dimension mismatch")
    node = node.copy()
    g = _group(1, node.theta.size, dtype)
    kw = _load(g, [node], _objs(obj, 1), noise, [True], h)
    g.set_center(center)
    upd = torch.empty(node.theta.size, dtype=torch.float64 if dtype == "f64" else torch.float32,
                      device=f"cuda:{g.device}")
    g.ea_set_update_out([upd.data_ptr()])
    try:
        _norm_update(grad_norm_out, g.ea_round(h, gated=True, **kw,
                                               grad_norm=grad_norm_out is not None))
        g.sync()
    finally:
        g.ea_set_update_out(None)
    return _store(g, [node])[0], upd.cpu().double().numpy()


def ea_server_apply(server: ServerState, update, dtype: str = "f64") -> ServerState:
    """protocols.cpp:155-159."""
    import torch
    update = np.asarray(update, dtype=np.float64)
    if update.size != server.theta_center.size:
        raise InvalidArgument("ParamVec dimension mismatch")
    g = _group(1, update.size, dtype)
    g.set_center(server.theta_center)
    u = torch.as_tensor(update, dtype=torch.float64 if dtype == "f64" else torch.float32).to(
        f"cuda:{g.device}")
    g.ea_server_apply(u.data_ptr())
    return ServerState(g.get_center(), server.applied_updates + 1)


def ea_sweep(nodes: Sequence[NodeState], server: ServerState, obj, noise: NoiseModel,
             h: Hyperparams, gated: bool = True, grad_norm_out: Optional[list] = None,
             dtype: str = "f64") -> Tuple[List[NodeState], ServerState]:
    """The synchronous EASGD sweep of run_sync (simulator.cpp:332-351): every
    client in node order against the serially updated center, one kernel."""
    nodes = _by_value(nodes)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    kw = _load(g, nodes, _objs(obj, len(nodes)), noise, [True] * len(nodes), h)
    g.set_center(server.theta_center)
    _norm_update(grad_norm_out, g.ea_round(h, gated=gated, **kw,
                                           grad_norm=grad_norm_out is not None))
    return _store(g, nodes), ServerState(g.get_center(),
                                         server.applied_updates + (len(nodes) if gated else 0))


def _check_partners(p: int, partner_of) -> np.ndarray:
    m = np.asarray(partner_of, dtype=np.int64).reshape(-1)
    if m.size != p:
        raise InvalidArgument("partner map size must equal node count")
    if (m < 0).any() or (m >= p).any():
        raise InvalidArgument("partner index out of range")
    return m.astype(np.uint32)


def pull_mix(nodes: Sequence[NodeState], partner_of, dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:161-171."""
    nodes = _by_value(nodes)
    m = _check_partners(len(nodes), partner_of)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    for i, n in enumerate(nodes):
        g.set_state(i, n.theta, n.delta_prev, n.t)
    g.pull_mix(m)
    return _store(g, nodes)


def pull_gossip_round(nodes: Sequence[NodeState], partner_of, obj, noise: NoiseModel,
                      h: Hyperparams, grad_norm_out: Optional[list] = None,
                      dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:173-185 (fused kernel k_step, mode pull)."""
    if any(n.t != nodes[0].t for n in nodes):
        raise InvalidArgument("synchronous round requires equal node clocks")
    nodes = _by_value(nodes)
    m = _check_partners(len(nodes), partner_of)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    kw = _load(g, nodes, _objs(obj, len(nodes)), noise, [True] * len(nodes), h)
    _norm_update(grad_norm_out, g.pull_gossip_round(h, m, **kw,
                                                    grad_norm=grad_norm_out is not None))
    return _store(g, nodes)


def _check_targets(p: int, target_of) -> np.ndarray:
    m = _check_partners(p, target_of)
    if any(int(m[k]) == k for k in range(p)):
        raise InvalidArgument("push target must differ from sender")
    return m


def push_mix(nodes: Sequence[NodeState], target_of, dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:195-228."""
    nodes = _by_value(nodes)
    m = _check_targets(len(nodes), target_of)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    for i, n in enumerate(nodes):
        g.set_state(i, n.theta, n.delta_prev, n.t)
    g.push_mix(m)
    return _store(g, nodes)


def push_gossip_round(nodes: Sequence[NodeState], target_of, obj, noise: NoiseModel,
                      h: Hyperparams, grad_norm_out: Optional[list] = None,
                      dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:230-242 (fused kernel k_push)."""
    if any(n.t != nodes[0].t for n in nodes):
        raise InvalidArgument("synchronous round requires equal node clocks")
    nodes = _by_value(nodes)
    m = _check_targets(len(nodes), target_of)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    kw = _load(g, nodes, _objs(obj, len(nodes)), noise, [True] * len(nodes), h)
    _norm_update(grad_norm_out, g.push_gossip_round(h, m, **kw,
                                                    grad_norm=grad_norm_out is not None))
    return _store(g, nodes)


def _pair(node: NodeState, partner_theta) -> List[NodeState]:
    pt = np.asarray(partner_theta, dtype=np.float64).reshape(-1)
    if pt.size != node.theta.size:
        raise InvalidArgument("mixing dimension mismatch")
    other = NodeState(node.id, pt.copy(), np.zeros_like(pt), node.t, node.rng)
    return [node, other]


def gossip_stale_step(node: NodeState, partner_theta, obj: Objective, noise: NoiseModel,
                      h: Hyperparams, grad_norm_out: Optional[list] = None,
                      dtype: str = "f64") -> NodeState:
    """protocols.cpp:252-263 (fused kernel k_step, mode stale)."""
    node = node.copy()
    pair = _pair(node, partner_theta)
    g = _group(2, node.theta.size, dtype)
    objs = [obj, obj if isinstance(obj, (QuadraticObjective, LogisticObjective)) else GradientObjective(
        np.zeros(node.theta.size))]
    kw = _load(g, pair, objs, noise, [True, False], h)
    _norm_update(grad_norm_out, g.gossip_stale_round(h, [1, 1], **kw,
                                                     grad_norm=grad_norm_out is not None))
    return _store(g, pair)[0]


def gossip_fresh_mix(stepped: NodeState, partner_theta_fresh, beta: float,
                     dtype: str = "f64") -> NodeState:
    """protocols.cpp:265-269."""
    stepped = stepped.copy()
    pair = _pair(stepped, partner_theta_fresh)
    g = _group(2, stepped.theta.size, dtype)
    for i, n in enumerate(pair):
        g.set_state(i, n.theta, n.delta_prev, n.t)
    g.gossip_fresh_mix([1, 1], beta)
    return _store(g, pair)[0]


def gossip_fresh_step(node: NodeState, partner_theta_fresh, obj: Objective, noise: NoiseModel,
                      h: Hyperparams, grad_norm_out: Optional[list] = None,
                      dtype: str = "f64") -> NodeState:
    """protocols.cpp:271-276."""
    stepped = local_sgd_step(node, obj, noise, h, grad_norm_out, dtype)
    return gossip_fresh_mix(stepped, partner_theta_fresh, h.beta_gossip, dtype)


def async_pull_event(nodes: Sequence[NodeState], i: int, j: int, obj: Objective,
                     noise: NoiseModel, h: Hyperparams, grad_norm_out: Optional[list] = None,
                     dtype: str = "f64") -> List[NodeState]:
    """protocols.cpp:278-297 (fused kernel k_step, mode async)."""
    if i >= len(nodes) or j >= len(nodes) or i < 0 or j < 0:
        raise InvalidArgument("async_pull_event node index out of range")
    nodes = _by_value(nodes)
    g = _group(len(nodes), nodes[0].theta.size, dtype)
    objs = [obj] * len(nodes)
    kw = _load(g, nodes, objs, noise, [k == i for k in range(len(nodes))], h)
    _norm_update(grad_norm_out, g.async_pull_event(h, i, j, **kw,
                                                   grad_norm=grad_norm_out is not None))
    return _store(g, nodes)


def spatial_mean(thetas: Sequence[np.ndarray], dtype: str = "f64") -> np.ndarray:
    """param_vec.cpp:19-40 (device pivot-form mean kernel)."""
    if len(thetas) == 0:
        raise InvalidArgument("spatial_mean over empty node set")
    d = np.asarray(thetas[0]).size
    if any(np.asarray(t).size != d for t in thetas):
        raise InvalidArgument("spatial_mean dimension mismatch")
    g = _group(len(thetas), d, dtype)
    for i, t in enumerate(thetas):
        g.set_state(i, t)
    g.ea_init_center()
    return g.get_center()
