"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the B200 product path.

ctypes bindings over
  * ``libdsgd_oracle.so``  -- the plain-C restatement of the reference update
    rules (dsgd_oracle.c, each function cites the reference file:line it
    follows), in fp64 (reference arithmetic) and fp32 (same op order);
  * ``_ref/libdsgd_ref.so`` -- the unmodified reference sources compiled by
    oracle/Makefile with a C shim (ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1611_04581_b200`` never imports it.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libdsgd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdsgd_ref.so")

# protocol ids (dsgd_oracle.h)
ALLREDUCE, ELASTIC, PULL, PUSH, STALE, FRESH, ASYNC_PULL = range(7)
INIT_ZEROS, INIT_OFFSET_ONES, INIT_GAUSSIAN, INIT_EXPLICIT = range(4)
PURPOSE = {"gradient-noise": 0, "sample": 1, "partner-choice": 2, "clock": 3,
           "straggler": 4, "init": 5}
OBJ_QUADRATIC, OBJ_FIXED = 0, 1


def build(force: bool = False) -> None:
    """Build the checker libraries (make -C oracle)."""
    if force or not os.path.exists(ORACLE_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


class Hyper(C.Structure):
    _fields_ = [("alpha0", C.c_double), ("anneal_factor", C.c_double),
                ("anneal_at", C.POINTER(C.c_uint64)), ("n_anneal", C.c_uint32),
                ("mu", C.c_double), ("weight_decay", C.c_double),
                ("beta_gossip", C.c_double), ("beta_ea", C.c_double),
                ("tau", C.c_uint32), ("batch", C.c_uint32)]


class Sim(C.Structure):
    _fields_ = [("protocol", C.c_int), ("p", C.c_uint32), ("d", C.c_uint64),
                ("hyper", Hyper), ("noise_gaussian", C.c_int), ("sigma", C.c_double),
                ("spectrum", C.POINTER(C.c_double)), ("opt", C.POINTER(C.c_double)),
                ("init_kind", C.c_int), ("target_sq_err", C.c_double),
                ("init_scale", C.c_double), ("init_values", C.POINTER(C.c_double)),
                ("scope_per_node", C.c_int), ("poisson", C.c_int),
                ("rounds", C.c_uint64), ("events", C.c_uint64),
                ("rate_per_node", C.c_double), ("seed", C.c_uint64),
                ("run_id", C.c_char_p)]


@dataclass
class HyperParams:
    """Mirror of dsgd::Hyperparams (core.hpp:54-70); defaults are the reference's."""
    alpha0: float = 0.1
    anneal_factor: float = 0.1
    anneal_at: Sequence[int] = (150000, 300000)
    mu: float = 0.9
    weight_decay: float = 1e-4
    beta_gossip: float = 0.5
    beta_ea: float = 0.1
    tau: int = 1
    batch: int = 1

    def to_c(self) -> Hyper:
        arr = (C.c_uint64 * max(1, len(self.anneal_at)))(*self.anneal_at)
        h = Hyper(self.alpha0, self.anneal_factor, arr, len(self.anneal_at), self.mu,
                  self.weight_decay, self.beta_gossip, self.beta_ea, self.tau, self.batch)
        h._keep = arr  # keep the array alive with the struct
        return h


def plain(alpha: float, mu: float = 0.0) -> HyperParams:
    """The reference tests' ``plain`` helper (test_protocols.cpp:29-36)."""
    return HyperParams(alpha0=alpha, anneal_at=(), mu=mu, weight_decay=0.0)


@dataclass
class SimConfig:
    protocol: int = ALLREDUCE
    p: int = 8
    hyper: HyperParams = field(default_factory=HyperParams)
    sigma: Optional[float] = None      # None: NoiseModel::zero
    spectrum: Sequence[float] = (1.0, 2.0, 5.0, 10.0)
    opt: Optional[Sequence[float]] = None
    init_kind: int = INIT_OFFSET_ONES
    target_sq_err: float = 8.0
    init_scale: float = 1.0
    init_values: Optional[Sequence[float]] = None
    per_node_scope: bool = True        # SimConfig default (simulator.hpp:80)
    poisson: bool = False
    rounds: int = 100
    events: int = 1000
    rate_per_node: float = 1.0
    seed: int = 1
    run_id: str = "run"

    @property
    def d(self) -> int:
        return len(self.spectrum)

    def to_c(self):
        d = self.d
        spec = np.ascontiguousarray(self.spectrum, dtype=np.float64)
        opt = np.ascontiguousarray(self.opt if self.opt is not None else np.zeros(d), np.float64)
        init = np.ascontiguousarray(self.init_values if self.init_values is not None
                                    else np.zeros(d), np.float64)
        h = self.hyper.to_c()
        run_id = self.run_id.encode()
        s = Sim(self.protocol, self.p, d, h, int(self.sigma is not None),
                float(self.sigma or 0.0), _dp(spec), _dp(opt), self.init_kind,
                self.target_sq_err, self.init_scale, _dp(init), int(self.per_node_scope),
                int(self.poisson), self.rounds, self.events, self.rate_per_node,
                self.seed, run_id)
        s._keep = (spec, opt, init, h, run_id)
        return s


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(ORACLE_SO)
        _lib.dsgdo_derive_stream_seed.restype = C.c_uint64
        _lib.dsgdo_derive_stream_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint32, C.c_int]
        _lib.dsgdo_rng_next.restype = C.c_uint64
        _lib.dsgdo_uniform01.restype = C.c_double
        _lib.dsgdo_normal.restype = C.c_double
        _lib.dsgdo_exponential.restype = C.c_double
        _lib.dsgdo_exponential.argtypes = [C.c_void_p, C.c_double]
        _lib.dsgdo_uniform_index.restype = C.c_uint32
        _lib.dsgdo_uniform_index.argtypes = [C.c_void_p, C.c_uint32]
        _lib.dsgdo_step_size_at.restype = C.c_double
        _lib.dsgdo_step_size_at.argtypes = [C.POINTER(Hyper), C.c_uint64]
        _lib.dsgdo_pull_schedule.argtypes = [C.c_uint64, C.c_char_p, C.c_uint32, C.c_uint32,
                                             C.c_uint64, C.c_void_p]
        _lib.dsgdo_sigmoid.restype = C.c_double
        _lib.dsgdo_sigmoid.argtypes = [C.c_double]
        _lib.dsgdo_logistic_value.restype = C.c_double
        _lib.dsgdo_logistic_value.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                              C.c_double, C.c_void_p]
        _lib.dsgdo_draw_rows.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                         C.c_void_p]
        for sfx in ("f64", "f32"):
            getattr(_lib, f"dsgdo_logistic_grad_{sfx}").argtypes = [
                C.c_uint64, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_uint32,
                C.c_void_p, C.c_void_p]
            getattr(_lib, f"dsgdo_run_{sfx}").argtypes = [C.POINTER(Sim), C.c_void_p,
                                                         C.c_void_p, C.c_void_p, C.c_void_p]
            getattr(_lib, f"dsgdo_push_mix_{sfx}").restype = C.c_int
            getattr(_lib, f"dsgdo_push_gossip_round_{sfx}").restype = C.c_int
    return _lib


def ref_available() -> bool:
    try:
        build()
    except Exception:
        pass
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libdsgd_ref.so not built (needs /root/reference)")
        _ref = _configure_ref(C.CDLL(REF_SO))
    return _ref


@contextlib.contextmanager
def ref_library(path: str):
    """Temporarily route every ref_* helper to another build of the same
    shim, e.g. integration/_build/libdsgd_ref_b200_harness.so: the UNMODIFIED
    reference drivers with protocols.cpp replaced by the B200 binding."""
    global _ref
    old = _ref
    _ref = _configure_ref(C.CDLL(path))
    try:
        yield _ref
    finally:
        _ref = old


def _configure_ref(_ref):
    _ref.ref_last_error.restype = C.c_char_p
    _ref.ref_derive_stream_seed.restype = C.c_uint64
    _ref.ref_derive_stream_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint32, C.c_int]
    _ref.ref_stream_draws.argtypes = [C.c_uint64, C.c_int, C.c_uint32, C.c_uint64, C.c_void_p]
    _ref.ref_run.argtypes = [C.POINTER(Sim), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    _ref.ref_run_max_grad_norm.argtypes = [C.POINTER(Sim), C.c_void_p]
    if hasattr(_ref, "ref_run_resident"):  # the integration harness only
        _ref.ref_run_resident.argtypes = [C.POINTER(Sim), C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
    _ref.ref_run_transport.argtypes = [C.POINTER(Sim), C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_uint64]
    _ref.ref_round.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_char_p,
                               C.POINTER(Hyper), C.c_int, C.c_void_p, C.c_int,
                               C.c_uint32, C.c_uint32]
    _ref.ref_ring_allreduce.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.c_uint64]
    _ref.ref_set_logistic.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                      C.c_double, C.c_void_p, C.c_uint32]
    _ref.ref_logistic_grad.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                       C.c_uint64, C.c_uint64, C.c_void_p]
    _ref.ref_logistic_value.restype = C.c_double
    _ref.ref_logistic_value.argtypes = [C.c_void_p, C.c_uint64]
    _ref.ref_run_traced.restype = C.c_long
    _ref.ref_run_traced.argtypes = [C.POINTER(Sim), C.c_uint64, C.c_void_p, C.c_uint64,
                                    C.c_char_p, C.c_uint64]
    _ref.ref_time_rounds.restype = C.c_double
    _ref.ref_time_rounds.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                     C.POINTER(Hyper), C.c_int]
    if hasattr(_ref, "ref_time_rounds_sharded"):
        _ref.ref_time_rounds_sharded.restype = C.c_double
        _ref.ref_time_rounds_sharded.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_uint64,
                                                 C.c_int, C.POINTER(Hyper), C.c_int, C.c_uint32]
    return _ref


# --------------------------------------------------------------------------
# RNG (rng.hpp / rng.cpp restated)
class Stream:
    """A reference RngStream restated: mt19937_64 + samplers."""

    _SIZE = 312 * 8 + 8

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(self._SIZE)
        lib().dsgdo_rng_seed(self._buf, C.c_uint64(seed))

    @classmethod
    def make(cls, seed: int, run_id: str, node: int, purpose: str) -> "Stream":
        return cls(derive_stream_seed(seed, run_id, node, purpose))

    def next_u64(self) -> int:
        return lib().dsgdo_rng_next(self._buf)

    def uniform01(self) -> float:
        return lib().dsgdo_uniform01(self._buf)

    def normal(self) -> float:
        return lib().dsgdo_normal(self._buf)

    def normals(self, n: int, sigma: float = 1.0) -> np.ndarray:
        """sigma * normal(), n draws (NoiseModel::sample objectives.cpp:175-183)."""
        out = np.empty(n, dtype=np.float64)
        lib().dsgdo_fill_normal(self._buf, C.c_double(sigma), _ptr(out), C.c_uint64(n))
        return out

    def exponential(self, rate: float) -> float:
        return lib().dsgdo_exponential(self._buf, rate)

    def uniform_index(self, n: int) -> int:
        return lib().dsgdo_uniform_index(self._buf, n)

    def draw_rows(self, begin: int, end: int, batch: int) -> np.ndarray:
        """LogisticObjective minibatch rows (objectives.cpp:154-157)."""
        out = np.zeros(batch, dtype=np.uint64)
        lib().dsgdo_draw_rows(self._buf, begin, end, batch, _ptr(out))
        return out


def derive_stream_seed(seed: int, run_id: str, node: int, purpose: str) -> int:
    return lib().dsgdo_derive_stream_seed(seed, run_id.encode(), node, PURPOSE[purpose])


def step_size_at(h: HyperParams, t: int) -> float:
    hc = h.to_c()
    return lib().dsgdo_step_size_at(C.byref(hc), t)


def pull_schedule(seed: int, run_id: str, p: int, tau: int, rounds: int) -> np.ndarray:
    out = np.zeros((rounds, p), dtype=np.uint32)
    lib().dsgdo_pull_schedule(seed, run_id.encode(), p, tau, rounds, _ptr(out))
    return out


def noise_for_step(seed: int, run_id: str, node: int, sigma: float, d: int,
                   step: int = 0) -> np.ndarray:
    """Noise of node's `step`-th draw (NoiseModel::sample objectives.cpp:175-183)."""
    s = Stream.make(seed, run_id, node, "gradient-noise")
    for _ in range(step * d):
        s.normal()
    return sigma * s.normals(d)


# --------------------------------------------------------------------------
# Update rules on numpy arrays (fp64 or fp32 -- dtype picks the restatement)
def _sfx(dtype) -> str:
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _arr(a, dtype, shape=None):
    if a is None:
        return None
    x = np.ascontiguousarray(a, dtype=dtype)
    return x.reshape(shape) if shape is not None else x


class Nodes:
    """p nodes' state as flat numpy arrays (SoA), dtype float64 or float32."""

    def __init__(self, theta, dprev=None, t=None, dtype=np.float64):
        self.theta = np.array(theta, dtype=dtype, copy=True, ndmin=2)
        self.p, self.d = self.theta.shape
        self.dprev = (np.zeros_like(self.theta) if dprev is None
                      else np.array(dprev, dtype=dtype, copy=True).reshape(self.p, self.d))
        self.t = (np.zeros(self.p, dtype=np.uint64) if t is None
                  else np.array(t, dtype=np.uint64, copy=True).reshape(self.p))

    @property
    def dtype(self):
        return self.theta.dtype

    def copy(self) -> "Nodes":
        return Nodes(self.theta, self.dprev, self.t, self.dtype)


def _obj_args(nodes: Nodes, spec, opt, gfixed):
    dt = nodes.dtype
    if gfixed is not None:
        return OBJ_FIXED, None, None, _arr(gfixed, dt, (nodes.p, nodes.d))
    spec = _arr(spec, dt)
    opt = _arr(opt if opt is not None else np.zeros(nodes.d), dt)
    return OBJ_QUADRATIC, spec, opt, None


def local_sgd_step(nodes: Nodes, h: HyperParams, spec=None, opt=None, gfixed=None, noise=None):
    """local_sgd_step on every node (protocols.cpp:102-108)."""
    kind, s, o, g = _obj_args(nodes, spec, opt, gfixed)
    nz = _arr(noise, nodes.dtype, (nodes.p, nodes.d))
    hc = h.to_c()
    f = getattr(lib(), f"dsgdo_local_sgd_step_{_sfx(nodes.dtype)}")
    es = nodes.theta.itemsize
    for i in range(nodes.p):
        tp = nodes.t[i:i + 1]
        f(C.c_uint64(nodes.d), C.c_void_p(nodes.theta.ctypes.data + i * nodes.d * es),
          C.c_void_p(nodes.dprev.ctypes.data + i * nodes.d * es), _ptr(tp), C.c_int(kind),
          _ptr(s), _ptr(o),
          None if g is None else C.c_void_p(g.ctypes.data + i * nodes.d * es),
          None if nz is None else C.c_void_p(nz.ctypes.data + i * nodes.d * es), C.byref(hc))
        nodes.t[i] = tp[0]
    return nodes


def _round(name, nodes, h, spec, opt, gfixed, noise, *extra_pre, extra_post=()):
    kind, s, o, g = _obj_args(nodes, spec, opt, gfixed)
    nz = _arr(noise, nodes.dtype, (nodes.p, nodes.d))
    hc = h.to_c()
    f = getattr(lib(), f"dsgdo_{name}_{_sfx(nodes.dtype)}")
    rc = f(C.c_uint32(nodes.p), C.c_uint64(nodes.d), _ptr(nodes.theta), _ptr(nodes.dprev),
           _ptr(nodes.t), *extra_pre, C.c_int(kind), _ptr(s), _ptr(o), _ptr(g), _ptr(nz),
           C.byref(hc), *extra_post)
    return rc


def allreduce_round(nodes: Nodes, h, spec=None, opt=None, gfixed=None, noise=None,
                    per_node=False):
    _round("allreduce_round", nodes, h, spec, opt, gfixed, noise,
           extra_post=(C.c_int(int(per_node)), None))
    return nodes


def ea_round(nodes: Nodes, center: np.ndarray, gated: bool, h, spec=None, opt=None,
             gfixed=None, noise=None):
    """Synchronous EASGD sweep; `center` (d,) is updated in place."""
    assert center.dtype == nodes.dtype and center.flags.c_contiguous
    _round("ea_round", nodes, h, spec, opt, gfixed, noise, _ptr(center), C.c_int(int(gated)))
    return nodes


def pull_gossip_round(nodes: Nodes, partner, h, spec=None, opt=None, gfixed=None, noise=None):
    pm = np.ascontiguousarray(partner, dtype=np.uint32)
    _round("pull_gossip_round", nodes, h, spec, opt, gfixed, noise, _ptr(pm))
    return nodes


def push_gossip_round(nodes: Nodes, target, h, spec=None, opt=None, gfixed=None, noise=None):
    pm = np.ascontiguousarray(target, dtype=np.uint32)
    if _round("push_gossip_round", nodes, h, spec, opt, gfixed, noise, _ptr(pm)) != 0:
        raise ValueError("push target must differ from sender")
    return nodes


def stale_round(nodes: Nodes, partner, h, spec=None, opt=None, gfixed=None, noise=None):
    pm = np.ascontiguousarray(partner, dtype=np.uint32)
    _round("stale_round", nodes, h, spec, opt, gfixed, noise, _ptr(pm))
    return nodes


def fresh_round(nodes: Nodes, partner, h, spec=None, opt=None, gfixed=None, noise=None):
    pm = np.ascontiguousarray(partner, dtype=np.uint32)
    _round("fresh_round", nodes, h, spec, opt, gfixed, noise, _ptr(pm))
    return nodes


def async_pull_event(nodes: Nodes, i: int, j: int, h, spec=None, opt=None, gfixed=None,
                     noise=None):
    kind, s, o, g = _obj_args(nodes, spec, opt, gfixed)
    nz = _arr(noise, nodes.dtype, (nodes.p, nodes.d))
    hc = h.to_c()
    f = getattr(lib(), f"dsgdo_async_pull_event_{_sfx(nodes.dtype)}")
    f(C.c_uint32(nodes.p), C.c_uint64(nodes.d), _ptr(nodes.theta), _ptr(nodes.t),
      C.c_uint32(i), C.c_uint32(j), C.c_int(kind), _ptr(s), _ptr(o), _ptr(g), _ptr(nz),
      C.byref(hc))
    return nodes


def pull_mix(theta: np.ndarray, partner) -> np.ndarray:
    x = np.array(theta, copy=True)
    pm = np.ascontiguousarray(partner, dtype=np.uint32)
    getattr(lib(), f"dsgdo_pull_mix_{_sfx(x.dtype)}")(
        C.c_uint32(x.shape[0]), C.c_uint64(x.shape[1]), _ptr(x), _ptr(pm))
    return x


def push_mix(theta: np.ndarray, target) -> np.ndarray:
    x = np.array(theta, copy=True)
    pm = np.ascontiguousarray(target, dtype=np.uint32)
    rc = getattr(lib(), f"dsgdo_push_mix_{_sfx(x.dtype)}")(
        C.c_uint32(x.shape[0]), C.c_uint64(x.shape[1]), _ptr(x), _ptr(pm))
    if rc != 0:
        raise ValueError("push target must differ from sender")
    return x


def spatial_mean(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    out = np.zeros(x.shape[1], dtype=x.dtype)
    getattr(lib(), f"dsgdo_spatial_mean_{_sfx(x.dtype)}")(
        C.c_uint32(x.shape[0]), C.c_uint64(x.shape[1]), _ptr(x), _ptr(out))
    return out


def ring_allreduce(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    out = np.zeros_like(x)
    getattr(lib(), f"dsgdo_ring_allreduce_{_sfx(x.dtype)}")(
        C.c_uint32(x.shape[0]), C.c_uint64(x.shape[1]), _ptr(x), _ptr(out))
    return out


def trace(theta: np.ndarray, spec, opt=None):
    theta = np.ascontiguousarray(theta)
    p, d = theta.shape
    spec = _arr(spec, theta.dtype)
    opt = _arr(opt if opt is not None else np.zeros(d), theta.dtype)
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    getattr(lib(), f"dsgdo_trace_{_sfx(theta.dtype)}")(
        C.c_uint32(p), C.c_uint64(d), _ptr(theta), _ptr(spec), _ptr(opt),
        C.byref(a), C.byref(b), C.byref(c))
    return {"sq_err_consensus": a.value, "loss_mean": b.value, "sq_err_opt": c.value}


def run(cfg: SimConfig, dtype=np.float64):
    """run_sync / run_async restated; returns (theta[p,d], dprev[p,d], t[p], center[d])."""
    p, d = cfg.p, cfg.d
    theta = np.zeros((p, d), dtype=dtype)
    dprev = np.zeros((p, d), dtype=dtype)
    t = np.zeros(p, dtype=np.uint64)
    center = np.zeros(d, dtype=dtype)
    s = cfg.to_c()
    rc = getattr(lib(), f"dsgdo_run_{_sfx(dtype)}")(C.byref(s), _ptr(theta), _ptr(dprev),
                                                      _ptr(t), _ptr(center))
    if rc != 0:
        raise ValueError("invalid oracle configuration")
    return theta, dprev, t, center


def sigmoid(z: float) -> float:
    """objectives.cpp:34-38"""
    return lib().dsgdo_sigmoid(z)


def logistic_grad(X: np.ndarray, y, l2: float, theta: np.ndarray, rows) -> np.ndarray:
    """LogisticObjective::stochastic_gradient (objectives.cpp:147-162) restated
    for given minibatch rows; dtype of X/theta picks fp64 or the fp32 policy."""
    X = np.ascontiguousarray(X)
    theta = np.ascontiguousarray(theta, dtype=X.dtype)
    y = np.ascontiguousarray(y, dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.zeros(X.shape[1], dtype=X.dtype)
    getattr(lib(), f"dsgdo_logistic_grad_{_sfx(X.dtype)}")(
        C.c_uint64(X.shape[1]), _ptr(X), _ptr(y), C.c_double(l2), _ptr(theta),
        C.c_uint32(len(rows)), _ptr(rows), _ptr(out))
    return out


def logistic_value(X, y, l2: float, theta) -> float:
    """LogisticObjective::value (objectives.cpp:116-125), fp64."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    return lib().dsgdo_logistic_value(X.shape[0], X.shape[1], _ptr(X), _ptr(y), l2, _ptr(theta))


def ref_logistic_value(theta) -> float:
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    return ref().ref_logistic_value(_ptr(theta), len(theta))


# --------------------------------------------------------------------------
# The compiled reference (oracle/_ref)
def ref_set_logistic(X, y, l2: float, ranges=None):
    """Install a LogisticObjective dataset for ref_round(obj='logistic') and
    ref_run (node i samples rows ranges[i]); ref_set_logistic(None, ...) clears."""
    if X is None:
        ref().ref_clear_logistic()
        return
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    rg = None if ranges is None else np.ascontiguousarray(ranges, dtype=np.uint64).reshape(-1)
    _ref_check(ref().ref_set_logistic(_ptr(X), _ptr(y), X.shape[0], X.shape[1], l2, _ptr(rg),
                                      0 if rg is None else len(rg) // 2))


def ref_logistic_grad(theta, batch: int, sample_seed: int, begin: int, end: int) -> np.ndarray:
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    out = np.zeros_like(theta)
    _ref_check(ref().ref_logistic_grad(_ptr(theta), len(theta), batch, sample_seed, begin, end,
                                       _ptr(out)))
    return out


def _ref_check(rc):
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())


def ref_run(cfg: SimConfig, transport: bool = False, chaos_seed: int = 0):
    p, d = cfg.p, cfg.d
    theta = np.zeros((p, d))
    dprev = np.zeros((p, d))
    t = np.zeros(p, dtype=np.uint64)
    center = np.zeros(d)
    s = cfg.to_c()
    if transport:
        _ref_check(ref().ref_run_transport(C.byref(s), _ptr(theta), _ptr(dprev), _ptr(t),
                                           _ptr(center), chaos_seed))
    else:
        _ref_check(ref().ref_run(C.byref(s), _ptr(theta), _ptr(dprev), _ptr(t), _ptr(center)))
    return theta, dprev, t, center


def ref_run_max_grad_norm(cfg: SimConfig) -> float:
    """RunResult::max_grad_norm of the reference's run_simulation."""
    out = C.c_double(0.0)
    s = cfg.to_c()
    _ref_check(ref().ref_run_max_grad_norm(C.byref(s), C.byref(out)))
    return out.value


def ref_run_resident(cfg: SimConfig):
    """integration/run_sync_b200.cpp through the harness (ref_library):
    (theta, dprev, t, center, max_grad_norm)."""
    p, d = cfg.p, cfg.d
    theta, dprev = np.zeros((p, d)), np.zeros((p, d))
    t, center = np.zeros(p, dtype=np.uint64), np.zeros(d)
    gn = C.c_double(0.0)
    s = cfg.to_c()
    _ref_check(ref().ref_run_resident(C.byref(s), _ptr(theta), _ptr(dprev), _ptr(t),
                                      _ptr(center), C.byref(gn)))
    return theta, dprev, t, center, gn.value


def ref_run_traced(cfg: SimConfig, trace_every: int, max_records: int = 4096):
    """run_simulation with trace_every: records [n, 6] = (t, sim_time,
    sq_err_opt, sq_err_consensus, loss_mean, alpha), NaN for an absent
    optional, and the reference's own JSONL text (trace_io.cpp) when built."""
    rec = np.zeros((max_records, 6))
    buf = C.create_string_buffer(1 << 20)
    s = cfg.to_c()
    n = ref().ref_run_traced(C.byref(s), trace_every, _ptr(rec), max_records, buf, len(buf))
    if n < 0:
        raise ValueError(ref().ref_last_error().decode())
    return rec[:n], buf.value.decode()


REF_ROUND = {"allreduce": 0, "ea": 1, "pull": 2, "push": 3, "stale": 4, "fresh": 5,
             "async": 6, "local": 7, "pull_mix": 8, "push_mix": 9}


def ref_round(kind: str, nodes: Nodes, h: HyperParams, partner=None, spec=None, opt=None,
              gfixed=None, sigma=None, seed=1, run_id="test", per_node=False, center=None,
              gated=True, i=0, j=0):
    """One reference round from explicit state (streams fresh from (seed, run_id))."""
    assert nodes.dtype == np.float64
    kind_id = REF_ROUND[kind]
    if isinstance(spec, str) and spec == "logistic":  # the dataset of ref_set_logistic
        okind, s, o, g = 2, None, None, None
    else:
        okind, s, o, g = _obj_args(nodes, spec, opt, gfixed)
    pm = None if partner is None else np.ascontiguousarray(partner, dtype=np.uint32)
    hc = h.to_c()
    _ref_check(ref().ref_round(kind_id, nodes.p, nodes.d, _ptr(nodes.theta), _ptr(nodes.dprev),
                               _ptr(nodes.t), _ptr(pm), okind, _ptr(s), _ptr(o), _ptr(g),
                               int(sigma is not None), float(sigma or 0.0), seed,
                               run_id.encode(), C.byref(hc), int(per_node), _ptr(center),
                               int(gated), i, j))
    return nodes


def ref_ring_allreduce(x: np.ndarray, chaos_seed: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    _ref_check(ref().ref_ring_allreduce(x.shape[0], x.shape[1], _ptr(x), _ptr(out), chaos_seed))
    return out


def ref_stream(seed: int, kind: int, count: int, n: int = 0):
    out = np.zeros(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    ref().ref_stream_draws(seed, kind, n, count, _ptr(out))
    return out


def ref_time_rounds(protocol: int, p: int, d: int, rounds: int, threaded: bool,
                    h: HyperParams, grad: str = "quadratic", shards: int = 1) -> float:
    """Seconds for `rounds` rounds of the compiled reference (simulator
    rules on 1 thread, or run_transport's threads); grad: 'quadratic'
    (QuadraticObjective(1, 0)) or 'pool' (4 synthetic N(0,1) gradient
    vectors through the Objective plugin slot, served in turn).  shards > 1:
    d split into coordinate ranges, one independent reference run per shard
    on its own thread(s), all concurrently (ref_time_rounds_sharded)."""
    hc = h.to_c()
    gk = {"quadratic": 0, "pool": 1}[grad]
    if shards > 1:
        sec = ref().ref_time_rounds_sharded(protocol, p, d, rounds, int(threaded), C.byref(hc),
                                            gk, shards)
    else:
        sec = ref().ref_time_rounds(protocol, p, d, rounds, int(threaded), C.byref(hc), gk)
    if sec < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return sec


def run_transport_allreduce(cfg: SimConfig, dtype=np.float64) -> "Nodes":
    """run_transport's all-reduce worker loop (transport.cpp:350-360) restated
    with the oracle primitives: per node compute_local_delta, ring_allreduce
    mean (transport.cpp:183-248, fixed chunking and fold order), theta +=
    avg, delta_prev = aggregate ? avg : own.  Offset-ones init only.
    Pinned against the compiled reference by tests/test_oracle_golden.py."""
    p, d = cfg.p, cfg.d
    if cfg.init_kind != INIT_OFFSET_ONES:
        raise ValueError("offset-ones init only")
    opt = np.zeros(d) if cfg.opt is None else np.asarray(cfg.opt, dtype=np.float64)
    c = np.sqrt(cfg.target_sq_err / (p * d))
    n = Nodes(np.tile(opt + c, (p, 1)).astype(dtype), dtype=dtype)
    streams = [Stream.make(cfg.seed, cfg.run_id, i, "gradient-noise") for i in range(p)]
    for _ in range(cfg.rounds):
        noise = None
        if cfg.sigma is not None:
            noise = np.array([s.normals(d, cfg.sigma) for s in streams]).astype(dtype)
        deltas = np.zeros((p, d), dtype=dtype)
        for i in range(p):
            m = Nodes(n.theta[i:i + 1], n.dprev[i:i + 1], n.t[i:i + 1], dtype=dtype)
            local_sgd_step(m, cfg.hyper, spec=cfg.spectrum, opt=opt,
                           noise=None if noise is None else noise[i:i + 1])
            deltas[i] = m.dprev[0]
        avg = ring_allreduce(deltas)
        n.theta = (n.theta + avg).astype(dtype)
        n.dprev = deltas.copy() if cfg.per_node_scope else avg.copy()
        n.t += 1
    return n


# --------------------------------------------------------------------------
# LogisticObjective run_sync restated (pull-gossip and all-reduce), composed
# from the primitives above exactly as simulator.cpp:234-369 drives them:
# per round, every node draws its minibatch rows from its sample stream and
# its noise from its noise stream; pull rounds mix first and take the
# gradient at the mixed point (protocols.cpp:173-185).
def logistic_run(cfg: SimConfig, X, y, l2: float, ranges, dtype=np.float64):
    """Returns (theta[p,d], dprev[p,d], t[p]) for cfg.protocol in {PULL,
    ALLREDUCE} with the gaussian-spread or zeros init."""
    p, d = cfg.p, X.shape[1]
    f = np.dtype(dtype).type
    Xf = np.ascontiguousarray(X, dtype=dtype)
    y = np.ascontiguousarray(y, dtype=np.int32)
    base = np.zeros(d)
    th = np.tile(base, (p, 1))
    if cfg.init_kind == INIT_GAUSSIAN:  # simulator.cpp:196-205
        for i in range(p):
            s = Stream.make(cfg.seed, cfg.run_id, i, "init")
            th[i] = base + cfg.init_scale * s.normals(d)
    elif cfg.init_kind != INIT_ZEROS:
        raise ValueError("gaussian-spread or zeros init only")
    n = Nodes(th.astype(dtype), dtype=dtype)
    sample = [Stream.make(cfg.seed, cfg.run_id, i, "sample") for i in range(p)]
    noise_s = [Stream.make(cfg.seed, cfg.run_id, i, "gradient-noise") for i in range(p)]
    partner_s = [Stream.make(cfg.seed, cfg.run_id, i, "partner-choice") for i in range(p)]
    h = cfg.hyper
    mu = f(h.mu)

    def point(theta, dprev):
        if h.mu == 0.0:
            return theta.copy()
        return (theta + (mu * dprev).astype(dtype)).astype(dtype)

    def grads(theta, dprev):
        pts = point(theta, dprev)
        return np.stack([logistic_grad(Xf, y, l2, pts[i],
                                       sample[i].draw_rows(int(ranges[i][0]), int(ranges[i][1]),
                                                           h.batch)) for i in range(p)])

    for r in range(cfg.rounds):
        gated = r > 0 and r % h.tau == 0
        noise = None  # NoiseModel::sample per node, after its rows (own stream)
        if cfg.protocol == PULL and gated:
            partners = np.array([partner_s[i].uniform_index(p) for i in range(p)], dtype=np.uint32)
            mixed = pull_mix(n.theta, partners)
            G = grads(mixed, n.dprev)
            if cfg.sigma is not None:
                noise = np.stack([cfg.sigma * noise_s[i].normals(d) for i in range(p)]).astype(dtype)
            n = Nodes(mixed, n.dprev, n.t, dtype=dtype)
            local_sgd_step(n, h, gfixed=G, noise=noise)
        elif cfg.protocol == ALLREDUCE:
            G = grads(n.theta, n.dprev)
            if cfg.sigma is not None:
                noise = np.stack([cfg.sigma * noise_s[i].normals(d) for i in range(p)]).astype(dtype)
            allreduce_round(n, h, gfixed=G, noise=noise, per_node=cfg.per_node_scope)
        elif cfg.protocol == PULL:
            G = grads(n.theta, n.dprev)
            if cfg.sigma is not None:
                noise = np.stack([cfg.sigma * noise_s[i].normals(d) for i in range(p)]).astype(dtype)
            local_sgd_step(n, h, gfixed=G, noise=noise)
        else:
            raise ValueError("pull-gossip or all-reduce only")
    return n.theta, n.dprev, n.t
