"""Device-resident worker groups over the C ABI (include/dsgd_b200.h).

``Group`` is one process's context on one GPU hosting ``n_local`` nodes
(workers).  Two shapes are supported, exactly as the C ABI:

* all ``p`` nodes on one GPU (``Group(d, p)``) -- the single-process
  simulator's shape (simulator.cpp run_sync) with every round one fused
  kernel;
* one node per GPU, one process per GPU (``Group.distributed(...)``) --
  the threaded transport's shape (transport.cpp run_transport) with NVLink
  peer memory (CUDA IPC) for gossip / EASGD and NCCL for the all-reduce.

Hyperparameters, partner maps and gate bits are host data, exactly as in the
reference's update-rule interface (protocols.hpp:45-152).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N

DTYPES = {"f32": N.F32, "f64": N.F64, np.float32: N.F32, np.float64: N.F64}
NP_OF = {N.F32: np.float32, N.F64: np.float64}


@dataclass
class Hyperparams:
    """dsgd::Hyperparams (core.hpp:54-70); defaults are the reference regime."""
    alpha0: float = 0.1
    anneal_factor: float = 0.1
    anneal_at: Sequence[int] = (150000, 300000)
    mu: float = 0.9
    weight_decay: float = 1e-4
    beta_gossip: float = 0.5
    beta_ea: float = 0.1
    tau: int = 1
    batch: int = 1

    def to_c(self) -> N.Hyper:
        arr = (C.c_uint64 * max(1, len(self.anneal_at)))(*self.anneal_at)
        h = N.Hyper(self.alpha0, self.anneal_factor, arr, len(self.anneal_at), self.mu,
                    self.weight_decay, self.beta_gossip, self.beta_ea, self.tau, self.batch)
        h._keep = arr
        return h

    def validate(self) -> None:
        """Hyperparams::validate core.cpp:62-80 (raises InvalidArgument)."""
        hc = self.to_c()
        N.check(N.load().dsgd_hyperparams_validate(C.byref(hc)))


def step_size_at(h: Hyperparams, t: int) -> float:
    hc = h.to_c()
    return N.load().dsgd_step_size_at(C.byref(hc), t)


class Stream:
    """dsgd::RngStream (rng.hpp:50-85), held natively (std::mt19937_64)."""

    def __init__(self, engine_seed: Optional[int] = None, _handle=None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            N.check(N.load().dsgd_stream_create(C.c_uint64(engine_seed or 0), C.byref(self._h)))

    @classmethod
    def make(cls, seed: int, run_id: str, node: int, purpose: str) -> "Stream":
        h = C.c_void_p()
        N.check(N.load().dsgd_stream_make(seed, run_id.encode(), node, N.PURPOSE[purpose],
                                          C.byref(h)))
        return cls(_handle=h)

    def clone(self) -> "Stream":
        h = C.c_void_p()
        N.check(N.load().dsgd_stream_clone(self._h, C.byref(h)))
        return Stream(_handle=h)

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.dsgd_stream_destroy(self._h)
            self._h = None

    def next_u64(self) -> int:
        return N.load().dsgd_stream_next_u64(self._h)

    def uniform01(self) -> float:
        return N.load().dsgd_stream_uniform01(self._h)

    def normal(self) -> float:
        return N.load().dsgd_stream_normal(self._h)

    def uniform_index(self, n: int) -> int:
        out = C.c_uint32()
        N.check(N.load().dsgd_stream_uniform_index(self._h, n, C.byref(out)))
        return out.value

    def exponential(self, rate: float) -> float:
        out = C.c_double()
        N.check(N.load().dsgd_stream_exponential(self._h, rate, C.byref(out)))
        return out.value

    def fill_normal(self, sigma: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        N.load().dsgd_stream_fill_normal(self._h, sigma, out.ctypes.data, n)
        return out


def derive_stream_seed(seed: int, run_id: str, node: int, purpose: str) -> int:
    return N.load().dsgd_derive_stream_seed(seed, run_id.encode(), node, N.PURPOSE[purpose])


def draw_pull_partners(streams: Sequence[Stream]) -> np.ndarray:
    p = len(streams)
    arr = (C.c_void_p * p)(*[s._h.value for s in streams])
    out = np.zeros(p, dtype=np.uint32)
    N.check(N.load().dsgd_draw_pull_partners(arr, p, out.ctypes.data_as(N._U32P)))
    return out


def draw_push_targets(streams: Sequence[Stream]) -> np.ndarray:
    p = len(streams)
    arr = (C.c_void_p * p)(*[s._h.value for s in streams])
    out = np.zeros(p, dtype=np.uint32)
    N.check(N.load().dsgd_draw_push_targets(arr, p, out.ctypes.data_as(N._U32P)))
    return out


def _u32(a) -> tuple:
    arr = np.ascontiguousarray(a, dtype=np.uint32)
    return arr, arr.ctypes.data_as(N._U32P)


class Group:
    """One context (one GPU) hosting ``n_local`` of the group's ``p`` nodes."""

    def __init__(self, d: int, p: int = 1, dtype="f32", device: int = 0, first_node: int = 0,
                 n_local: Optional[int] = None, quadratic: bool = False, grad: bool = False,
                 noise: bool = False, center: bool = False, stream: Optional[int] = None):
        self.lib = N.load()
        self.d, self.p = int(d), int(p)
        self.dtype = DTYPES[dtype]
        self.np_dtype = NP_OF[self.dtype]
        self.first = first_node
        self.n_local = p if n_local is None else n_local
        flags = ((N.CTX_QUADRATIC if quadratic else 0) | (N.CTX_GRAD if grad else 0) |
                 (N.CTX_NOISE if noise else 0) | (N.CTX_CENTER if center else 0))
        self.flags = flags
        desc = N.CtxDesc(device, self.d, self.dtype, self.p, first_node, self.n_local, flags,
                         stream)
        self._ctx = C.c_void_p()
        N.check(self.lib.dsgd_ctx_create(C.byref(desc), C.byref(self._ctx)))
        self.device = device
        self._norm = C.c_double(0.0)

    @classmethod
    def inproc(cls, d: int, p: int, dtype="f32", devices: Optional[Sequence[int]] = None,
               device: int = 0, quadratic: bool = False, grad: bool = False,
               noise: bool = False, center: bool = False) -> list:
        """dsgd_group_create_inproc: p one-node contexts of this process wired
        by raw device pointers (rank r on devices[r], or all on `device`).
        Drive them in node order every round (``run_rounds_inproc`` does)."""
        lib = N.load()
        flags = ((N.CTX_QUADRATIC if quadratic else 0) | (N.CTX_GRAD if grad else 0) |
                 (N.CTX_NOISE if noise else 0) | (N.CTX_CENTER if center else 0))
        desc = N.CtxDesc(device, int(d), DTYPES[dtype], p, 0, 1, flags, None)
        out = (C.c_void_p * p)()
        devs = (C.c_int * p)(*(devices if devices is not None else [device] * p))
        N.check(lib.dsgd_group_create_inproc(C.byref(desc), p, devs, out))
        groups = []
        for r in range(p):
            g = cls.__new__(cls)
            g.lib = lib
            g.d, g.p = int(d), int(p)
            g.dtype = DTYPES[dtype]
            g.np_dtype = NP_OF[g.dtype]
            g.first, g.n_local, g.flags = r, 1, flags
            g.device = devs[r]
            g._ctx = C.c_void_p(out[r])
            g._norm = C.c_double(0.0)
            groups.append(g)
        return groups

    # ------------------------------------------------------------ lifetime
    def close(self) -> None:
        if self._ctx:
            self.lib.dsgd_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._ctx

    def stream(self) -> int:
        s = C.c_void_p()
        N.check(self.lib.dsgd_ctx_stream(self._ctx, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        N.check(self.lib.dsgd_ctx_sync(self._ctx))

    # --------------------------------------------------------------- state
    def buffer_ptr(self, local: int, which: int) -> int:
        p = C.c_void_p()
        N.check(self.lib.dsgd_buffer_ptr(self._ctx, local, which, C.byref(p)))
        return p.value

    def set_state(self, local: int, theta, delta=None, t: int = 0) -> None:
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(self.d)
        dp = None if delta is None else np.ascontiguousarray(delta, dtype=np.float64).reshape(self.d)
        N.check(self.lib.dsgd_set_state(self._ctx, local, th.ctypes.data,
                                        None if dp is None else dp.ctypes.data, t))

    def get_state(self, local: int):
        th = np.empty(self.d)
        dp = np.empty(self.d)
        t = C.c_uint64()
        N.check(self.lib.dsgd_get_state(self._ctx, local, th.ctypes.data, dp.ctypes.data,
                                        C.byref(t)))
        return th, dp, t.value

    def set_vector(self, local: int, which: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(self.d)
        N.check(self.lib.dsgd_set_vector(self._ctx, local, which, v.ctypes.data))

    def get_vector(self, local: int, which: int) -> np.ndarray:
        v = np.empty(self.d)
        N.check(self.lib.dsgd_get_vector(self._ctx, local, which, v.ctypes.data))
        return v

    def set_quadratic(self, spectrum, opt=None) -> None:
        self.set_vector(0, N.BUF_SPECTRUM, spectrum)
        self.set_vector(0, N.BUF_OPT, np.zeros(self.d) if opt is None else opt)

    def set_center(self, c) -> None:
        self.set_vector(0, N.BUF_CENTER, c)

    def get_center(self) -> np.ndarray:
        return self.get_vector(0, N.BUF_CENTER)

    def set_t(self, local: int, t: int) -> None:
        N.check(self.lib.dsgd_set_t(self._ctx, local, t))

    def get_t(self, local: int) -> int:
        t = C.c_uint64()
        N.check(self.lib.dsgd_get_t(self._ctx, local, C.byref(t)))
        return t.value

    def upload_async(self, local: int, which: int, host_ptr: int, count: int) -> None:
        N.check(self.lib.dsgd_upload_async(self._ctx, local, which, host_ptr, count))

    def copy_in_async(self, local: int, which: int, src_ptr: int, count: int) -> None:
        N.check(self.lib.dsgd_copy_in_async(self._ctx, local, which, src_ptr, count))

    def download_async(self, local: int, which: int, host_ptr: int, count: int) -> None:
        N.check(self.lib.dsgd_download_async(self._ctx, local, which, host_ptr, count))

    # -------------------------------------------------------- update rules
    def set_logistic(self, features, labels, l2: float) -> None:
        """LogisticObjective(features, labels, l2) (objectives.cpp:80-106) on
        this context; use grad='logistic' in the rules."""
        X = np.ascontiguousarray(features, dtype=np.float64)
        if X.ndim != 2 or (X.shape[0] and X.shape[1] != self.d):
            raise ValueError("logistic feature rows have inconsistent width")
        y = np.ascontiguousarray(labels, dtype=np.int32)
        if len(y) != X.shape[0]:
            raise ValueError("logistic features/labels size mismatch")
        N.check(self.lib.dsgd_set_logistic(self._ctx, X.ctypes.data if X.size else None,
                                           y.ctypes.data if y.size else None, X.shape[0], l2))

    def logistic_set_sample_range(self, local: int, begin: int, end: int) -> None:
        N.check(self.lib.dsgd_logistic_set_sample_range(self._ctx, local, begin, end))

    def _grad(self, grad, noise, grad_norm: bool, rows=None):
        """grad: None -> quadratic objective if present else the context's
        gradient buffers; 'quadratic'; 'logistic' (the dataset of
        set_logistic; rows = n_local x batch minibatch rows, or None to draw
        them from the nodes' sample streams); or a list of device pointers.
        noise: False (zero noise), True (the context's noise buffers) or
        ('device', sigma, seed) for Philox noise drawn inside the kernel."""
        keep = None
        if grad is None:
            src = N.GRAD_QUADRATIC if self.flags & N.CTX_QUADRATIC else N.GRAD_BUFFER
            ptr = None
        elif isinstance(grad, str):
            src, ptr = {"quadratic": N.GRAD_QUADRATIC, "buffer": N.GRAD_BUFFER,
                        "logistic": N.GRAD_LOGISTIC}[grad], None
        else:
            keep = (C.c_void_p * len(grad))(*grad)
            src, ptr = N.GRAD_BUFFER, C.cast(keep, C.POINTER(C.c_void_p))
        mode, sigma, seed = 0, 0.0, 0
        if isinstance(noise, tuple):
            mode, sigma, seed = 2, float(noise[1]), int(noise[2])
        elif noise:
            mode = 1
        rp = None
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.uint64)
            rp = rows.ctypes.data_as(C.POINTER(C.c_uint64))
        gs = N.GradSpec(src, ptr, mode, C.pointer(self._norm) if grad_norm else None,
                        sigma, seed, rp)
        gs._keep = (keep, rows)
        return gs

    def _run(self, fn, *args, grad=None, noise=False, grad_norm=False, rows=None):
        self._norm.value = 0.0
        gs = self._grad(grad, noise, grad_norm, rows)
        N.check(fn(self._ctx, *args[:1], C.byref(gs), *args[1:]))
        if not grad_norm:
            return None
        # the library raises grad_norm_out lazily (no per-round host wait)
        N.check(self.lib.dsgd_grad_norm_flush(self._ctx))
        return self._norm.value

    def local_sgd_step(self, h: Hyperparams, **kw):
        hc = h.to_c()
        return self._run(self.lib.dsgd_local_sgd_step, C.byref(hc), **kw)

    def allreduce_round(self, h: Hyperparams, scope: str = "aggregate", **kw):
        hc = h.to_c()
        sc = N.SCOPE_PER_NODE if scope == "per-node" else N.SCOPE_AGGREGATE
        return self._run(self.lib.dsgd_allreduce_round, C.byref(hc), sc, **kw)

    def ea_round(self, h: Hyperparams, gated: bool = True, **kw):
        hc = h.to_c()
        return self._run(self.lib.dsgd_ea_round, C.byref(hc), int(gated), **kw)

    def pull_gossip_round(self, h: Hyperparams, partner_of=None, **kw):
        hc = h.to_c()
        if partner_of is None:
            return self._run(self.lib.dsgd_pull_gossip_round, C.byref(hc), None, **kw)
        arr, ptr = _u32(partner_of)
        return self._run(self.lib.dsgd_pull_gossip_round, C.byref(hc), ptr, **kw)

    def push_gossip_round(self, h: Hyperparams, target_of, **kw):
        hc = h.to_c()
        arr, ptr = _u32(target_of)
        return self._run(self.lib.dsgd_push_gossip_round, C.byref(hc), ptr, **kw)

    def gossip_stale_round(self, h: Hyperparams, partner_of, **kw):
        hc = h.to_c()
        arr, ptr = _u32(partner_of)
        return self._run(self.lib.dsgd_gossip_stale_round, C.byref(hc), ptr, **kw)

    def gossip_fresh_round(self, h: Hyperparams, partner_of, **kw):
        hc = h.to_c()
        arr, ptr = _u32(partner_of)
        return self._run(self.lib.dsgd_gossip_fresh_round, C.byref(hc), ptr, **kw)

    def async_pull_event(self, h: Hyperparams, i: int, j: int, **kw):
        hc = h.to_c()
        return self._run(self.lib.dsgd_async_pull_event, C.byref(hc), i, j, **kw)

    def eval_point(self, h: Hyperparams, local: int, out_ptr: int) -> None:
        """dsgd_eval_point: theta + mu * delta_prev of one node into a device buffer."""
        hc = h.to_c()
        N.check(self.lib.dsgd_eval_point(self._ctx, C.byref(hc), local, out_ptr))

    def pull_mix(self, partner_of) -> None:
        arr, ptr = _u32(partner_of)
        N.check(self.lib.dsgd_pull_mix(self._ctx, ptr))

    def push_mix(self, target_of) -> None:
        arr, ptr = _u32(target_of)
        N.check(self.lib.dsgd_push_mix(self._ctx, ptr))

    def gossip_fresh_mix(self, partner_of, beta: float) -> None:
        arr, ptr = _u32(partner_of)
        N.check(self.lib.dsgd_gossip_fresh_mix(self._ctx, ptr, beta))

    def ea_init_center(self) -> None:
        N.check(self.lib.dsgd_ea_init_center(self._ctx))

    def ea_client_event(self, h: Hyperparams, i: int, gated: bool, **kw):
        """One asynchronous EASGD client tick (run_async simulator.cpp:419-428)."""
        hc = h.to_c()
        return self._run(self.lib.dsgd_ea_client_event, C.byref(hc), i, int(gated), **kw)

    def trace(self) -> dict:
        """make_trace_record (simulator.cpp:92-123) on the device."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        N.check(self.lib.dsgd_trace(self._ctx, C.byref(a), C.byref(b), C.byref(c)))
        return {"sq_err_consensus": a.value, "loss_mean": b.value, "sq_err_opt": c.value}

    def ea_set_update_out(self, ptrs) -> None:
        if ptrs is None:
            N.check(self.lib.dsgd_ea_set_update_out(self._ctx, None))
            return
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        N.check(self.lib.dsgd_ea_set_update_out(self._ctx, arr))

    def ea_server_apply(self, update_dev_ptr: int) -> None:
        N.check(self.lib.dsgd_ea_server_apply(self._ctx, update_dev_ptr))

    # --------------------------------------------------------- worker loop
    def seed_streams(self, seed: int, run_id: str) -> None:
        N.check(self.lib.dsgd_ctx_seed_streams(self._ctx, seed, run_id.encode()))

    def run_rounds(self, protocol: int, h: Hyperparams, rounds: int, scope: str = "aggregate",
                   grad=None, grad_pool: Optional[Sequence[int]] = None,
                   host_noise_sigma: float = 0.0, noise: bool = False,
                   grad_norm: bool = False):
        """run_sync's round loop (simulator.cpp:234-369) on this context;
        grad_norm: also track max ||g|| like run_sync's &result.max_grad_norm
        (device-side, read once at the end) and return it."""
        self._norm.value = 0.0
        gs = self._grad(grad, noise, grad_norm)
        pool = None
        if grad_pool:
            pool = (C.c_void_p * len(grad_pool))(*grad_pool)
        rd = N.RunDesc(protocol, h.to_c(), N.SCOPE_PER_NODE if scope == "per-node"
                       else N.SCOPE_AGGREGATE, gs,
                       (len(grad_pool) // self.n_local) if grad_pool else 0,
                       C.cast(pool, C.POINTER(C.c_void_p)) if pool else None,
                       host_noise_sigma, rounds)
        rd._keep = (gs, pool)
        N.check(self.lib.dsgd_run_rounds(self._ctx, C.byref(rd)))
        return self._norm.value if grad_norm else None

    def _run_desc(self, protocol: int, h: Hyperparams, rounds: int, scope: str, grad,
                  grad_pool, host_noise_sigma: float, noise: bool):
        gs = self._grad(grad, noise, False)
        pool = None
        if grad_pool:
            pool = (C.c_void_p * len(grad_pool))(*grad_pool)
        rd = N.RunDesc(protocol, h.to_c(), N.SCOPE_PER_NODE if scope == "per-node"
                       else N.SCOPE_AGGREGATE, gs,
                       (len(grad_pool) // self.n_local) if grad_pool else 0,
                       C.cast(pool, C.POINTER(C.c_void_p)) if pool else None,
                       host_noise_sigma, rounds)
        rd._keep = (gs, pool)
        return rd

    def run_events(self, protocol: int, h: Hyperparams, events: int, rate_per_node: float,
                   grad=None, host_noise_sigma: float = 0.0, sim_time: float = 0.0,
                   alpha: float = 0.0):
        """run_async's event loop (simulator.cpp:380-449) on this context:
        returns (accumulated sim_time, alpha of the last event)."""
        gs = self._grad(grad, False, False)
        rd = N.RunDesc(protocol, h.to_c(), N.SCOPE_AGGREGATE, gs, 0, None, host_noise_sigma, 0)
        rd._keep = gs
        st, al = C.c_double(sim_time), C.c_double(alpha)
        N.check(self.lib.dsgd_run_events(self._ctx, C.byref(rd), events, rate_per_node,
                                         C.byref(st), C.byref(al)))
        return st.value, al.value

    def rounds_done(self) -> int:
        r = C.c_uint64()
        N.check(self.lib.dsgd_ctx_round(self._ctx, C.byref(r)))
        return r.value

    # ----------------------------------------------------------- multi-GPU
    def export_handle(self) -> bytes:
        buf = C.create_string_buffer(N.HANDLE_BYTES)
        N.check(self.lib.dsgd_ctx_export_handle(self._ctx, buf))
        return buf.raw

    def connect_peers(self, blobs: Sequence[bytes]) -> None:
        raw = b"".join(blobs)
        buf = C.create_string_buffer(raw, len(raw))
        N.check(self.lib.dsgd_ctx_connect_peers(self._ctx, buf))

    def init_nccl(self, uid: bytes, rank: int, nranks: int) -> None:
        buf = C.create_string_buffer(uid, N.NCCL_ID_BYTES)
        N.check(self.lib.dsgd_ctx_init_nccl(self._ctx, buf, rank, nranks))

    def set_timeout(self, seconds: float) -> None:
        N.check(self.lib.dsgd_ctx_set_timeout(self._ctx, seconds))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(N.NCCL_ID_BYTES)
        N.check(N.load().dsgd_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def distributed(cls, d: int, rank: int, world: int, device: int, dtype="f32",
                    nccl: bool = True, **kw) -> "Group":
        """One node per process/GPU; wires IPC peers (and, for the NVLS
        all-reduce, the library's own NVSwitch multicast object) and NCCL
        through the already-initialised torch.distributed process group (any
        backend) as the out-of-band channel.  The all-reduce backend is the
        library's choice (``allreduce_backend``)."""
        g = cls(d, p=world, dtype=dtype, device=device, first_node=rank, n_local=1, **kw)
        g.connect_peers(exchange_blobs(g.export_handle(), rank, world))
        if nccl and world > 1:
            g.init_nccl(broadcast_nccl_id(rank, world), rank, world)
        return g

    @property
    def allreduce_backend(self) -> str:
        """dsgd_ctx_allreduce_backend: local / oneshot / nvls / p2p / nccl."""
        return self.allreduce_info()[0]

    def allreduce_info(self):
        name, note = C.c_char_p(), C.c_char_p()
        N.check(self.lib.dsgd_ctx_allreduce_backend(self._ctx, C.byref(name), C.byref(note)))
        return name.value.decode(), (note.value or b"").decode()

    def attach_multicast(self, x: int, x_mc: int, avg: int, avg_mc: int) -> None:
        N.check(self.lib.dsgd_ctx_attach_multicast(self._ctx, x, x_mc, avg, avg_mc))

    # --------------------------------------------------------- measurement
    def profile(self, enable: bool) -> None:
        N.check(self.lib.dsgd_profile_enable(self._ctx, int(enable)))

    def profile_read(self, kernel: int, reset: bool = False):
        ms = C.c_double()
        n = C.c_uint64()
        N.check(self.lib.dsgd_profile_read(self._ctx, kernel, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def trace_dump(self, max_records: int = 65536) -> np.ndarray:
        """DSGD_TRACE records: [kind, round, t_entry, t_after_wait, t_done] (ns)."""
        out = np.zeros((max_records, 5), dtype=np.uint64)
        n = C.c_uint32()
        N.check(self.lib.dsgd_trace_dump(self._ctx, out.ctypes.data_as(N._U64P), max_records,
                                         C.byref(n)))
        return out[:n.value]

    def launch_count(self):
        k = C.c_uint64()
        n = C.c_uint64()
        N.check(self.lib.dsgd_launch_count(self._ctx, C.byref(k), C.byref(n)))
        return k.value, n.value


# ------------------------------------------------------ out-of-band wiring
def exchange_blobs(blob: bytes, rank: int, world: int) -> list:
    """All-gather the per-context handle blobs in node order over the
    torch.distributed group (the host-side half of dsgd_ctx_connect_peers)."""
    if len(blob) != N.HANDLE_BYTES:
        raise N.InvalidArgument("handle blob size")
    if world == 1:
        return [blob]
    import torch.distributed as dist
    blobs = [None] * world
    dist.all_gather_object(blobs, (rank, blob))
    blobs.sort(key=lambda x: x[0])
    if [r for r, _ in blobs] != list(range(world)):
        raise N.InvalidArgument("ranks must be 0..world-1")
    return [b for _, b in blobs]


def broadcast_nccl_id(rank: int, world: int, make=None) -> bytes:
    """Rank 0 creates the NCCL unique id, everyone receives it."""
    import torch.distributed as dist
    uid = [(make or Group.nccl_unique_id)() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    return uid[0]


def run_rounds_inproc(groups: Sequence[Group], protocol: int, h: Hyperparams, rounds: int,
                      scope: str = "aggregate", grad=None, grad_pools=None,
                      host_noise_sigma: float = 0.0, noise: bool = False) -> None:
    """dsgd_group_run_rounds: run_sync's round loop over an in-process group
    (every rank's round r in node order, then round r+1)."""
    n = len(groups)
    descs = [g._run_desc(protocol, h, rounds, scope, grad,
                         grad_pools[i] if grad_pools else None, host_noise_sigma, noise)
             for i, g in enumerate(groups)]
    arr = (N.RunDesc * n)(*descs)
    ctxs = (C.c_void_p * n)(*[g._ctx.value for g in groups])
    N.check(N.load().dsgd_group_run_rounds(ctxs, n, arr))
