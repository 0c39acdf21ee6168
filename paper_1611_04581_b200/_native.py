"""ctypes binding of the C ABI in include/dsgd_b200.h (libdsgd_b200.so).

There is no fallback: if the CUDA library is missing or cannot be loaded the
import fails loudly.  Status codes map onto the reference's exception
conventions: DSGD_EINVAL -> InvalidArgument (std::invalid_argument,
protocols.cpp:43-77), DSGD_ETIMEOUT -> TransportError (transport.hpp:57-60).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libdsgd_b200.so")

OK, EINVAL, ECUDA, ENCCL, ETIMEOUT, ENOMEM, ESTATE = range(7)
F32, F64 = 0, 1
ALLREDUCE, ELASTIC_AVG, PULL_GOSSIP, PUSH_GOSSIP, GOSSIP_STALE, GOSSIP_FRESH, ASYNC_PULL = range(7)
SCOPE_AGGREGATE, SCOPE_PER_NODE = 0, 1
PURPOSE = {"gradient-noise": 0, "sample": 1, "partner-choice": 2, "clock": 3,
           "straggler": 4, "init": 5}
CTX_QUADRATIC, CTX_GRAD, CTX_NOISE, CTX_CENTER = 1, 2, 4, 8
BUF_THETA, BUF_DELTA, BUF_GRAD, BUF_NOISE, BUF_SPECTRUM, BUF_OPT, BUF_CENTER = range(7)
GRAD_QUADRATIC, GRAD_BUFFER, GRAD_LOGISTIC = 0, 1, 2
K_STEP, K_ALLREDUCE, K_AR_DELTA, K_AR_APPLY, K_NCCL, K_EA, K_PUSH, K_OTHER = range(8)
KERNEL_NAMES = ["step", "allreduce_local", "ar_delta", "ar_apply", "allreduce_comm",
                "ea", "push", "other"]
HANDLE_BYTES = 512
NCCL_ID_BYTES = 128
MAX_LOCAL = 32


class DsgdError(RuntimeError):
    """A CUDA / NCCL / state error reported by the library."""


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class TransportError(RuntimeError):
    """dsgd::TransportError in the reference (a peer never arrived)."""


class Hyper(C.Structure):
    _fields_ = [("alpha0", C.c_double), ("anneal_factor", C.c_double),
                ("anneal_at", C.POINTER(C.c_uint64)), ("n_anneal", C.c_uint32),
                ("mu", C.c_double), ("weight_decay", C.c_double),
                ("beta_gossip", C.c_double), ("beta_ea", C.c_double),
                ("tau", C.c_uint32), ("batch", C.c_uint32)]


class CtxDesc(C.Structure):
    _fields_ = [("device", C.c_int), ("dim", C.c_uint64), ("dtype", C.c_int),
                ("p", C.c_uint32), ("first_node", C.c_uint32), ("n_local", C.c_uint32),
                ("flags", C.c_uint32), ("stream", C.c_void_p)]


class GradSpec(C.Structure):
    _fields_ = [("source", C.c_int), ("grad", C.POINTER(C.c_void_p)),
                ("use_noise", C.c_uint32), ("grad_norm_out", C.POINTER(C.c_double)),
                ("noise_sigma", C.c_double), ("noise_seed", C.c_uint64),
                ("rows", C.POINTER(C.c_uint64))]


class RunDesc(C.Structure):
    _fields_ = [("protocol", C.c_int), ("hyper", Hyper), ("scope", C.c_int),
                ("grad", GradSpec), ("n_grad_pool", C.c_uint32),
                ("grad_pool", C.POINTER(C.c_void_p)), ("host_noise_sigma", C.c_double),
                ("rounds", C.c_uint64)]


_P = C.c_void_p
_U32P = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)
_DP = C.POINTER(C.c_double)

# name -> (restype, argtypes)
_SIGS = {
    "dsgd_last_error": (C.c_char_p, []),
    "dsgd_abi_version": (C.c_int, []),
    "dsgd_derive_stream_seed": (C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint32, C.c_int]),
    "dsgd_stream_create": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "dsgd_stream_make": (C.c_int, [C.c_uint64, C.c_char_p, C.c_uint32, C.c_int, C.POINTER(_P)]),
    "dsgd_stream_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "dsgd_stream_destroy": (None, [_P]),
    "dsgd_stream_next_u64": (C.c_uint64, [_P]),
    "dsgd_stream_uniform01": (C.c_double, [_P]),
    "dsgd_stream_normal": (C.c_double, [_P]),
    "dsgd_stream_uniform_index": (C.c_int, [_P, C.c_uint32, _U32P]),
    "dsgd_stream_exponential": (C.c_int, [_P, C.c_double, _DP]),
    "dsgd_stream_fill_normal": (None, [_P, C.c_double, _P, C.c_uint64]),
    "dsgd_step_size_at": (C.c_double, [C.POINTER(Hyper), C.c_uint64]),
    "dsgd_hyperparams_validate": (C.c_int, [C.POINTER(Hyper)]),
    "dsgd_draw_pull_partners": (C.c_int, [C.POINTER(_P), C.c_uint32, _U32P]),
    "dsgd_draw_push_targets": (C.c_int, [C.POINTER(_P), C.c_uint32, _U32P]),
    "dsgd_ctx_create": (C.c_int, [C.POINTER(CtxDesc), C.POINTER(_P)]),
    "dsgd_ctx_destroy": (None, [_P]),
    "dsgd_ctx_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "dsgd_ctx_sync": (C.c_int, [_P]),
    "dsgd_grad_norm_flush": (C.c_int, [_P]),
    "dsgd_buffer_ptr": (C.c_int, [_P, C.c_uint32, C.c_int, C.POINTER(_P)]),
    "dsgd_set_state": (C.c_int, [_P, C.c_uint32, _P, _P, C.c_uint64]),
    "dsgd_get_state": (C.c_int, [_P, C.c_uint32, _P, _P, _U64P]),
    "dsgd_set_vector": (C.c_int, [_P, C.c_uint32, C.c_int, _P]),
    "dsgd_get_vector": (C.c_int, [_P, C.c_uint32, C.c_int, _P]),
    "dsgd_set_logistic": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_double]),
    "dsgd_logistic_set_sample_range": (C.c_int, [_P, C.c_uint32, C.c_uint64, C.c_uint64]),
    "dsgd_upload_async": (C.c_int, [_P, C.c_uint32, C.c_int, _P, C.c_uint64]),
    "dsgd_download_async": (C.c_int, [_P, C.c_uint32, C.c_int, _P, C.c_uint64]),
    "dsgd_copy_in_async": (C.c_int, [_P, C.c_uint32, C.c_int, _P, C.c_uint64]),
    "dsgd_get_t": (C.c_int, [_P, C.c_uint32, _U64P]),
    "dsgd_set_t": (C.c_int, [_P, C.c_uint32, C.c_uint64]),
    "dsgd_local_sgd_step": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec)]),
    "dsgd_allreduce_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), C.c_int]),
    "dsgd_ea_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), C.c_int]),
    "dsgd_pull_gossip_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), _U32P]),
    "dsgd_push_gossip_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), _U32P]),
    "dsgd_gossip_stale_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), _U32P]),
    "dsgd_gossip_fresh_round": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), _U32P]),
    "dsgd_async_pull_event": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), C.c_uint32,
                                        C.c_uint32]),
    "dsgd_gossip_stale_step": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), C.c_uint32,
                                         _P]),
    "dsgd_mix_toward": (C.c_int, [_P, C.c_uint32, _P, C.c_double]),
    "dsgd_eval_point": (C.c_int, [_P, C.POINTER(Hyper), C.c_uint32, _P]),
    "dsgd_pull_mix": (C.c_int, [_P, _U32P]),
    "dsgd_push_mix": (C.c_int, [_P, _U32P]),
    "dsgd_ea_init_center": (C.c_int, [_P]),
    "dsgd_gossip_fresh_mix": (C.c_int, [_P, _U32P, C.c_double]),
    "dsgd_ea_set_update_out": (C.c_int, [_P, C.POINTER(_P)]),
    "dsgd_ea_server_apply": (C.c_int, [_P, _P]),
    "dsgd_ea_client_event": (C.c_int, [_P, C.POINTER(Hyper), C.POINTER(GradSpec), C.c_uint32,
                                       C.c_int]),
    "dsgd_trace": (C.c_int, [_P, _DP, _DP, _DP]),
    "dsgd_ctx_seed_streams": (C.c_int, [_P, C.c_uint64, C.c_char_p]),
    "dsgd_run_rounds": (C.c_int, [_P, C.POINTER(RunDesc)]),
    "dsgd_run_events": (C.c_int, [_P, C.POINTER(RunDesc), C.c_uint64, C.c_double,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "dsgd_ctx_round": (C.c_int, [_P, _U64P]),
    "dsgd_ctx_export_handle": (C.c_int, [_P, _P]),
    "dsgd_ctx_connect_peers": (C.c_int, [_P, _P]),
    "dsgd_group_create_inproc": (C.c_int, [C.POINTER(CtxDesc), C.c_uint32, C.POINTER(C.c_int),
                                           C.POINTER(_P)]),
    "dsgd_group_run_rounds": (C.c_int, [C.POINTER(_P), C.c_uint32, C.POINTER(RunDesc)]),
    "dsgd_ctx_allreduce_backend": (C.c_int, [_P, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]),
    "dsgd_nccl_unique_id": (C.c_int, [_P]),
    "dsgd_ctx_attach_multicast": (C.c_int, [_P, _P, _P, _P, _P]),
    "dsgd_ctx_init_nccl": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "dsgd_ctx_set_timeout": (C.c_int, [_P, C.c_double]),
    "dsgd_profile_enable": (C.c_int, [_P, C.c_int]),
    "dsgd_profile_read": (C.c_int, [_P, C.c_int, _DP, _U64P, C.c_int]),
    "dsgd_launch_count": (C.c_int, [_P, _U64P, _U64P]),
    "dsgd_trace_dump": (C.c_int, [_P, _U64P, C.c_uint32, C.POINTER(C.c_uint32)]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load():
    """Load libdsgd_b200.so (raises if it is missing: there is no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        raise ImportError(f"{SO} is not built; run `python -m paper_1611_04581_b200.build` "
                          "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(SO)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if lib.dsgd_abi_version() != 2:
        raise ImportError("libdsgd_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == OK:
        return
    msg = load().dsgd_last_error().decode(errors="replace")
    if status == EINVAL:
        raise InvalidArgument(msg)
    if status == ETIMEOUT:
        raise TransportError(msg)
    raise DsgdError(f"status {status}: {msg}")
