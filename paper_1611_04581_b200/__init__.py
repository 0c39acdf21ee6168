"""B200-native parameter-aggregation and update path of arXiv 1611.04581
(synchronous all-reduce SGD, elastic averaging SGD, gossiping SGD with
Nesterov momentum).

* ``include/dsgd_b200.h`` -- the C ABI (libdsgd_b200.so, sm_100a kernels);
* ``engine.Group`` -- device-resident worker groups (1 GPU x p nodes, or one
  node per GPU over NVLink peer memory + NCCL);
* ``protocols`` -- the reference's value-semantic update-rule interface
  (protocols.hpp) executed by the kernels;
* ``driver`` -- the per-step worker loop (run_sync / async-pull).
"""
from . import _native
from .engine import Group, Hyperparams, Stream, derive_stream_seed, step_size_at

__all__ = ["Group", "Hyperparams", "Stream", "derive_stream_seed", "step_size_at", "_native"]
