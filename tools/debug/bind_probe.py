"""Bisect helper: the reference drivers through the binding after a given
process-state change (argv[1]: 'torch' = import torch + device_count)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "torch":
    import torch
    print("devices", torch.cuda.device_count(), flush=True)

import oracle as O  # noqa: E402
from tests.golden.make_golden import RUN_CASES  # noqa: E402

HARNESS = os.path.join(ROOT, "integration", "_build", "libdsgd_ref_b200_harness.so")
g = np.load(os.path.join(ROOT, "tests", "golden", "runs.npz"))
bad = 0
for name in ("c1_allreduce", "async8", "pull8", "ea8"):
    with O.ref_library(HARNESS):
        O.ref_set_logistic(None, None, 0.0)
        th, dp, t, c = O.ref_run(RUN_CASES[name])
    ref = g[f"{name}_theta"]
    same = np.asarray(th).tobytes() == ref.tobytes()
    err = float(np.max(np.abs(np.asarray(th) - ref)))
    print(name, "same" if same else "DIFF", "max_abs", err, flush=True)
    bad += not same
sys.exit(1 if bad else 0)
