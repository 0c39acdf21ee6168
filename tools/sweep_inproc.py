"""Sweep runtime knobs of the multi-GPU kernels with single-process runs of
tools/nvlink_profile.py (an in-process group over --gpus GPUs), one fresh
process per configuration (the knobs are read once per process).

    python tools/sweep_inproc.py --gpus 4 --protocol all-reduce --d 25000000 \\
        --grid "DSGD_AR_PIPES=2,3,4;DSGD_AR_DELTA_FRAC=1.25,1.5;DSGD_NVLS_UNROLL=4,8"

Prints one JSON line per configuration (the knob values + the tool's line).
"""
import argparse
import itertools
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--protocol", default="all-reduce")
    ap.add_argument("--d", type=int, default=25_000_000)
    ap.add_argument("--rounds", type=int, default=30)
    ap.add_argument("--grid", default="")
    ap.add_argument("--timeout", type=float, default=180)
    a = ap.parse_args()
    axes = []
    for part in filter(None, a.grid.split(";")):
        k, vals = part.split("=", 1)
        axes.append([(k, v) for v in vals.split(",")])
    for combo in itertools.product(*axes) if axes else [()]:
        env = dict(os.environ)
        env.update(dict(combo))
        cmd = [sys.executable, os.path.join(HERE, "nvlink_profile.py"), "--gpus", str(a.gpus),
               "--protocol", a.protocol, "--d", str(a.d), "--rounds", str(a.rounds)]
        try:
            out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=a.timeout)
            lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
            res = json.loads(lines[-1]) if lines else {"error": out.stderr[-400:]}
        except subprocess.TimeoutExpired:
            res = {"error": "timeout"}
        print(json.dumps({"knobs": dict(combo), **res}), flush=True)


if __name__ == "__main__":
    main()
