"""CPU baselines of SURVEY §8(d): the compiled reference (oracle/_ref) timed on
the host cores for every config's (d, p), single-threaded through the
simulator rules and multi-threaded through its own threaded
transport (run_transport, p worker threads + 1 EASGD server thread).
Median of `--reps` repetitions of `--rounds` rounds each; prints one JSON line
per measurement plus the host's CPU model and thread count.

    python tools/cpu_reference.py [--rounds 1] [--reps 3]

Test/measurement infrastructure (it executes oracle/_ref, never the product)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def host():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": len(os.sched_getaffinity(0))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import oracle as O
    h = O.HyperParams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    cases = [  # (config, protocol, p, d, threaded)
        ("configs[3] all-reduce", O.ALLREDUCE, 1, 25_000_000, False),
        ("configs[3] all-reduce", O.ALLREDUCE, 2, 25_000_000, False),
        ("configs[3] all-reduce", O.ALLREDUCE, 2, 25_000_000, True),
        ("configs[3] all-reduce", O.ALLREDUCE, 4, 25_000_000, True),
        ("configs[3] all-reduce", O.ALLREDUCE, 8, 25_000_000, True),
        ("configs[1] pull-gossip", O.PULL, 8, 10_000_000, False),
        ("configs[2] elastic-avg", O.ELASTIC, 8, 25_000_000, False),
        ("configs[2] elastic-avg", O.ELASTIC, 8, 25_000_000, True),
    ]
    print(json.dumps({"host": host()}), flush=True)
    for name, proto, p, d, threaded in cases:
        secs = []
        for _ in range(a.reps):
            secs.append(O.ref_time_rounds(proto, p, d, a.rounds, threaded, h) / a.rounds)
        med = statistics.median(secs)
        print(json.dumps({"config": name, "p": p, "d": d,
                          "path": "run_transport (threads)" if threaded else "simulator rules (1 thread)",
                          "threads": (p + (1 if proto == O.ELASTIC else 0)) if threaded else 1,
                          "s_per_round_median": med, "s_per_round_all": secs,
                          "param_updates_per_s": p * d / med}), flush=True)


if __name__ == "__main__":
    main()
