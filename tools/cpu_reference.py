"""CPU baselines of SURVEY §8(d): the compiled reference (oracle/_ref) timed on
the host cores for every config's (d, p), single-threaded through the
simulator rules and multi-threaded through its own threaded
transport (run_transport, p worker threads + 1 EASGD server thread).
Median of `--reps` repetitions of `--rounds` rounds each; prints one JSON line
per measurement plus the host's CPU model and thread count.

    python tools/cpu_reference.py [--rounds 1] [--reps 3]
    python tools/cpu_reference.py --sweep [--max-seconds 1800]   (configs[4])

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


def mem_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def sweep(a):
    """configs[4]: d = 1M..1B per worker x {pull-gossip, elastic-avg,
    all-reduce} x p = 2/4/8, one round each (the reference's cost is linear
    in d), through the reference's threaded transport (p worker threads, +1
    EASGD server) -- its own parallel path -- and, up to 64M, the
    single-thread simulator rules.  Sizes whose fp64 state (~6 vectors of
    d doubles per node) exceeds half the available RAM are skipped and
    reported as such; the sweep stops issuing new sizes after
    --max-seconds."""
    import time
    import oracle as O
    h = O.HyperParams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    avail = mem_bytes()
    print(json.dumps({"host": host(), "mem_available_bytes": avail}), flush=True)
    protos = [("pull-gossip", O.PULL), ("elastic-avg", O.ELASTIC), ("all-reduce", O.ALLREDUCE)]
    t_start = time.time()
    for d in [int(float(x)) for x in a.sizes.split(",")]:
        for p in (2, 4, 8):
            for name, proto in protos:
                need = 6 * 8 * d * p
                if avail and need > avail // 2:
                    print(json.dumps({"config": "configs[4]", "protocol": name, "p": p, "d": d,
                                      "skipped": f"fp64 state ~{need / 2**30:.0f} GiB > half of "
                                                 f"{avail / 2**30:.0f} GiB available"}), flush=True)
                    continue
                if time.time() - t_start > a.max_seconds:
                    print(json.dumps({"config": "configs[4]", "protocol": name, "p": p, "d": d,
                                      "skipped": "time budget"}), flush=True)
                    continue
                nthr = len(os.sched_getaffinity(0))
                # every host thread: d split into coordinate shards, one
                # reference run (simulator rules) per shard, concurrently
                runs = [("simulator rules, all threads (coordinate shards)", False, nthr)]
                if d <= (64 << 20):  # the reference's own threaded transport
                    runs.append(("run_transport (threads)", True, 1))
                if d <= (16 << 20):
                    runs.append(("simulator rules (1 thread)", False, 1))
                for path, threaded, shards in runs:
                    try:
                        # the transport is timed as (R + 1) - 1 rounds of whole runs:
                        # R = 3 keeps the difference well above the run-to-run noise
                        r = 3 if threaded else 1
                        sec = O.ref_time_rounds(proto, p, d, r, threaded, h, "pool", shards) / r
                    except RuntimeError as e:  # e.g. the transport's own receive timeout
                        print(json.dumps({"config": "configs[4]", "protocol": name, "p": p,
                                          "d": d, "path": path,
                                          "error": str(e) or "reference raised"}), flush=True)
                        continue
                    threads = (p + (1 if proto == O.ELASTIC else 0)) if threaded else shards
                    print(json.dumps({"config": "configs[4]", "protocol": name, "p": p, "d": d,
                                      "path": path, "threads": threads,
                                      "s_per_round": sec, "param_updates_per_s": p * d / sec,
                                      "grad": "pool of 4 synthetic N(0,1) vectors (plugin slot)"}),
                          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--max-seconds", type=float, default=1800)
    ap.add_argument("--sizes", default=f"{1 << 20},{4 << 20},{16 << 20},{64 << 20},{256 << 20},{1 << 30}")
    a = ap.parse_args()
    if a.sweep:
        return sweep(a)
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
