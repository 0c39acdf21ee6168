"""Benchmark of the B200 aggregation/update hot path (BASELINE.json).

Workload (BASELINE.json configs[3]): synchronous all-reduce SGD with
Nesterov momentum, d = 25M fp32 parameters per worker, one worker per GPU
(p = N), synthetic N(0,1) gradients (a pool of 4 distinct device buffers per
worker, cycled; every step's working set -- theta, delta, gradient, ~400 MB
-- exceeds the 126 MB L2, so no flush is needed).  A step is one
allreduce_round (protocols.cpp:110-131): at N = 1 the single fused round
kernel (k_local_tma, streams staged through smem by cp.async.bulk); at N > 1
the library's multi-GPU all-reduce over NVLink (one-shot peer-memory kernel
at N <= 2, NVLS multimem two-shot with two pipelines at N > 2; see
DESIGN.md §5), with the apply fused into the next round's delta.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` is the whole-job worker
param-updates/s with inputs resident in HBM; `e2e` is the same metric through
the C ABI with each step's gradient copied host->device from pinned memory
and the step's result (the gradient norm, protocols.cpp:34-36) read back.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "worker param-updates/sec and aggregation-step GB/s vs HBM/NVLink roofline"
UNIT = "param-updates/s"
D_DEFAULT = 25_000_000
POOL = 4
SPEC_HBM_GBS = 8000.0  # the north star's ~8 TB/s HBM denominator (DGX B200 spec)
# highest raw NVLink rate per direction seen on this pool (ncu nvltx on the N=2
# one-shot round's serving side; profiles/r2_nvlink_ncu.md)
RAW_CEIL = 755.0


def workload_config(d: int, world: int) -> dict:
    """The `config` of BOTH arms (ours and --impl reference): the same
    workload, key for key."""
    return {"workload": "configs[3]: synchronous all-reduce SGD round (allreduce_round, Nesterov "
                        "momentum 0.9, wd 1e-4, aggregate momentum scope), synthetic gradients",
            "d_per_worker": d, "p": world, "parallelism": f"dp{world}",
            "grad_source": f"pool of {POOL} synthetic N(0,1) gradient vectors per worker, served "
                           "in turn through the Objective plugin slot",
            "l2": "inputs larger than L2 (~400 MB/step/worker working set)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # --params: the same (torchrun's own parser rejects "--d" as ambiguous)
    ap.add_argument("--d", "--params", dest="d", type=int, default=D_DEFAULT)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--no-extras", action="store_true", help="skip the gossip/EASGD extra lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.path = f"/tmp/dsgd_clocks_{os.getpid()}.csv"

    def _load(self):
        try:
            with open(self.path) as f:
                self.rows = [[x.strip() for x in line.split(",")] for line in f if line.strip()]
        except OSError:
            self.rows = []

    def __enter__(self):
        # written to a file (a pipe would sit in nvidia-smi's stdio buffer)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 10:   # wait until the sampler is live
                self._load()
                if self.rows:
                    break
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self._load()
        try:
            os.remove(self.path)
        except OSError:
            pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------ reference arm
def host_info() -> dict:
    """CPU model and usable host threads of the box the baseline ran on."""
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


def cpu_reference(protocol: int, p: int, d: int, rounds: int, threaded: bool, grad="pool",
                  shards: int = 1):
    import oracle as O
    h = O.HyperParams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    return O.ref_time_rounds(protocol, p, d, rounds, threaded, h, grad, shards)


def host_shards(p: int, threaded: bool) -> int:
    """Concurrent reference runs that fill the host: one per usable thread
    (simulator rules), or nproc // p for run_transport's p threads each."""
    n = len(os.sched_getaffinity(0))
    return max(1, n // p) if threaded else max(1, n)


def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle as O
    p = max(1, args.gpus)
    d_sample = args.d              # the same per-worker size as our arm
    # the simulator's rule over p workers (the reference's implementation of
    # the round), d split over every host thread: the fastest way the
    # reference's own code runs this workload on this host (its threaded
    # run_transport uses p threads only; tools/cpu_reference.py times it)
    threaded = False
    # bounded sample: at most 2 warm-up and 20 timed rounds (a 25M-param
    # fp64 round takes ~0.7 s on one core), so the arm ends within minutes
    steps = max(1, min(args.steps, 20 if p == 1 else 10))
    shards = host_shards(p, threaded)
    cpu_reference(O.ALLREDUCE, p, d_sample, max(1, min(args.warmup, 2)), threaded, shards=shards)
    sec = cpu_reference(O.ALLREDUCE, p, d_sample, steps, threaded, shards=shards)
    per = sec / steps
    value = p * d_sample / per
    kind = "reference" if O.ref_available() else "port"
    cores = shards * (p if threaded else 1)
    sample = (f"{steps} allreduce_round steps of the compiled reference "
              f"({'run_transport, ring_allreduce over p threads' if threaded else 'simulator rules'})"
              f", p={p}, d={d_sample} per worker (of {args.d}), split into {shards} coordinate "
              f"shards run concurrently (one reference run per shard, {cores} host threads)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args.d, p),
            "reference_path": (f"run_transport (ring_allreduce over p worker threads) x {shards} "
                               "coordinate shards" if threaded
                               else f"simulator rules (allreduce_round) x {shards} coordinate shards"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d = args.d
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4)

    if world > 1:
        grp = Group.distributed(d, rank, world, local, dtype=args.dtype, grad=True)
    else:
        grp = Group(d, 1, dtype=args.dtype, grad=True, device=local)
    gen = torch.Generator(device=f"cuda:{local}")
    gen.manual_seed(1234 + rank)
    pool = [torch.randn(d, generator=gen, device=f"cuda:{local}", dtype=tdt) for _ in range(POOL)]
    torch.cuda.synchronize()
    # initial theta: a common start on every worker (N(0,1), rank-0 seed)
    g0 = torch.Generator(device=f"cuda:{local}")
    g0.manual_seed(99)
    theta0 = torch.randn(d, generator=g0, device=f"cuda:{local}", dtype=tdt)
    torch.cuda.synchronize()
    grp.copy_in_async(0, N.BUF_THETA, theta0.data_ptr(), d)
    grp.sync()
    del theta0
    import ctypes
    stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
    pool_ptrs = [t.data_ptr() for t in pool]

    def barrier():
        if world > 1:
            dist.barrier()

    def rounds(k):
        grp.run_rounds(N.ALLREDUCE, h, k, grad_pool=pool_ptrs)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (also sizes the clock-sampling load below)
    t_w = time.perf_counter()
    rounds(max(3, args.warmup))
    grp.sync()
    est = max_over_ranks((time.perf_counter() - t_w) / max(3, args.warmup))
    barrier()
    torch.cuda.synchronize()
    load_rounds = int(min(20000, max(50, 0.6 / max(est, 1e-6))))  # same count on every rank

    def load():
        # untimed sustained load around the (milliseconds-long) timed region so
        # the nvidia-smi samples see the GPU under this kernel
        rounds(load_rounds)
        grp.sync()

    # ---------------- timed region (device-resident inputs)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        load()
        barrier()
        torch.cuda.synchronize()
        # no per-launch events inside the timed region: an event between two
        # back-to-back kernels costs ~5 us per step here (measured,
        # tools/step_gap.py)
        k0, n0 = grp.launch_count()
        ev0.record(stream)
        rounds(args.steps)
        ev1.record(stream)
        grp.sync()
        torch.cuda.synchronize()
        k1, n1 = grp.launch_count()
        barrier()
        # per-kernel breakdown: the same K rounds again with per-launch events
        grp.profile(True)
        pe0 = torch.cuda.Event(enable_timing=True)
        pe1 = torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        rounds(args.steps)
        pe1.record(stream)
        grp.sync()
        torch.cuda.synchronize()
        prof = {N.KERNEL_NAMES[k]: grp.profile_read(k, reset=True) for k in range(8)}
        prof_ms = pe0.elapsed_time(pe1)
        barrier()
        grp.profile(False)
        load()
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms)
    step_ms = ms_max / args.steps
    value = world * d / (step_ms * 1e-3)

    # dominant kernel + roofline (algorithmic bytes per launch)
    backend = getattr(grp, "allreduce_backend", "local")
    peak, peak_src = peaks()
    nv_peak = 770.0  # measured peer copy per direction (B200_PROFILING.md)
    if backend == "oneshot":
        nv_bytes = (world - 1) * es * d              # each rank reads every peer's exchange
    elif backend == "nvls":
        nv_bytes = (1 + 1 / world) * es * d          # switch reads every x once + multicast avg
    else:
        nv_bytes = 2 * (world - 1) / world * es * d  # two-shot / ring, per direction per GPU
    if world == 1:
        kname, bpp = "allreduce_local", 5 * es  # read theta, delta, g; write theta', delta'
        kdesc = ("k_local_tma (p=1 round: fused delta + mean + apply; theta, delta, g staged "
                 "through smem by cp.async.bulk; back-to-back rounds with programmatic dependent "
                 "launch), 12 B read + 8 B write per param")
    elif backend == "oneshot":
        kname, bpp = "allreduce_comm", (5 + (world - 1)) * es
        kdesc = ("k_ar_oneshot_tma2: one kernel per round; every rank's previous exchange tile and "
                 "this rank's theta/g staged in smem by cp.async.bulk (2 stages x 3 CTAs/SM; P-1 "
                 "tiles over NVLink), ring-order average fused with theta += "
                 "avg and the next delta; HBM: theta, g, own x read + theta', x' write + x served "
                 f"to {world - 1} peer(s); NVLink {nv_bytes / d:.0f} B/param each direction")
    elif backend == "nvls":
        kname, bpp = "allreduce_comm", 2 * es
        kdesc = ("k_ar_nvls: multimem.ld_reduce of this rank's slice of every GPU's exchange "
                 "buffer (sum in the NVSwitch) + multimem.st of the average to every GPU; "
                 f"NVLink ~{nv_bytes / d:.1f} B/param each direction")
    elif backend == "p2p":
        kname, bpp = "allreduce_comm", 2 * es
        kdesc = ("k_ar_reduce: ring-order reduce of this rank's chunk from every rank + average "
                 f"to every rank; NVLink {nv_bytes / d:.1f} B/param each direction")
    else:
        kname, bpp = "ar_delta", 5 * es
        kdesc = "k_step<ApplyDelta>: read theta, avg, g; write theta', delta' (then ncclAllReduce)"
    kms_p, kn = prof.get(kname, (0.0, 0))
    share = (kms_p / prof_ms) if prof_ms else None
    # one launch of the dominant kernel per step (+ the run's final deferred
    # apply, which run_rounds materialises once at the end at N > 1)
    single = kn == args.steps and (k1 - k0) in (args.steps, args.steps + 1) and (n1 - n0) == 0
    if single:
        # the step IS one launch of this kernel: its duration is the timed
        # region / launches (CUDA events around the region on this stream;
        # includes the ~1 us launch gap, so conservative)
        kms = ms
        timing = "timed region / launches (one launch of this kernel per step, no per-launch events)"
    else:
        kms = kms_p
        timing = "per-launch CUDA events in a second pass of the same K rounds"
    kavg_ms = kms / max(1, kn)
    # parameters one launch processes: d, or d / K with K pipelines per round
    units = d * args.steps / kn if kn else d
    achieved = (bpp * units / (kavg_ms * 1e-3) / 1e9) if kn else None
    t_hbm = bpp * units / (peak * 1e9)
    t_nv = (nv_bytes * units / d / (nv_peak * 1e9)
            if (world > 1 and kname == "allreduce_comm") else 0.0)
    bound = "nvlink" if t_nv > t_hbm else "hbm"
    traffic, traffic_src = None, None
    if world == 1 and es == 4:  # DRAM bytes of the same kernel: a PRIOR ncu capture (committed)
        for cap in ("r2_ncu_traffic.json", "r1_ncu_traffic.json"):
            try:
                with open(os.path.join(ROOT, "profiles", cap)) as f:
                    t = json.load(f).get(f"k_local_tma<float>/d={d}")
                if t:
                    traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
                    traffic_src = (f"prior ncu --set full capture of the same kernel and size "
                                   f"(profiles/{cap}), not measured in this run")
                    break
            except (OSError, ValueError, KeyError):
                continue
    roofline = {"bound": bound, "kernel": kdesc, "achieved": achieved, "peak": peak,
                "peak_source": peak_src, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "frac_of_spec_hbm": (achieved / SPEC_HBM_GBS) if achieved else None,
                "spec_hbm_gbs": SPEC_HBM_GBS,
                "algorithmic_bytes_per_launch": bpp * units,
                "params_per_launch": units,
                "kernel_avg_us": kavg_ms * 1e3,
                "roofline_time_us": max(t_hbm, t_nv) * 1e6,
                "frac_of_roofline_time": (max(t_hbm, t_nv) / (kavg_ms * 1e-3)) if kn else None,
                "kernel_timing": timing,
                "share_of_step": share}
    step_bytes = 5 * es * d if world == 1 else 7 * es * d
    if world > 1:
        nms, nn = prof.get("allreduce_comm", (0.0, 0))
        t_c = nms / max(1, nn) * 1e-3
        if single and kname == "allreduce_comm":
            t_c = kavg_ms * 1e-3  # the timed region's own per-launch time
        nv_launch = nv_bytes * (args.steps / nn if nn else 1.0)  # per launch (K pipelines)
        if nn and nn > args.steps:
            # K > 1 pipelines: their reduce kernels overlap each other and the
            # delta kernels, so a per-launch event span includes the others'
            # time; the comm kernels are active across the whole round, so the
            # round's NVLink bytes over the round time is the kernel's rate
            t_c = step_ms * 1e-3
            nv_launch = nv_bytes
            roofline["kernel_timing"] = ("K overlapping pipelines: NVLink bytes per round / "
                                         "round time (per-launch events would double-count "
                                         "the overlap)")
            roofline["kernel_avg_us"] = step_ms * 1e3
            if roofline.get("achieved") and kname == "allreduce_comm":
                roofline["achieved"] = bpp * d / (step_ms * 1e-3) / 1e9
                roofline["frac"] = roofline["achieved"] / peak
                roofline["frac_of_roofline_time"] = roofline["roofline_time_us"] * kn / args.steps \
                    / (step_ms * 1e3)
        roofline["allreduce_backend"] = backend
        roofline["allreduce_launches_per_round"] = nn / args.steps if nn else None
        note = grp.allreduce_info()[1]
        if note:
            roofline["nvls_unavailable"] = note
        roofline["allreduce_comm_us"] = t_c * 1e6
        roofline["nvlink_bytes_per_direction_per_round"] = nv_bytes
        roofline["nvlink_achieved_gbs"] = nv_launch / t_c / 1e9 if nn else None
        roofline["nvlink_peak_gbs"] = nv_peak
        roofline["nvlink_frac"] = (nv_launch / t_c / 1e9 / nv_peak) if nn else None
        # SM-issued symmetric exchange measured on this pool (both GPUs of a
        # pair reading / writing each other at once, profiles/r1_nvlink_probe.txt)
        roofline["nvlink_sm_exchange_gbs"] = {"peer_read": 630.0, "peer_write": 668.0}
        if bound == "nvlink" and nn:
            # the dominant kernel is NVLink-bound: report it against the link
            roofline["hbm_achieved"] = roofline["achieved"]
            roofline["hbm_frac"] = roofline["frac"]
            roofline["achieved"] = nv_launch / t_c / 1e9
            roofline["peak"] = nv_peak
            roofline["peak_source"] = "B200_PROFILING.md measured peer copy per direction"
            roofline["frac"] = roofline["achieved"] / nv_peak
        # the same kernel against the raw link: NVLink packet bytes per data
        # byte and the best raw rate of one SM-issued stream, both from
        # PRIOR ncu link-counter captures (profiles/r2_nvlink_ncu.md)
        if nn:
            # busiest direction: NVLS 1.41 both ways; one-shot tx = served
            # reads (1.125) + the peer's read requests (0.1875); p2p two-shot
            # tx (stores + requests) 1.37-1.50
            raw = {"nvls": 1.41, "oneshot": 1.3125, "p2p": 1.44}.get(backend)
            if raw:
                roofline["nvlink_raw"] = {
                    "raw_bytes_per_data_byte": raw,
                    "achieved_raw_gbs": nv_launch / t_c / 1e9 * raw,
                    # the highest raw rate seen on this pool: the tx side of
                    # the N=2 one-shot round (served reads + requests)
                    "raw_ceiling_gbs": RAW_CEIL,
                    "frac_of_raw_ceiling": nv_launch / t_c / 1e9 * raw / RAW_CEIL,
                    "source": "prior ncu nvl{rx,tx}__bytes captures (profiles/r2_nvlink_ncu.md, "
                              "r2_ncu_nvlink/*.csv), not measured in this run"}
    per_kernel = {k: {"ms_total": v[0], "launches": v[1]} for k, v in prof.items() if v[1]}

    # ---------------- end-to-end through the C ABI (host gradients, pinned)
    e2e = None
    if True:
        host = [torch.randn(d, dtype=tdt).pin_memory() for _ in range(2)]
        barrier()
        torch.cuda.synchronize()
        steps_e2e = max(3, min(args.steps, 20))
        # a user's input pipeline: step s+1's gradient streams host -> device
        # on a copy stream (double-buffered) while step s's round runs; the
        # round reads it as its external gradient buffer and returns ||g||
        # to the host (D2H + sync) every step
        copy_stream = torch.cuda.Stream(device=f"cuda:{local}")
        dbuf = [torch.empty(d, dtype=tdt, device=f"cuda:{local}") for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]

        def upload(s):
            with torch.cuda.stream(copy_stream):
                # dbuf[s % 2] was last read by round s - 2, which has completed
                # (every round syncs for its gradient norm)
                dbuf[s % 2].copy_(host[s % 2], non_blocking=True)
                ready[s % 2].record(copy_stream)

        def e2e_steps(n):
            upload(0)
            for s in range(n):
                if s + 1 < n:
                    upload(s + 1)
                stream.wait_event(ready[s % 2])
                grp.allreduce_round(h, grad=[dbuf[s % 2].data_ptr()], grad_norm=True)

        e2e_steps(2)  # warm
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(copy_stream)
        e2e_steps(steps_e2e)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3))
        e2e = {"value": world * d / (e_ms / steps_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": es * d * world, "d2h_bytes_per_step": 8 * world,
               "steps": steps_e2e, "ms_per_step": e_ms / steps_e2e,
               "path": "pinned host gradient -> device (copy stream, double-buffered) + "
                       "dsgd_allreduce_round(external gradient, grad_norm_out -> host)"}

    # ---------------- e2e, the Objective plugin contract (objectives.hpp:43-48):
    # every step the evaluation point theta + mu*delta_prev goes device ->
    # host, the host Objective (here QuadraticObjective(spectrum 1, optimum 0):
    # g = point) produces the gradient, which goes host -> device and the
    # round runs on it -- the round trip a host-side model forces per step
    e2e_plugin = None
    if True:
        pin = torch.empty(d, dtype=tdt).pin_memory()
        dgrad = torch.empty(d, dtype=tdt, device=f"cuda:{local}")
        steps_p = max(3, min(args.steps, 10))

        def plugin_steps(n):
            for _ in range(n):
                grp.eval_point(h, 0, dgrad.data_ptr())
                with torch.cuda.stream(stream):
                    pin.copy_(dgrad, non_blocking=True)  # D2H: the evaluation point
                stream.synchronize()
                # host Objective: g = spectrum * (point - optimum) = point
                with torch.cuda.stream(stream):
                    dgrad.copy_(pin, non_blocking=True)  # H2D: the gradient
                grp.allreduce_round(h, grad=[dgrad.data_ptr()])
            grp.sync()

        plugin_steps(2)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plugin_steps(steps_p)
        torch.cuda.synchronize()
        p_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
        e2e_plugin = {"value": world * d / (p_ms / steps_p * 1e-3), "unit": UNIT,
                      "h2d_bytes_per_step": es * d * world, "d2h_bytes_per_step": es * d * world,
                      "steps": steps_p, "ms_per_step": p_ms / steps_p,
                      "path": "dsgd_eval_point (theta + mu*delta_prev) -> host, host "
                              "QuadraticObjective(1, 0) gradient -> device, "
                              "dsgd_allreduce_round(external gradient); wall clock"}
        del pin, dgrad

    # ---------------- extras: gossip / EASGD shapes
    extras = {}
    if world == 1 and not args.no_extras:
        extras = run_extras(args, local, h)
    elif world > 1 and not args.no_extras:
        extras = run_extras_dist(args, world, rank, local, h, max_over_ranks, barrier)

    # ---------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        try:
            import oracle as O
            d_s = d
            rounds_cpu = 8
            shards = host_shards(1, False)
            sec = cpu_reference(O.ALLREDUCE, 1, d_s, rounds_cpu, False, shards=shards)
            sec1 = cpu_reference(O.ALLREDUCE, 1, d_s, 2, False) / 2
            cpu = {"value": d_s / (sec / rounds_cpu), "unit": UNIT, "cores": shards,
                   "kind": "reference" if O.ref_available() else "port",
                   "sample": f"{rounds_cpu} allreduce_round (p=1, d={d_s}) of the compiled "
                             f"reference (oracle/_ref, -O3, fp64), d split into {shards} "
                             f"coordinate shards run concurrently on {shards} host threads",
                   "single_thread_value": d_s / sec1,
                   "host": host_info()}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic",
                "config": workload_config(d, world),
                "gbs": step_bytes / (step_ms * 1e-3) / 1e9,
                "gbs_note": "aggregation-step algorithmic HBM GB/s per GPU",
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "e2e_objective_plugin": e2e_plugin,
                "gpu_launches": (k1 - k0) + (n1 - n0),
                "gpu_launches_detail": {"kernels": k1 - k0, "nccl_calls": n1 - n0},
                "per_kernel": per_kernel,
                "clocks": dict(clocks.summary(), window="nvidia-smi -lms 50 over ~0.6 s of the same "
                               "rounds before and after the timed region, and during it"),
                "extras": extras}
        print(json.dumps(line), flush=True)
    grp.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_extras(args, local, h):
    """configs[1]/[2] shapes with all workers on ONE GPU (node-emulated):
    pull-gossip 8 x 10M and EASGD 8 x 25M; one fused kernel per round."""
    import torch
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group
    out = {}
    for name, proto, p, d, bpp in (("pull-gossip p=8 x 10M (1 GPU)", N.PULL_GOSSIP, 8, 10_000_000, 24),
                                   ("elastic-avg p=8 x 25M (1 GPU)", N.ELASTIC_AVG, 8, 25_000_000, 20)):
        try:
            grp = Group(d, p, dtype="f32", device=local, center=(proto == N.ELASTIC_AVG))
            gen = torch.Generator(device=f"cuda:{local}")
            gen.manual_seed(7)
            pool = [torch.randn(d, generator=gen, device=f"cuda:{local}") for _ in range(p * 2)]
            for i in range(p):
                grp.copy_in_async(i, N.BUF_THETA, pool[i].data_ptr(), d)
            grp.sync()
            if proto == N.ELASTIC_AVG:
                grp.ea_init_center()
            grp.seed_streams(1, "run/trial0")
            ptrs = [t.data_ptr() for t in pool]
            grp.run_rounds(proto, h, 3, grad_pool=ptrs)
            grp.sync()
            stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            k = 20
            e0.record(stream)
            grp.run_rounds(proto, h, k, grad_pool=ptrs)
            e1.record(stream)
            grp.sync()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / k
            # EASGD: 8 clients x (theta, delta, g read + theta, delta write) + center R/W once
            byts = p * d * bpp + (8 * d if proto == N.ELASTIC_AVG else 0)
            out[name] = {"ms_per_round": ms, "param_updates_per_s": p * d / (ms * 1e-3),
                         "hbm_gbs": byts / (ms * 1e-3) / 1e9,
                         "bytes_per_param": byts / (p * d)}
            grp.close()
            del pool
            torch.cuda.empty_cache()
        except Exception as e:  # pragma: no cover
            out[name] = {"error": str(e)}
    # run_sync's own call pattern: every round raises grad_norm_out
    # (simulator.cpp:239) -- accumulated on the device, read once per run
    name = "all-reduce p=1 x 25M with grad_norm_out (run_sync pattern)"
    try:
        from paper_1611_04581_b200.engine import Hyperparams
        d = args.d
        grp = Group(d, 1, dtype="f32", device=local, grad=True)
        gen = torch.Generator(device=f"cuda:{local}")
        gen.manual_seed(5)
        pool = [torch.randn(d, generator=gen, device=f"cuda:{local}") for _ in range(POOL)]
        ptrs = [t.data_ptr() for t in pool]
        grp.copy_in_async(0, N.BUF_THETA, pool[0].data_ptr(), d)
        grp.run_rounds(N.ALLREDUCE, h, 5, grad_pool=ptrs, grad_norm=True)
        grp.sync()
        stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
        res = {}
        for norm in (False, True):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            k = 50
            e0.record(stream)
            gn = grp.run_rounds(N.ALLREDUCE, h, k, grad_pool=ptrs, grad_norm=norm)
            e1.record(stream)
            grp.sync()
            torch.cuda.synchronize()
            res[norm] = (e0.elapsed_time(e1) / k, gn)
        out[name] = {"ms_per_round": res[True][0], "ms_per_round_without_norm": res[False][0],
                     "overhead": res[True][0] / res[False][0] - 1.0,
                     "max_grad_norm": res[True][1],
                     "param_updates_per_s": d / (res[True][0] * 1e-3)}
        grp.close()
        del pool
        torch.cuda.empty_cache()
    except Exception as e:  # pragma: no cover
        out[name] = {"error": str(e)}
    # the reference arm's own arithmetic on the GPU: fp64, gradient from the
    # fused QuadraticObjective(spectrum 1, optimum 0) -- bit-exact with the
    # reference in fp64 (tests/test_gpu_parity.py); 48 B/param
    name = "all-reduce p=1 x 25M fp64, QuadraticObjective(1, 0) (reference arithmetic)"
    try:
        d = args.d
        grp = Group(d, 1, dtype="f64", device=local, quadratic=True)
        ones = torch.ones(d, dtype=torch.float64, device=f"cuda:{local}")
        zeros = torch.zeros(d, dtype=torch.float64, device=f"cuda:{local}")
        gen = torch.Generator(device=f"cuda:{local}")
        gen.manual_seed(6)
        th = torch.randn(d, generator=gen, device=f"cuda:{local}", dtype=torch.float64)
        torch.cuda.synchronize()
        grp.copy_in_async(0, N.BUF_SPECTRUM, ones.data_ptr(), d)
        grp.copy_in_async(0, N.BUF_OPT, zeros.data_ptr(), d)
        grp.copy_in_async(0, N.BUF_THETA, th.data_ptr(), d)
        grp.run_rounds(N.ALLREDUCE, h, 3, grad="quadratic")
        grp.sync()
        stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        k = 30
        e0.record(stream)
        grp.run_rounds(N.ALLREDUCE, h, k, grad="quadratic")
        e1.record(stream)
        grp.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        hbm, _ = peaks()
        byts = 48 * d  # theta, delta, s, opt read + theta', delta' written, fp64
        shards = host_shards(1, False)
        ref_s = cpu_reference(0, 1, d, 4, False, grad="quadratic", shards=shards) / 4 \
            if not args.no_cpu else None
        out[name] = {"ms_per_round": ms, "param_updates_per_s": d / (ms * 1e-3),
                     "hbm_gbs": byts / (ms * 1e-3) / 1e9, "hbm_frac": byts / (ms * 1e-3) / 1e9 / hbm,
                     "bytes_per_param": 48,
                     "reference_cpu_param_updates_per_s": (d / ref_s) if ref_s else None,
                     "reference_cpu_sample": f"4 allreduce_round of the compiled reference, "
                                             f"QuadraticObjective(1, 0), p=1, d split over "
                                             f"{shards} host threads"}
        grp.close()
        del ones, zeros, th
        torch.cuda.empty_cache()
    except Exception as e:  # pragma: no cover
        out[name] = {"error": str(e)}
    # F4: the asynchronous event loop in the library (dsgd_run_events): one
    # async_pull_event kernel per Poisson tick, 8 nodes x 10M on one GPU
    name = "async-pull p=8 x 10M (1 GPU, events)"
    try:
        from paper_1611_04581_b200.engine import Hyperparams
        p, d = 8, 10_000_000
        grp = Group(d, p, dtype="f32", device=local, grad=True)
        gen = torch.Generator(device=f"cuda:{local}")
        gen.manual_seed(9)
        for i in range(p):
            t = torch.randn(d, generator=gen, device=f"cuda:{local}")
            grp.copy_in_async(i, N.BUF_THETA, t.data_ptr(), d)
            grp.copy_in_async(i, N.BUF_GRAD, t.data_ptr(), d)
            grp.sync()
        grp.seed_streams(2, "c4/trial0")
        ha = Hyperparams(alpha0=0.05, anneal_at=(), mu=0.0, weight_decay=1e-4, beta_gossip=0.5)
        grp.run_events(N.ASYNC_PULL, ha, 10, 1.0, grad="buffer")
        grp.sync()
        stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        k = 200
        e0.record(stream)
        grp.run_events(N.ASYNC_PULL, ha, k, 1.0, grad="buffer")
        e1.record(stream)
        grp.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        out[name] = {"ms_per_event": ms, "events_per_s": 1e3 / ms,
                     "param_updates_per_s": d / (ms * 1e-3),
                     "hbm_gbs": 16 * d / (ms * 1e-3) / 1e9, "bytes_per_param": 16}
        grp.close()
        torch.cuda.empty_cache()
    except Exception as e:  # pragma: no cover
        out[name] = {"error": str(e)}
    return out


def run_extras_dist(args, world, rank, local, h, max_over_ranks, barrier):
    """Multi-GPU gossip (10M/worker, NVLink peer reads) and EASGD chain
    (25M/worker, center on GPU0)."""
    import torch
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group
    out = {}
    for name, proto, d in (("pull-gossip 10M/worker", N.PULL_GOSSIP, 10_000_000),
                           ("elastic-avg 25M/worker", N.ELASTIC_AVG, 25_000_000)):
        try:
            grp = Group.distributed(d, rank, world, local, dtype="f32",
                                    nccl=(proto == N.ELASTIC_AVG),  # center init = mean
                                    center=(proto == N.ELASTIC_AVG))
            gen = torch.Generator(device=f"cuda:{local}")
            gen.manual_seed(7 + rank)
            pool = [torch.randn(d, generator=gen, device=f"cuda:{local}") for _ in range(2)]
            grp.copy_in_async(0, N.BUF_THETA, pool[0].data_ptr(), d)
            grp.sync()
            if proto == N.ELASTIC_AVG:
                grp.ea_init_center()
            grp.seed_streams(1, "run/trial0")
            ptrs = [t.data_ptr() for t in pool]
            grp.run_rounds(proto, h, 3, grad_pool=ptrs)
            grp.sync()
            barrier()
            stream = torch.cuda.ExternalStream(grp.stream(), device=f"cuda:{local}")
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            k = 20
            torch.cuda.synchronize()
            barrier()
            e0.record(stream)
            grp.run_rounds(proto, h, k, grad_pool=ptrs)
            e1.record(stream)
            grp.sync()
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1)) / k
            hbm, _ = peaks()
            nv = 770.0
            if proto == N.PULL_GOSSIP:
                # the rounds' partner maps (same reference streams as the run):
                # GPU i reads 4 B/param from its partner and serves 4 B/param to
                # each remote puller; bound per round = slowest GPU's NVLink / HBM
                from paper_1611_04581_b200.engine import Stream, draw_pull_partners
                st = [Stream.make(1, "run/trial0", i, "partner-choice") for i in range(world)]
                t_bound = t_raw = 0.0
                for r in range(3 + k):
                    pm = draw_pull_partners(st) if r > 0 else list(range(world))
                    if r < 3:
                        continue
                    worst = raw_worst = 0.0
                    for i in range(world):
                        pullers = sum(1 for q in range(world) if pm[q] == i and q != i)
                        nin = 4 * d if pm[i] != i else 0
                        t_nv = max(nin, 4 * d * pullers) / (nv * 1e9)
                        t_hbm = (20 + 4 * pullers) * d / (hbm * 1e9)
                        worst = max(worst, t_nv, t_hbm)
                        # raw link: bulk peer reads carry 1.125 raw bytes per
                        # data byte in, plus 0.1875 of read requests out
                        raw_in, raw_out = 1.125 * nin, 1.125 * 4 * d * pullers + 0.1875 * nin
                        raw_worst = max(raw_worst, max(raw_in, raw_out) / (RAW_CEIL * 1e9),
                                        t_hbm)
                    t_bound += worst
                    t_raw += raw_worst
                bound_ms = t_bound / k * 1e3
                raw_ms = t_raw / k * 1e3
            else:
                # chain: every rank 24 B/param HBM + 4 B/param center over NVLink
                bound_ms = max(24 * d / (hbm * 1e9), 4 * d / (nv * 1e9)) * 1e3
                # raw link: 16-B peer stores carry 1.196 raw bytes per data byte
                raw_ms = max(24 * d / (hbm * 1e9), 1.196 * 4 * d / (RAW_CEIL * 1e9)) * 1e3
            out[name] = {"ms_per_round": ms, "param_updates_per_s": world * d / (ms * 1e-3),
                         "roofline_ms_per_round": bound_ms, "frac_of_roofline": bound_ms / ms,
                         "raw_link_ms_per_round": raw_ms, "frac_of_raw_link": raw_ms / ms,
                         "raw_link_note": f"packet overhead per access type and a {RAW_CEIL:.0f} "
                                          "GB/s raw ceiling from prior ncu link-counter captures "
                                          "(profiles/r2_nvlink_ncu.md)"}
            barrier()
            grp.close()
            del pool
            torch.cuda.empty_cache()
        except Exception as e:  # pragma: no cover
            out[name] = {"error": str(e)}
    return out


if __name__ == "__main__":
    main()
