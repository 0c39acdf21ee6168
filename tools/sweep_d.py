"""configs[4]: parameter-size sweep d = 1M .. 1B fp32 per worker for gossip vs
EASGD vs all-reduce, one worker per GPU (run under torchrun, N = 2/4/8).

    torchrun --nproc-per-node N tools/sweep_d.py [--sizes 1e6,4e6,...] [--rounds 20]

Prints one JSON line per (protocol, d) on rank 0 with the max-over-ranks
device time per round (CUDA events on the library stream), whole-job
param-updates/s and the round's roofline time (HBM 6551 GB/s measured copy,
NVLink 770 GB/s measured peer copy)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e6,4e6,16e6,64e6,256e6,1e9")
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--protocols", default="all-reduce,pull-gossip,elastic-avg")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h = Hyperparams(alpha0=0.05, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    protos = {"all-reduce": N.ALLREDUCE, "pull-gossip": N.PULL_GOSSIP,
              "elastic-avg": N.ELASTIC_AVG}
    hbm, nv = 6551.0, 770.0
    for d in [int(float(x)) for x in a.sizes.split(",")]:
        for name in a.protocols.split(","):
            proto = protos[name]
            try:
                g = Group.distributed(d, rank, world, local, dtype="f32",
                                      nccl=proto != N.PULL_GOSSIP,
                                      quadratic=True, center=proto == N.ELASTIC_AVG)
                gen = torch.Generator(device=f"cuda:{local}")
                gen.manual_seed(11 + rank)
                th = torch.randn(d, generator=gen, device=f"cuda:{local}")
                g.copy_in_async(0, N.BUF_THETA, th.data_ptr(), d)
                g.sync()
                del th
                if proto == N.ELASTIC_AVG:
                    g.ea_init_center()
                g.seed_streams(1, "run/trial0")
                # quadratic objective with s = opt = 0 buffers (zeros) + device noise:
                # the gradient term is the in-kernel Philox noise (synthetic gradient)
                noise = ("device", 1.0, 5)
                _run(g, proto, h, 3, noise)
                g.sync()
                dist.barrier()
                s = torch.cuda.ExternalStream(g.stream(), device=f"cuda:{local}")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                _run(g, proto, h, a.rounds, noise)
                e1.record(s)
                g.sync()
                torch.cuda.synchronize()
                t = torch.tensor([e0.elapsed_time(e1) / a.rounds], device="cuda",
                                 dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
                if proto == N.ALLREDUCE:
                    be = getattr(g, "allreduce_backend", "")
                    nvb = (world - 1) * 4 * d if be == "oneshot" else (
                        (1 + 1 / world) * 4 * d if be == "nvls" else 2 * (world - 1) / world * 4 * d)
                    bound = max(24 * d / (hbm * 1e9), nvb / (nv * 1e9))
                elif proto == N.ELASTIC_AVG:
                    be = "chain"
                    bound = max(28 * d / (hbm * 1e9), 4 * d / (nv * 1e9))
                else:
                    be = "peer-read"
                    bound = gossip_bound(world, d, 3, a.rounds, hbm, nv)
                if rank == 0:
                    print(json.dumps({"protocol": name, "backend": be, "d": d, "gpus": world,
                                      "ms_per_round": ms,
                                      "param_updates_per_s": world * d / (ms * 1e-3),
                                      "roofline_ms": bound * 1e3,
                                      "frac_of_roofline": bound * 1e3 / ms}), flush=True)
                g.close()
                torch.cuda.empty_cache()
            except Exception as e:  # pragma: no cover
                if rank == 0:
                    print(json.dumps({"protocol": name, "d": d, "error": str(e)}), flush=True)
            dist.barrier()
    dist.destroy_process_group()


def gossip_bound(world, d, warm, rounds, hbm, nv):
    """Mean over the timed rounds of the busiest GPU's bound, from the
    rounds' actual partner maps (the reference partner streams the run
    draws): GPU i reads 4 B/param from a remote partner and serves 4 B/param
    to each remote puller over NVLink, and streams (24 + 4 r_i) B/param of
    HBM (quadratic objective: theta, delta, s, opt read, theta', delta'
    written, + the snapshot served to r_i pullers)."""
    from paper_1611_04581_b200.engine import Stream, draw_pull_partners
    st = [Stream.make(1, "run/trial0", i, "partner-choice") for i in range(world)]
    total = 0.0
    for r in range(warm + rounds):
        pm = draw_pull_partners(st) if r > 0 else list(range(world))  # round 0: ungated
        if r < warm:
            continue
        worst = 0.0
        for i in range(world):
            pullers = sum(1 for q in range(world) if pm[q] == i and q != i)
            t_in = (4 * d if pm[i] != i else 0) / (nv * 1e9)
            t_out = 4 * d * pullers / (nv * 1e9)
            t_hbm = (24 + 4 * pullers) * d / (hbm * 1e9)
            worst = max(worst, t_in, t_out, t_hbm)
        total += worst
    return total / rounds


def _run(g, proto, h, rounds, noise):
    """run_rounds with the quadratic objective (s = opt = 0, so the model
    gradient is zero) plus device Philox noise: a synthetic N(0,1) gradient
    generated inside the update kernel (no gradient buffer traffic)."""
    from paper_1611_04581_b200 import _native as N
    import ctypes as C
    gs = g._grad("quadratic", noise, False)
    rd = N.RunDesc(proto, h.to_c(), N.SCOPE_AGGREGATE, gs, 0, None, 0.0, rounds)
    rd._keep = gs
    N.check(g.lib.dsgd_run_rounds(g._ctx, C.byref(rd)))


if __name__ == "__main__":
    main()
