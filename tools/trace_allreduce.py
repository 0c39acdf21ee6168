"""Timeline of the multi-GPU all-reduce kernels (device %globaltimer stamps).

    DSGD_TRACE=4096 torchrun --nproc-per-node N tools/trace_allreduce.py [--d 25000000]

Per rank, per launch: wait = after_wait - entry, work = done - after_wait.
Writes gpurun_out/trace_rank<r>.npy and prints a per-kernel summary."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", "--params", dest="d", type=int, default=25_000_000)
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--protocol", default="all-reduce",
                    choices=["all-reduce", "pull-gossip", "elastic-avg"])
    a = ap.parse_args()
    os.environ.setdefault("DSGD_TRACE", "4096")
    import torch
    import torch.distributed as dist
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    proto = {"all-reduce": N.ALLREDUCE, "pull-gossip": N.PULL_GOSSIP,
             "elastic-avg": N.ELASTIC_AVG}[a.protocol]
    g = Group.distributed(a.d, rank, world, local, dtype="f32", grad=True,
                          center=proto == N.ELASTIC_AVG)
    pool = [torch.randn(a.d, device="cuda") for _ in range(2)]
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    if proto == N.ELASTIC_AVG:
        g.ea_init_center()
    g.seed_streams(1, "run/trial0")
    g.run_rounds(proto, h, 5, grad_pool=[t.data_ptr() for t in pool])
    g.sync()
    dist.barrier()
    g.run_rounds(proto, h, a.rounds, grad_pool=[t.data_ptr() for t in pool])
    g.sync()
    tr = g.trace_dump()
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/trace_rank{rank}.npy", tr)
    rows = tr[tr[:, 1] >= 5]  # skip warm-up rounds
    names = {int(k): n for k, n in enumerate(N.KERNEL_NAMES)}
    out = [f"rank {rank} backend {getattr(g, 'allreduce_backend', '?')}"]
    kinds = sorted(set(int(x) for x in rows[:, 0]))
    for kd in kinds:
        r = rows[rows[:, 0] == kd].astype(np.float64)
        wait = (r[:, 3] - r[:, 2]) / 1e3
        work = (r[:, 4] - r[:, 3]) / 1e3
        out.append(f"  {names.get(kd % 16, kd)}[pipe {kd // 16}] n={len(r)} wait {np.median(wait):7.1f} us "
                   f"work {np.median(work):7.1f} us")
    t = rows[:, 2:5].astype(np.float64)
    if len(t):
        span = (t.max() - t.min()) / 1e3
        out.append(f"  span {span:.1f} us over {a.rounds} rounds = {span / a.rounds:.1f} us/round")
        # launch gap: the next kernel's entry stamp after this one's done stamp
        order = np.argsort(t[:, 0])
        ts = t[order]
        gaps = (ts[1:, 0] - ts[:-1, 2]) / 1e3
        if len(gaps):
            out.append(f"  entry(k+1) - done(k): median {np.median(gaps):.1f} us "
                       f"(negative = overlapped by programmatic dependent launch)")
        # per round: first entry to last done
    res = [None] * world
    dist.all_gather_object(res, "\n".join(out))
    if rank == 0:
        print("\n".join(res), flush=True)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
