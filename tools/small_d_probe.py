"""Where a small-d round's time goes (configs[4] 1M-4M rows): per round,
the host time to issue it (dsgd_run_rounds returns once everything is
enqueued) against the device time (CUDA events on the library stream),
max over ranks.  Host-bound when the two are equal.

    torchrun --nproc-per-node N tools/small_d_probe.py [--sizes 1e6,4e6]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e6,4e6")
    ap.add_argument("--rounds", type=int, default=200)
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
    for d in [int(float(x)) for x in a.sizes.split(",")]:
        for name in a.protocols.split(","):
            proto = protos[name]
            g = Group.distributed(d, rank, world, local, dtype="f32", nccl=True, grad=True,
                                  center=proto == N.ELASTIC_AVG)
            pool = [torch.randn(d, device=f"cuda:{local}") for _ in range(2)]
            ptrs = [t.data_ptr() for t in pool]
            g.copy_in_async(0, N.BUF_THETA, pool[0].data_ptr(), d)
            g.sync()
            if proto == N.ELASTIC_AVG:
                g.ea_init_center()
            g.seed_streams(1, "run/trial0")
            g.run_rounds(proto, h, 20, grad_pool=ptrs)
            g.sync()
            dist.barrier()
            stream = torch.cuda.ExternalStream(g.stream(), device=f"cuda:{local}")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t0 = time.perf_counter()
            g.run_rounds(proto, h, a.rounds, grad_pool=ptrs)
            host = (time.perf_counter() - t0) / a.rounds
            e1.record(stream)
            g.sync()
            torch.cuda.synchronize()
            dev = e0.elapsed_time(e1) / a.rounds * 1e-3
            t = torch.tensor([host, dev], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            launches = g.launch_count()[0]
            if rank == 0:
                print(json.dumps({"tool": "small_d_probe", "gpus": world, "protocol": name, "d": d,
                                  "host_us_per_round": t[0].item() * 1e6,
                                  "device_us_per_round": t[1].item() * 1e6,
                                  "backend": g.allreduce_info()[0],
                                  "kernels_total": launches}), flush=True)
            g.close()
            del pool
            torch.cuda.empty_cache()
            dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
