"""Library baseline for the all-reduce step: ncclAllReduce (torch.distributed,
NCCL's own algorithm choice, or NCCL_ALGO=...) of a d-element fp32 vector per
rank, CUDA-event timed, max over ranks.  One process per GPU (torchrun).

    torchrun --nproc-per-node 4 tools/nccl_allreduce_probe.py [--d 25000000]

This is the "only calls NCCL" baseline the fused kernels are compared with:
it moves the bytes of the average alone, with no update math.
"""
import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=25_000_000)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--op", default="avg", choices=["avg", "sum"])
    a = ap.parse_args()
    op = dist.ReduceOp.AVG if a.op == "avg" else dist.ReduceOp.SUM
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    x = torch.randn(a.d, device="cuda")
    for _ in range(a.warmup):
        dist.all_reduce(x, op=op)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        dist.all_reduce(x, op=op)
    e1.record()
    torch.cuda.synchronize()
    us = torch.tensor([e0.elapsed_time(e1) / a.iters * 1e3], device="cuda")
    dist.all_reduce(us, op=dist.ReduceOp.MAX)
    if rank == 0:
        t = us.item()
        algbw = a.d * 4 / (t * 1e-6) / 1e9
        print(json.dumps({"tool": "nccl_allreduce_probe", "gpus": world, "d": a.d,
                          "nccl_algo": os.environ.get("NCCL_ALGO", "auto"), "op": a.op,
                          "us_per_allreduce": t, "algbw_gbs": algbw,
                          "busbw_gbs": algbw * 2 * (world - 1) / world}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
