"""Grid-size sweep of the fused update kernels on one GPU (CUDA events).

    python tools/kernel_sweep.py [--d 25000000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=25_000_000)
    ap.add_argument("--bps", default="2,3,4,5,6,8,12,16")
    ap.add_argument("--rounds", type=int, default=200)
    a = ap.parse_args()
    import torch
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4)
    d = a.d
    pool = [torch.randn(d, device="cuda") for _ in range(4)]
    res = []
    for bps in [int(x) for x in a.bps.split(",")]:
        os.environ["DSGD_BLOCKS_PER_SM"] = str(bps)
        for name, proto, p, dd, bpp in (("allreduce p=1", N.ALLREDUCE, 1, d, 20),
                                        ("pull p=8", N.PULL_GOSSIP, 8, d // 2.5, 24),
                                        ("ea p=8", N.ELASTIC_AVG, 8, d // 2.5, 20)):
            dd = int(dd)
            g = Group(dd, p, dtype="f32", center=proto == N.ELASTIC_AVG)
            ptrs = [t.data_ptr() for t in pool[:min(4, p)]] * (1 if p >= 4 else 1)
            ptrs = (ptrs * ((p + len(ptrs) - 1) // len(ptrs)))[:p] if p > 1 else ptrs
            g.seed_streams(1, "run/trial0")
            g.run_rounds(proto, h, 5, grad_pool=ptrs)
            g.sync()
            s = torch.cuda.ExternalStream(g.stream())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.run_rounds(proto, h, a.rounds, grad_pool=ptrs)
            e1.record(s)
            g.sync()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.rounds
            gbs = p * dd * bpp / (ms * 1e-3) / 1e9
            res.append({"bps": bps, "kernel": name, "us": ms * 1e3, "gbs": gbs})
            print(json.dumps(res[-1]), flush=True)
            g.close()


if __name__ == "__main__":
    main()
