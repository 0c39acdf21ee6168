"""Per-step time of the N = 1 all-reduce round with and without per-launch
profiling events (the events sit between consecutive kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    d = 25_000_000
    g = Group(d, 1, dtype="f32", grad=True)
    pool = [torch.randn(d, device="cuda") for _ in range(4)]
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4)
    ptrs = [t.data_ptr() for t in pool]
    s = torch.cuda.ExternalStream(g.stream())
    for prof in (False, True, False, True):
        g.profile(prof)
        g.run_rounds(N.ALLREDUCE, h, 20, grad_pool=ptrs)
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.run_rounds(N.ALLREDUCE, h, 200, grad_pool=ptrs)
        e1.record(s)
        g.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 200
        extra = ""
        if prof:
            kms, kn = g.profile_read(N.KERNEL_NAMES.index("allreduce_local"), reset=True)
            extra = f" kernel {kms / kn * 1e3:.1f} us"
        print(f"profile={prof}: {ms * 1e3:.1f} us/step{extra}", flush=True)
        g.profile(False)
    # the per-call API path (one dsgd_allreduce_round per step, no run loop)
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(200):
            g.allreduce_round(h, grad=[ptrs[i % 4]])
        e1.record(s)
        g.sync()
        torch.cuda.synchronize()
        print(f"per-call: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us/step", flush=True)


if __name__ == "__main__":
    main()
