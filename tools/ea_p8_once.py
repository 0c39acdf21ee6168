"""configs[2] on one GPU for a profiler: p = 8 nodes x 25M fp32 in one
context (+ center), a few EASGD rounds through dsgd_run_rounds (external
gradient pool), for `ncu -k regex:k_ea_local`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1611_04581_b200 import _native as N
    from paper_1611_04581_b200.engine import Group, Hyperparams
    d, p = 25_000_000, 8
    g = Group(d, p, dtype="f32", grad=True, center=True, device=0)
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(3)
    pool = [torch.randn(d, generator=gen, device="cuda:0") for _ in range(2)]
    for i in range(p):
        g.copy_in_async(i, N.BUF_THETA, pool[i % 2].data_ptr(), d)
    g.sync()
    g.ea_init_center()
    g.seed_streams(1, "run/trial0")
    h = Hyperparams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    g.run_rounds(N.ELASTIC_AVG, h, 4, grad_pool=[t.data_ptr() for t in pool])
    g.sync()
    g.close()
    print("ok")


if __name__ == "__main__":
    main()
