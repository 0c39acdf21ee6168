import torch, time
d = 25_000_000
h = [torch.randn(d).pin_memory() for _ in range(2)]
dv = [torch.empty(d, device="cuda") for _ in range(2)]
for nst in (1, 2, 4):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in sts: st.wait_event(e0)
        for s in range(20):
            n = d // nst
            for q, st in enumerate(sts):
                with torch.cuda.stream(st):
                    dv[s % 2][q * n:(q + 1) * n].copy_(h[s % 2][q * n:(q + 1) * n], non_blocking=True)
        for st in sts:
            ev = torch.cuda.Event(); ev.record(st); torch.cuda.current_stream().wait_event(ev)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    print(f"streams={nst}: {best:.3f} ms per 100 MB -> {4*d/best/1e6:.1f} GB/s")
