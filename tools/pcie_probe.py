"""Raw PCIe copy timings with pinned buffers, repeated (per-process variance check)."""
import torch

n = 100_000_000
dev = torch.device("cuda", 0)
d = torch.empty((n, 3), dtype=torch.float32, device=dev)
o = torch.empty(n, dtype=torch.float32, device=dev)
for how in ("pin_memory()", "empty(pin_memory=True)"):
    if how == "pin_memory()":
        hp = torch.rand((n, 3)).pin_memory()
        ho = torch.empty(n).pin_memory()
    else:
        hp = torch.empty((n, 3), pin_memory=True)
        hp.copy_(torch.rand((n, 3)))
        ho = torch.empty(n, pin_memory=True)
    res = []
    for _ in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        d.copy_(hp, non_blocking=True)
        o2 = ho.copy_(o, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        res.append(round(s.elapsed_time(e), 1))
    print(how, "H2D 1.2GB + D2H 0.4GB (serial) ms:", res, flush=True)
