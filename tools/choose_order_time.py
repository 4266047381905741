"""Time runtime.choose_order (the order="auto" heuristic) on a 4M-point device batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch
from paper_2102_08514_b200.runtime import choose_order
dev = torch.device("cuda", 0)
p = torch.rand((1 << 22, 3), device=dev) * 256
for _ in range(3): choose_order(p)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20): choose_order(p)
torch.cuda.synchronize(); print("choose_order ms", (time.perf_counter() - t) / 20 * 1e3, choose_order(p))
