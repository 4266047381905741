"""Run the C5-size BCC quintic prefilter a few times (for ncu).  python tools/prof_prefilter.py [hi]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_08514_b200 import corpus  # noqa: E402
from paper_2102_08514_b200.prefilter import apply_prefilter  # noqa: E402
from paper_2102_08514_b200.runtime import CoefficientGrid  # noqa: E402

hi = int(sys.argv[1]) if len(sys.argv) > 1 else 811
_, cos = corpus.lattice_of("bcc_quintic_rd")
grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi] * 3, device="cuda", dtype=torch.float32)
for a in grid.arrays:
    a.uniform_()
taps = corpus.prefilter_taps("bcc_quintic_rd")
out = apply_prefilter(grid, taps)
for _ in range(3):
    apply_prefilter(grid, taps, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    apply_prefilter(grid, taps, out=out)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"prefilter {hi}: {ms:.3f} ms/step, {2 * grid.nbytes() / ms / 1e6:.1f} GB/s")
