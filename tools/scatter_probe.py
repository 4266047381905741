"""Random 4-byte scatter of 1e8 values: direct vs L2-blocked windows (CUDA events).

Measured (round 2): direct 3.8 ms, 16M-element windows 2.2 ms (the protocol-B default).  A
radix partition by window before a single scatter pass was measured too: the partition is
0.56 ms but the scatter of window-grouped pairs still took 3.5 ms, so it was dropped."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_08514_b200 import _native  # noqa: E402


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


n = 100_000_000
dev = torch.device("cuda", 0)
src = torch.rand(n, device=dev)
perm = torch.randperm(n, device=dev, dtype=torch.int64).to(torch.int32)
out = torch.empty(n, device=dev)
lib = _native.lib()
st = torch.cuda.current_stream().cuda_stream
ref = torch.empty(n, device=dev)
ref[perm.long()] = src
print(f"torch index_put: {timed(lambda: ref.__setitem__(perm.long(), src)):.3f} ms")
for w in (0, 64 << 20, 32 << 20, 16 << 20, 8 << 20, 4 << 20):
    t = timed(lambda: lib.sp_scatter32_blocked(src.data_ptr(), perm.data_ptr(), n, _native.SP_F32, w, out.data_ptr(), st))
    ok = torch.equal(out, ref)
    print(f"window {w / 1e6 if w else n / 1e6:7.1f} M elems: {t:.3f} ms  equal={ok}")

