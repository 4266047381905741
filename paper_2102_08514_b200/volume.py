"""Volume documents -> coset grids in HBM.

The reference's on-disk input format (`runtime.py:445-494`): an ASCII header

    splinevol 1 / lattice NAME / dim s / diag d... / cosets M / boundary B /
    per coset: shift ..., origin ..., extent ... / data

followed by the M coset arrays as little-endian float64, C order.  `write_volume` and
`read_volume` keep the reference's names, bytes and errors; `load_volume` is the
B200 loader: it reads the file straight into one pinned host buffer, ships the float64
payload to the device asynchronously and converts it there to the compute dtype, so a
C5-size volume (2x406^3 BCC = 1.07 GB of float64) costs one PCIe pass and no host-side
conversion.  The device layout is exactly the layout the kernels read:
one contiguous C-order array per coset, boundary policies resolved at staging time, so
no padding is materialised.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .lattice import CosetDecomposition
from .runtime import CoefficientGrid, RuntimeError_

VOL_MAGIC = b"splinevol 1"


def _header_lines(grid: CoefficientGrid, lattice_name: str) -> list:
    head = [
        VOL_MAGIC.decode(),
        f"lattice {lattice_name or grid.cosets.parent.name}",
        f"dim {grid.cosets.parent.s}",
        "diag " + " ".join(str(d) for d in grid.cosets.diag),
        f"cosets {grid.cosets.M}",
        f"boundary {grid.boundary}",
    ]
    for k in range(grid.cosets.M):
        head.append("shift " + " ".join(str(v) for v in grid.cosets.shifts[k]))
        head.append("origin " + " ".join(str(v) for v in grid.origins[k]))
        head.append("extent " + " ".join(str(v) for v in grid.arrays[k].shape))
    head.append("data")
    return head


def write_volume(grid: CoefficientGrid, lattice_name: str = "") -> bytes:
    """runtime.py:448-467: header + float64 little-endian payload (device arrays are
    widened to float64 on the device and copied back once per coset)."""
    parts = [("\n".join(_header_lines(grid, lattice_name)) + "\n").encode()]
    for a in grid.arrays:
        parts.append(a.to(torch.float64).contiguous().cpu().numpy().astype("<f8", copy=False).tobytes(order="C"))
    return b"".join(parts)


def parse_header(data) -> tuple:
    """(fields, payload offset) of a volume document; runtime.py:470-482."""
    mv = memoryview(data)
    raw = bytes(mv[: min(len(mv), 1 << 16)])
    at = raw.find(b"data\n")
    if at < 0:
        raise RuntimeError_("not a volume document")
    nl = at + len(b"data\n")
    head = raw[:nl].decode().splitlines()
    if head[0] != VOL_MAGIC.decode():
        raise RuntimeError_("not a volume document")
    fields: dict = {"shift": [], "origin": [], "extent": []}
    for line in head[1:-1]:
        key, *rest = line.split()
        if key in ("shift", "origin", "extent"):
            fields[key].append(tuple(int(v) for v in rest))
        else:
            fields[key] = rest
    return fields, nl


def _check(fields: dict, cosets: CosetDecomposition) -> None:
    """runtime.py:483-487 (same checks, same errors)."""
    s = int(fields["dim"][0])
    if s != cosets.parent.s or tuple(int(v) for v in fields["diag"]) != tuple(cosets.diag):
        raise RuntimeError_("volume lattice does not match the coset decomposition")
    if tuple(fields["shift"]) != tuple(tuple(v) for v in cosets.shifts):
        raise RuntimeError_("volume coset shifts do not match")


def read_volume(data, cosets: CosetDecomposition, *, device=None, dtype: torch.dtype = torch.float64) -> CoefficientGrid:
    """runtime.py:470-494 on an in-memory document; the grid lands on `device` (default:
    the current CUDA device) in `dtype` (float64 like the reference, or float32)."""
    fields, pos = parse_header(data)
    _check(fields, cosets)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    arrays = []
    for extent in fields["extent"]:
        count = int(np.prod(extent))
        host = torch.from_numpy(np.frombuffer(data, dtype="<f8", count=count, offset=pos).copy())
        arrays.append(host.to(dev).to(dtype).reshape(extent))
        pos += count * 8
    return CoefficientGrid(cosets, arrays, fields["origin"], boundary=fields["boundary"][0], device=dev, dtype=dtype)


def load_volume(path: str, cosets: CosetDecomposition, *, device=None, dtype: torch.dtype = torch.float32,
                stream: torch.cuda.Stream | None = None) -> CoefficientGrid:
    """Volume file -> device coset grid: file read into one pinned buffer (readinto, no
    intermediate copies), one asynchronous H2D copy of the float64 payload per coset on
    `stream`, float64 -> `dtype` conversion on the device.  Returns when the grid is
    ready (the stream is synchronised)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    size = os.path.getsize(path)
    buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb", buffering=0) as fh:
        view = memoryview(buf.numpy())
        got = 0
        while got < size:
            r = fh.readinto(view[got:])
            if not r:
                raise RuntimeError_("truncated volume file")
            got += r
    fields, pos = parse_header(buf.numpy())
    _check(fields, cosets)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    arrays = []
    with torch.cuda.stream(st):
        for extent in fields["extent"]:
            count = int(np.prod(extent))
            if pos + 8 * count > size:
                raise RuntimeError_("truncated volume file")
            raw = torch.empty(8 * count, dtype=torch.uint8, device=dev)
            raw.copy_(buf[pos: pos + 8 * count], non_blocking=True)
            arrays.append(raw.view(torch.float64).to(dtype).reshape(extent))
            pos += 8 * count
    st.synchronize()
    return CoefficientGrid(cosets, arrays, fields["origin"], boundary=fields["boundary"][0], device=dev, dtype=dtype)


def save_volume(path: str, grid: CoefficientGrid, lattice_name: str = "") -> None:
    """write_volume to a file."""
    with open(path, "wb") as fh:
        fh.write(write_volume(grid, lattice_name))
