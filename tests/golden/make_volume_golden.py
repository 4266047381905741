"""Volume-document fixtures made by the REFERENCE itself (build container only).

    python tests/golden/make_volume_golden.py

For CC3 / BCC / FCC grids (seeded, small) this runs the reference `write_volume`
(runtime.py:448-467) and stores the bytes in tests/golden/volume/<lattice>_<boundary>.bin,
with the seeded arrays and origins in tests/golden/volume/fixtures.npz, so that the B200 loader
(`paper_2102_08514_b200.volume`) can be checked byte-for-byte without /root/reference.
"""
import os
import sys

import numpy as np

GOLD = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(GOLD))
HERE = os.path.join(GOLD, "volume")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

CASES = [("CC3", "zero", 7), ("BCC", "mirror", 9), ("FCC", "clamp", 9)]


def main():
    import_reference()
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.runtime import CoefficientGrid, read_volume, write_volume

    rng = np.random.default_rng(2102_08514)
    os.makedirs(HERE, exist_ok=True)
    payload = {}
    for lat_name, boundary, hi in CASES:
        cos = decompose_cartesian(named_lattice(lat_name))
        base = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], boundary)
        arrays = [rng.standard_normal(a.shape) for a in base.arrays]  # full float64 payloads
        grid = CoefficientGrid(cos, arrays, base.origins, boundary)
        data = write_volume(grid)
        back = read_volume(data, cos)
        assert all(np.array_equal(a, b) for a, b in zip(arrays, back.arrays))
        tag = f"{lat_name}_{boundary}"
        with open(os.path.join(HERE, f"{tag}.bin"), "wb") as fh:
            fh.write(data)
        payload[f"{tag}_origins"] = np.array(base.origins, dtype=np.int64)
        for k, a in enumerate(arrays):
            payload[f"{tag}_coset{k}"] = a
        print(tag, len(data), "bytes")
    np.savez_compressed(os.path.join(HERE, "fixtures.npz"), **payload)


if __name__ == "__main__":
    main()
