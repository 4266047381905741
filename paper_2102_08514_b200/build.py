"""Build libsplinerecon.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2102_08514_b200.build [--verbose] [--force] [--checked]

1. code-generates one translation unit per catalog plan the generator supports
   (codegen.py) into csrc/generated/,
2. compiles every TU with  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
   (in parallel), and links paper_2102_08514_b200/libsplinerecon.so.
The ptxas resource report (registers / spills / smem per kernel) is kept in
build/ptxas.log.  --checked builds libsplinerecon_checked.so instead: the same sources with
-DSP_BOUNDS_CHECK (device-side bounds checks on shared-tile, point and output indices that
trap with a message; load it with SP_CHECKED=1).
"""

from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
GEN = os.path.join(CSRC, "generated")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libsplinerecon.so")
LIB_CHECKED = os.path.join(PKG, "libsplinerecon_checked.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _catalog_plans():
    from .plan import deserialize_plan

    out = []
    for path in sorted(glob.glob(os.path.join(PKG, "plans", "*.plan.json"))):
        with open(path) as fh:
            out.append((os.path.basename(path)[: -len(".plan.json")], deserialize_plan(fh.read())))
    return out


def _digest(paths, flags) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        with open(p, "rb") as fh:
            h.update(p.encode())
            h.update(fh.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()


def _compile(src: str, obj: str, flags) -> tuple:
    cmd = [NVCC] + flags + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r.returncode, r.stdout + r.stderr, " ".join(cmd)


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> str:
    from .codegen import write_generated

    gen_tus = write_generated(_catalog_plans(), GEN)
    tus = [os.path.join(CSRC, "splinerecon.cu"), os.path.join(CSRC, "sp_texture.cu"),
           os.path.join(CSRC, "sp_prefilter.cu"), os.path.join(CSRC, "sp_render.cu")] + gen_tus
    deps = tus + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(GEN, "registry.inc"),
                                                           os.path.join(ROOT, "include", "splinerecon.h")]
    flags = FLAGS + (["-DSP_BOUNDS_CHECK"] if checked else [])
    lib_path = LIB_CHECKED if checked else LIB
    bdir = os.path.join(BUILD, "checked") if checked else BUILD
    digest = _digest(deps, flags)
    stamp = os.path.join(bdir, os.path.basename(lib_path).replace(".so", ".sha256"))
    if not force and os.path.exists(lib_path) and os.path.exists(stamp) and open(stamp).read() == digest:
        return lib_path
    os.makedirs(bdir, exist_ok=True)
    objs = [os.path.join(bdir, os.path.basename(t).replace(".cu", ".o")) for t in tus]
    logs = []
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        for src, rc, log, cmd in ex.map(lambda a: _compile(a[0], a[1], flags), zip(tus, objs)):
            logs.append(f"### {cmd}\n{log}")
            if rc != 0:
                sys.stderr.write(log)
                raise RuntimeError(f"nvcc failed on {src}")
    with open(os.path.join(bdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    link = [NVCC] + ARCH + ["-shared", "-o", lib_path] + objs + ["-lcudart"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    with open(stamp, "w") as fh:
        fh.write(digest)
    if verbose:
        print("\n".join(logs))
    return lib_path


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv, checked="--checked" in sys.argv))
