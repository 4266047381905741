"""Build libsplinerecon.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2102_08514_b200.build [--verbose]

1. code-generates one translation unit per catalog plan the generator supports
   (codegen.py) into csrc/generated/,
2. compiles every TU with  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
   (in parallel), and links paper_2102_08514_b200/libsplinerecon.so.
The ptxas resource report (registers / spills / smem per kernel) is kept in
build/ptxas.log.
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


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        with open(p, "rb") as fh:
            h.update(p.encode())
            h.update(fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def _compile(src: str, obj: str) -> tuple:
    cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r.returncode, r.stdout + r.stderr, " ".join(cmd)


def build(verbose: bool = False, force: bool = False) -> str:
    from .codegen import write_generated

    gen_tus = write_generated(_catalog_plans(), GEN)
    tus = [os.path.join(CSRC, "splinerecon.cu"), os.path.join(CSRC, "sp_texture.cu"),
           os.path.join(CSRC, "sp_prefilter.cu"), os.path.join(CSRC, "sp_render.cu")] + gen_tus
    deps = tus + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(GEN, "registry.inc"),
                                                           os.path.join(ROOT, "include", "splinerecon.h")]
    digest = _digest(deps)
    stamp = os.path.join(BUILD, "libsplinerecon.sha256")
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == digest:
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = [os.path.join(BUILD, os.path.basename(t).replace(".cu", ".o")) for t in tus]
    logs = []
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        for src, rc, log, cmd in ex.map(lambda a: _compile(*a), zip(tus, objs)):
            logs.append(f"### {cmd}\n{log}")
            if rc != 0:
                sys.stderr.write(log)
                raise RuntimeError(f"nvcc failed on {src}")
    with open(os.path.join(BUILD, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    link = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    with open(stamp, "w") as fh:
        fh.write(digest)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
