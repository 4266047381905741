"""Digests of the REFERENCE's lowered programs (build container only).

    python tests/golden/make_program_golden.py

For every catalog plan: the reference's own `deserialize_plan` (plancompile.py:542) and
`emit_kernel` (plancompile.py:702-703, the rendered `build_program`), frozen as sha256 + op
count in tests/golden/programs.json; tests/test_minilang.py requires our `emit_kernel` to
produce the same document.  /root/reference does not travel to the GPU box; this file does.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

PLANS = os.path.join(ROOT, "paper_2102_08514_b200", "plans")


def main():
    import_reference()
    from splineplan.plancompile import build_program, deserialize_plan

    out = {}
    for f in sorted(os.listdir(PLANS)):
        if not f.endswith(".plan.json"):
            continue
        name = f[: -len(".plan.json")]
        plan = deserialize_plan(open(os.path.join(PLANS, f)).read())
        prog = build_program(plan)
        text = prog.render()
        out[name] = {"sha256": hashlib.sha256(text.encode()).hexdigest(), "ops": len(prog.ops), "bytes": len(text)}
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
