"""Registers / spills per kernel from build/ptxas.log."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "build/ptxas.log").read().splitlines()
name = None
for i, line in enumerate(log):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = re.sub(r"sp::EvalArgs<\w+>", "", name).replace("sp::", "")
    m = re.search(r"Used (\d+) registers", line)
    if m and name and ("kernel" in name):
        spill = log[i - 1].strip() if "spill" in log[i - 1] else ""
        sp = re.search(r"(\d+) bytes spill stores", spill)
        print(f"{int(m.group(1)):4d} regs  spill={sp.group(1) if sp else '?':>4}  {name[:110]}")
        name = None
