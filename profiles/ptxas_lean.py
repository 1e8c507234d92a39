"""ptxas -v summary of the gate_eval_lean instances: registers, stack, spills.

    python profiles/ptxas_lean.py
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

cmd = [g._nvcc(), *g.NVCC_FLAGS, "-I", os.path.join(ROOT, "include"),
       os.path.join(g.CSRC, "glsim_cuda.cu"), "-o", "/tmp/ptxas_probe.so"]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur and "gate_eval_lean" in cur:
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            stack = m.groups()
        m2 = re.search(r"Used (\d+) registers", line)
        if m2:
            inst = re.search(r"gate_eval_leanILi(\d)ELi(\d)ELb(\d)", cur).groups()
            print(f"MODE {inst[0]} K {inst[1]} PCT100 {inst[2]}: regs {m2.group(1)}, "
                  f"stack {stack[0]}, spill st/ld {stack[1]}/{stack[2]}")
            cur = None
