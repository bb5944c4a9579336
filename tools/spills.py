"""Registers / spills per kernel of libnlg (ptxas -v), demangled: python tools/spills.py [filter]"""
import re
import subprocess
import sys

cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
       "-fPIC", "-shared", "-Xptxas", "-v", "-I", "include", "-o", "/tmp/spills.so",
       "paper_2207_03921_b200/csrc/nlg.cu"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr.splitlines()
cur, rows = None, []
for line in out:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(anonymous namespace\)::", "", cur)
        spill = None
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = (int(m.group(1)), int(m.group(2)), int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for name, regs, sp in rows:
    if flt in name:
        print(f"{regs:4d} regs  stack {sp[0]:4d} spill st {sp[1]:4d} ld {sp[2]:4d}  {name[:150]}")
