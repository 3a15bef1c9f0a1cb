"""Compile one .cu with -Xptxas -v and print a registers / spill table per
entry function (demangled, filtered by a substring)."""
import re
import subprocess
import sys

src, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
       "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr", "-Iinclude", "-c", src, "-o", "/dev/null"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr.splitlines()
name = None
for ln in out:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
        continue
    if name and "spill" in ln:
        spill = ln.split(":", 1)[-1].strip()
    if name and "registers" in ln:
        regs = re.search(r"Used (\d+) registers", ln).group(1)
        smem = re.search(r"(\d+) bytes smem", ln)
        if pat in name:
            short = name.replace("(anonymous namespace)::", "")
            short = re.sub(r"\((?:[^()]|\([^()]*\))*\)$", "", short)
            short = short.replace("void ", "")
            print(f"{regs:>4} regs  {spill:60s} {short}")
        name = None
