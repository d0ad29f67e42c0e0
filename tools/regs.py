"""Register / spill report of one translation unit (dev tool, CPU only).

    python tools/regs.py paper_2506_15976_b200/csrc/lbs_scan_fwd_bf16.cu [filter] [-D...]
"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("-D") else ""
defs = [a for a in sys.argv[2:] if a.startswith("-D")]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
       "--expt-relaxed-constexpr", "-I", "include", "-Xptxas", "-v", *defs, "-c", src, "-o", "/tmp/_regs.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name, spill = None, ""
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = name.replace("__nv_bfloat16", "bf16").replace("lbs::", "").replace("(lbs::FwdParams)", "").replace("(lbs::BwdParams)", "")
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and name and flt in name:
        print(f"{m.group(1):>4} regs {spill:>16}  {name}")
if "error" in out:
    print(out[-3000:])
