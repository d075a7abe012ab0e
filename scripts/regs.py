"""ptxas register / spill report per kernel of one csrc/*.cu file (sm_100a)."""
import re, subprocess, sys
src = sys.argv[1]
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
                    "--expt-relaxed-constexpr", "-c", src, "-o", "/tmp/_regs.o"], capture_output=True, text=True)
name = None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"saga::\(anonymous namespace\)::", "", name)
        name = name.split("(")[0] if "k_segreduce" not in name else name.split(">(")[0] + ">"
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{m.group(1):>4} regs  spill {spill:>4}  {name}")
        name = None
if r.returncode:
    print(r.stderr)
