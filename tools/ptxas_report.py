"""Per-kernel registers / spills from `build.py --force --verbose` (ptxas -v)."""
import re, subprocess, sys
out = subprocess.run([sys.executable, "paper_1711_04325_b200/build.py", "--force", "--verbose"],
                     capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"lmsgd::\(anonymous namespace\)::|\(.*", "", name).replace("void ", "")
    m = re.search(r"(\d+) bytes spill stores", line)
    if m: spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{name:32s} regs={m.group(1):>3s} spill={spill}")
        name = None
