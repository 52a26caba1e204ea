"""SASS evidence for the shipped library (no GPU needed): per kernel, registers / stack / shared memory
(cuobjdump -res-usage) and the memory-instruction histogram (cuobjdump -sass), plus the inner loop of
the production stencil.  Usage: python scripts/sass_summary.py [lib] > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2211_15716_b200/libigg.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True, check=True).stdout
demangle = lambda s: subprocess.run(["c++filt", s], capture_output=True, text=True).stdout.strip()
usage = {}
for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", res):
    usage[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(4)))
funcs = re.split(r"\n\s*Function : ", sass)[1:]
KEY = re.compile(r"\b(LDG[\w.]*|STG[\w.]*|LDGSTS[\w.]*|LDS[\w.]*|STS[\w.]*|UBLKCP[\w.]*|UTMA\w*|DFMA|DADD|DMUL|"
                 r"MEMBAR[\w.]*|FENCE[\w.]*|ATOMG?[\w.]*|RED[\w.]*|NANOSLEEP|SHFL[\w.]*|BAR[\w.]*|LDGDEPBAR|DEPBAR[\w.]*)\b")
print(f"# SASS summary of {lib} (cuobjdump, sm_100a)\n")
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if "igg" not in name:
        continue
    h = collections.Counter(m.group(1) for m in KEY.finditer(f))
    r = usage.get(name, ("?", "?", "?"))
    print(f"## {demangle(name)}\n   REG {r[0]}  STACK {r[1]}  SHARED {r[2]}")
    print("   " + ", ".join(f"{k} {v}" for k, v in sorted(h.items())))
    print()
# the production stencil's inner loop: the instructions between the loop's backward branch target and
# the branch (the longest backward branch in heat_box_async_kernel<4,3,1>)
box = next(f for f in funcs if f.startswith("_ZN3igg21heat_box_async_kernelILi4ELi3ELb1E"))
body = box.split("\n")
ins = [(int(m.group(1), 16), l) for l in body for m in [re.search(r"/\*([0-9a-f]{4})\*/", l)] if m]
best = None
for a, l in ins:
    t = re.search(r"BRA 0x([0-9a-f]+)", l)
    if t and int(t.group(1), 16) < a and (best is None or a - int(t.group(1), 16) > best[1] - best[0]):
        best = (int(t.group(1), 16), a)
if best:
    loop = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).strip() for a, l in ins if best[0] <= a <= best[1]]
    h = collections.Counter(m.group(1) for x in loop for m in KEY.finditer(x))
    print(f"## heat_box_async_kernel<4,3,1>: inner z loop, {len(loop)} instructions "
          f"(0x{best[0]:x}..0x{best[1]:x}); " + ", ".join(f"{k} {v}" for k, v in sorted(h.items())) + "\n")
    for x in loop:
        print("   " + x)
