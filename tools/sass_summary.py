"""SASS evidence for the hot kernels of the built library: resource usage and the
instruction mix (DFMA, shared/global loads and stores, bulk copies, mbarrier ops,
local-memory spills) of each K1/K2/transfer instance, from cuobjdump.

    python tools/sass_summary.py [build/obj/k_sem.o] > profiles/r02/sass_summary.txt
"""
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "build/obj/k_sem.o"
WANT = re.compile(r"k_sem_k1_greg|k_sem_k2ILi7|k_sem_k1_axILi3|k_prolong_w|k_restrict_w")
res = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout.splitlines()
usage = {}
for i, line in enumerate(res):
    m = re.search(r"Function (\S+):", line)
    if m and i + 1 < len(res):
        usage[m.group(1)] = res[i + 1].strip()
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
OPS = ["DFMA", "DADD", "DMUL", "LDS", "STS", "LDG", "STG", "UBLKCP", "SYNCS", "LDL", "STL", "BAR.SYNC", "CCTL"]
print("# SASS of the hot kernels (cuobjdump, sm_100a):", obj)
print("# columns: instruction counts in the kernel body (static, not executed)")
excerpt = None
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not WANT.search(name):
        continue
    body = f.split("\n", 1)[1] if "\n" in f else ""
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", body)
    cnt = {op: sum(1 for x in ins if re.search(r"(^|\s|\})" + re.escape(op) + r"[\s.]", x + " ")) for op in OPS}
    demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    print(f"\n{demangled}\n  {usage.get(name, '')}\n  " + "  ".join(f"{k}={v}" for k, v in cnt.items()))
    if excerpt is None and "k_sem_k1_greg<7, 2" in demangled:
        excerpt = [x.strip() for x in ins if re.search(r"UBLKCP|SYNCS|CCTL|BAR.SYNC", x)][:12]
if excerpt:
    print("\n# k_sem_k1_greg<7, 2, 2, 8> (middle Chebyshev step): bulk-copy / mbarrier / prefetch / barrier lines")
    for x in excerpt:
        print("   ", x)
