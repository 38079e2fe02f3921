"""Instruction mix of the softmax KV loop of svd_fwd_kernel<D, false> in a
built library (cuobjdump -sass): the loop is the backward branch whose body
holds the MUFU.EX2 exps.  Usage: sass_loop.py LIB.so [D]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1]
D = sys.argv[2] if len(sys.argv) > 2 else "128"
fn = f"_ZN3svd14svd_fwd_kernelILi{D}ELb0EEEv14CUtensorMap_stS1_S1_NS_9FwdParamsE"
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for l in out.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
mufu = [a for a, t in ins if "MUFU.EX2" in t]
best = None
for a, t in ins:
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and any(tgt <= x <= a for x in mufu):
            if best is None or (a - tgt) > (best[1] - best[0]):
                best = (tgt, a)
lo, hi = best
body = [(a, t) for a, t in ins if lo <= a <= hi]
c = Counter()
for a, t in body:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    c[op.split(".")[0]] += 1
print(f"loop {hex(lo)}..{hex(hi)}: {len(body)} instructions (incl. mask / rescale branches)")
print("LDL/STL in loop:", c["LDL"] + c["STL"], " whole kernel LDL:", sum(1 for _, t in ins if "LDL" in t))
print(c.most_common(25))
