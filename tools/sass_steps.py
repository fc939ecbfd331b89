"""Instruction histogram of one kernel in an object file, split at mbarrier waits / cp.async waits
(one segment per row-step form).  usage: sass_steps.py obj.o 'name-substring'"""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)[1:]
for f in funcs:
    name = subprocess.run(["c++filt", f.split("\n")[0].strip()], capture_output=True, text=True).stdout.strip()
    if pat not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s*([^;]*;)", l)
        if m:
            ins.append((int(m.group(1), 16), re.sub(r"\s+", " ", m.group(2))))
    print(name, "total", len(ins))
    seg, segs = [], []
    for a, t in ins:
        if "TRYWAIT" in t or "DEPBAR.LE" in t:
            segs.append(seg)
            seg = []
        seg.append(t)
    segs.append(seg)
    for i, sg in enumerate(segs):
        c = collections.Counter(re.sub(r"^@!?U?P\d+ ", "", t).split()[0].split(".")[0] for t in sg)
        fp = c["DADD"] + c["DMUL"] + c["DFMA"]
        print(f"  seg {i}: {len(sg)} instr, fp64 {fp}:", dict(c.most_common(14)))
    break
