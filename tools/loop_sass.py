"""Static SASS look at phase 1's hot loops (no GPU needed): for the band
PAIRS kernel, find the basic blocks that end in a backward branch and print
their instruction mix.  Usage: python tools/loop_sass.py [kernel-regex]"""
import re
import subprocess
import sys
from collections import Counter

import os
obj = os.environ.get("OBJ", "paper_2507_22901_b200/_build/cvg_kernels.o")
pat = sys.argv[1] if len(sys.argv) > 1 else r"phase1_kernelILi0ELi0ELi0E"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
f = [x for x in funcs if re.match(r"\S*" + pat, x)][0]
lines = []
for ln in f.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        lines.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(lines)}
for i, (a, ins) in enumerate(lines):
    m = re.search(r"BRA\s+(?:\S+,\s*)?`?\(?\.?L_x_\d+\)?|BRA\s+0x([0-9a-f]+)", ins)
    t = re.search(r"0x([0-9a-f]+)", ins) if "BRA" in ins else None
    if t:
        tgt = int(t.group(1), 16)
        if tgt < a and tgt in addr_idx:
            body = lines[addr_idx[tgt]:i + 1]
            if 20 <= len(body) <= 400:
                ops = Counter(x.split()[0].lstrip("@!P0123456789T ").split(".")[0] if not x.startswith("@") else x.split()[1].split(".")[0] for _, x in body)
                print(f"loop {tgt:#x}-{a:#x}: {len(body)} instrs  {dict(ops.most_common(12))}")

# Fast path of each hot loop: loop top .. the branch that skips the settle
# (the first "@!P BRA" after a VOTE.ANY), plus that branch's target .. the
# backward branch.
print("fast paths (no candidate needs attention):")
for i, (a, ins) in enumerate(lines):
    t = re.search(r"0x([0-9a-f]+)", ins) if "BRA" in ins else None
    if not t or int(t.group(1), 16) >= a or int(t.group(1), 16) not in addr_idx:
        continue
    top = addr_idx[int(t.group(1), 16)]
    body = lines[top:i + 1]
    if not (20 <= len(body) <= 3000):
        continue
    vote = next((j for j in range(top, i) if lines[j][1].startswith("VOTE.ANY")), None)
    if vote is None:
        continue
    skip = next((j for j in range(vote, i) if re.match(r"@!?P\d BRA", lines[j][1])), None)
    if skip is None:
        continue
    tgt = int(re.search(r"0x([0-9a-f]+)", lines[skip][1]).group(1), 16)
    if tgt not in addr_idx or tgt > a:
        continue
    path = lines[top:skip + 1] + lines[addr_idx[tgt]:i + 1]
    ops = Counter(x.split()[1].split(".")[0] if x.startswith("@") else x.split()[0].split(".")[0] for _, x in path)
    print(f"  loop {lines[top][0]:#x}: {len(path)} instrs  {dict(ops.most_common(14))}")
