"""Attribute an ncu capture's per-instruction stall samples and executed instructions to source
lines, by joining ncu's SASS page with `nvdisasm -g` of the same build (the CLI's CUDA source
view carries no metrics).  python scripts/ncu_lines.py <rep.ncu-rep> <object.o> <kernel substring> [top]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True, text=True).stdout.splitlines()
# the capture, or its source page already exported as CSV (captures too large to bring back)
out = open(rep).read() if rep.endswith(".csv") else subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"],
                                                                      capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h, data = rows[hi], [r for r in rows[hi + 1:] if len(r) > 5]


def parse(start):
    insts, cur = {}, None
    for l in dis[start + 1:]:
        if l.startswith(".section") or (l.startswith("_Z") and l.endswith(":")):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            insts[int(m.group(1), 16)] = cur
    return insts


# several instantiations can match the name: take the one whose length equals the profiled SASS
cands = [parse(i) for i, l in enumerate(dis) if l.startswith("_Z") and kname in l and l.endswith(":")]
insts = min(cands, key=lambda c: abs(len(c) - len(data)))
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(data[0][0], 16)
by = collections.defaultdict(lambda: [0, 0])
for r in data:
    ln = insts.get(int(r[0], 16) - base)
    by[ln][0] += int(r[si] or 0)
    by[ln][1] += int(r[ie] or 0)
ts, te = sum(v[0] for v in by.values()) or 1, sum(v[1] for v in by.values()) or 1
print(f"{len(data)} SASS instructions, {ts} stall samples, {te} warp instructions executed")
srcs = {}
for (ln, (st, ex)) in sorted(by.items(), key=lambda kv: -kv[1][0])[:top]:
    txt = ""
    if ln:
        path = next((p for p in ("paper_1707_03750_b200/csrc/" + ln[0],) if os.path.exists(p)), None)
        if path:
            srcs.setdefault(path, open(path).read().splitlines())
            txt = srcs[path][ln[1] - 1].strip()[:90]
    print(f"{100 * st / ts:5.1f}% stalls {100 * ex / te:5.1f}% instr  {ln}  {txt}")
