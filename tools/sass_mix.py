"""Executed-instruction mix of one kernel in an ncu report, and the source
lines behind selected opcodes (divergent-branch bookkeeping BSSY/BSYNC/BRA,
rematerialisation IMAD/S2R, spills LDL/STL):
  python tools/sass_mix.py <rep> [kernel-substring] [OPC,OPC,...]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", sys.argv[2]]
ops = (sys.argv[3] if len(sys.argv) > 3 else "BSSY,BSYNC,BRA,IMAD,LDL,S2R").split(",")
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
cur_file = cur = None
by = collections.defaultdict(collections.Counter)
tot = collections.Counter()
lines = collections.Counter()
samp = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No", "Kernel Name"):
        continue
    if r[0] != "":
        cur = (cur_file, r[0], r[1][:80])
        continue
    try:
        e, sm = int(r[7] or 0), int(r[4] or 0)
    except (ValueError, IndexError):
        continue
    op = r[3].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1] if " " in op else op
    op = op.split()[0].split(".")[0] if op else "?"
    by[op][cur] += e
    tot[op] += e
    lines[cur] += e
    samp[cur] += sm
T = sum(tot.values()) or 1
S = sum(samp.values()) or 1
print("executed warp instructions", T)
for op, e in tot.most_common(16):
    print(f"  {op:10s} {100 * e / T:5.1f}%")
for op in ops:
    print("==", op, f"{100 * tot[op] / T:.1f}%")
    for k, v in by[op].most_common(5):
        print(f"   {100 * v / T:5.2f}% {k[0]}:{k[1]} {k[2]}")
print("== top lines (executed / stall samples)")
for k, v in lines.most_common(12):
    print(f"   {100 * v / T:5.2f}% {100 * samp[k] / S:5.2f}% {k[0]}:{k[1]} {k[2]}")
