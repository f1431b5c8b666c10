"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo
and --import-source):  python tools/ncu_lines.py <rep> [top] [kernel-substring]
Aggregates warp-stall samples and L2 global sectors by CUDA source line."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"] +
                     (["-k", sys.argv[3]] if len(sys.argv) > 3 else []),
                     capture_output=True, text=True).stdout
samples = collections.Counter()
sectors = collections.Counter()
insts = collections.Counter()
text = {}
path = None
hdr = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    key = (path, r[0])
    text[key] = r[1].strip()[:90]

    def num(name):
        try:
            return float(r[hdr.index(name)])
        except (ValueError, IndexError):
            return 0.0
    samples[key] += num("Warp Stall Sampling (All Samples)")
    sectors[key] += num("L2 Theoretical Sectors Global")
    insts[key] += num("Instructions Executed")
tot_s = sum(samples.values()) or 1
tot_l2 = sum(sectors.values()) or 1
print(f"total samples {tot_s:.0f}, L2 global sectors {tot_l2:.3g}, warp insts {sum(insts.values()):.3g}")
print("== by stall samples")
for k, v in samples.most_common(top):
    print(f"{100 * v / tot_s:5.1f}%  L2 {100 * sectors[k] / tot_l2:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
print("== by L2 sectors")
for k, v in sectors.most_common(top // 2):
    print(f"L2 {100 * v / tot_l2:5.1f}%  stall {100 * samples[k] / tot_s:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
tot_i = sum(insts.values()) or 1
print("== by executed warp instructions")
for k, v in insts.most_common(top):
    print(f"inst {100 * v / tot_i:5.1f}%  stall {100 * samples[k] / tot_s:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
