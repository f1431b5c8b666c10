"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/<round>_launches.md
  python tools/summarize_ncu.py report gpurun_out/x.ncu-rep <kernel-name> [<kernel-name> ...]
        -> merges per-kernel metrics into profiles/ncu_summary.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    ik, iname, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[iname] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "").strip()
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    all_ns = sum(tot.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in tot.most_common():
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / all_ns:.1f}% |")
    out.append(f"\nTotal {sum(cnt.values())} launches, {all_ns / 1e6:.3f} ms (ncu-serialised, cold caches: "
               "compare shares, not absolutes).")
    print("\n".join(out))


WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed.sum": "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__average_warp_latency_per_inst_issued.ratio": "warp_cycles_per_issue",
    "sm__cycles_elapsed.avg": "sm_cycles",
}


def report(path, names):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
             "s": 1e9, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}

    def val(r, m):
        i = h.index(m)
        x = float(r[i].replace(",", ""))
        return x * scale.get(units[i], 1.0)

    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    pairs = [n.split("=", 1) if "=" in n else (n, n) for n in names]
    for r in rows[2:]:
        kname = r[h.index("Kernel Name")]
        for pat, n in pairs:
            if pat in kname:
                d = {"report": os.path.basename(path), "kernel": kname[:160]}
                for m, key in WANT.items():
                    if m in h:
                        try:
                            d[key] = val(r, m)
                        except ValueError:
                            d[key] = r[h.index(m)]
                stalls = {}
                for i, m in enumerate(h):
                    if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued"):
                        try:
                            stalls[m.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                        except ValueError:
                            pass
                tot = sum(stalls.values()) or 1.0
                d["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
                if "dram_read_bytes" in d and "dram_write_bytes" in d:
                    d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
                summ[n] = d
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(json.dumps({n: summ.get(n) for _, n in pairs}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3:])
