"""Digest an ncu report: per kernel duration, DRAM traffic, occupancy, top stall reasons and
the hottest SASS lines.  Usage: python scripts/ncu_digest.py report.ncu-rep [regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
def g(r, k):
    return float(r[hdr.index(k)]) if k in hdr and r[hdr.index(k)] not in ("", "n/a") else float("nan")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = re.sub(r"\(.*", "", name).split("::")[-1][:60]
    if pat and not pat.search(name):
        continue
    st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), g(r, k))
                 for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                key=lambda x: -x[1])[:4]
    print(f"{short:60s} {g(r,'gpu__time_duration.sum'):8.1f}us DRAM {g(r,'dram__bytes_read.sum'):.1f}+{g(r,'dram__bytes_write.sum'):.1f}MB "
          f"dram% {g(r,'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.0f} warps% {g(r,'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} "
          f"regs {g(r,'launch__registers_per_thread'):.0f} L2hit {g(r,'lts__t_sector_hit_rate.pct'):.0f} | " + ", ".join(f"{a}={b:.1f}" for a, b in st))

if len(sys.argv) > 3:  # hottest SASS lines of the first kernel matching argv[3]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + sys.argv[3],
                          "-c", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    h = rows[hi]
    si = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    data = [r for r in rows[hi + 1:] if len(r) > si and r[si].replace(".", "").isdigit()]
    tot = sum(float(r[si]) for r in data) or 1
    for r in sorted(data, key=lambda r: -float(r[si]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 20]:
        rs = sorted(((c[6:], float(r[h.index(c)] or 0)) for c in reasons), key=lambda x: -x[1])[:2]
        print("%5.1f%%  %-60s %s" % (100 * float(r[si]) / tot, r[h.index("Source")].strip()[:60], rs))
