"""Turn a round's ncu launch list + full capture into the committed summaries under profiles/.
Usage: python scripts/profile_summary.py <launches.csv> <prof.ncu-rep> <tag> [workload, default C3]"""
import collections, csv, io, json, re, subprocess, sys
launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else "C3"
rows = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    name = re.sub(r"<.*", "", name).split("::")[-1]
    v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1e-3)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
out = [f"# {tag}: ncu launch list of `python bench.py --config {workload} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e` (first 400 launches), gpu__time_duration.sum,",
       "# --clock-control none; cold-cache and serialised per launch: compare SHARES, not absolutes",
       "kernel,launches,total_us,share"]
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k},{c},{t:.1f},{t / tot:.4f}")
open(f"profiles/{tag}_launches_summary.csv", "w").write("\n".join(out) + "\n")
print("\n".join(out[:16]))
# the capture itself, or its raw page already exported as CSV (the report stays on the GPU box)
# several captures may be given comma-separated (raw pages are merged by column name)
def _rows(one):
    raw = open(one).read() if one.endswith(".csv") else subprocess.run(["ncu", "-i", one, "--page", "raw", "--csv"],
                                                                       capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(raw)))
parts = [_rows(x) for x in rep.split(",")]
hdr, units = parts[0][0], parts[0][1]
rr = [hdr, units] + parts[0][2:]
_S = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6, "nsecond": 1e-3, "usecond": 1.0,
      "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
for extra in parts[1:]:
    eh, eu = extra[0], extra[1]
    for r in extra[2:]:
        d = dict(zip(eh, r))
        du = dict(zip(eh, eu))
        row = []
        for k, u0 in zip(hdr, units):
            v = d.get(k, "")
            if v and du.get(k) in _S and u0 in _S and du[k] != u0:  # into the first capture's unit
                try:
                    v = repr(float(v.replace(",", "")) * _S[du[k]] / _S[u0])
                except ValueError:
                    pass
            row.append(v)
        rr.append(row)
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6,  # bytes -> MB
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,  # durations -> us
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
def g(r, k):
    if k not in hdr or r[hdr.index(k)] in ("", "n/a"):
        return None
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
keys = {"duration_us": "gpu__time_duration.sum", "dram_read_MB": "dram__bytes_read.sum", "dram_write_MB": "dram__bytes_write.sum",
        "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active", "registers": "launch__registers_per_thread",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct", "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        # sector efficiency of global loads / stores (bytes used per 32-B sector moved, %): the
        # random-access gathers' figure of merit
        "ld_bytes_per_sector_pct": "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "st_bytes_per_sector_pct": "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct"}
names = {"k_onesweep": "radix_onesweep", "k_rank_update": "sa_rank_update", "k_hash_insert": "intern_hash", "k_plcp": "lcp_plcp", "k_compact_local": "compact",
         "k_ansv": "ansv_intervals", "k_scan": "compact", "k_refine_detect": "sa_refine_detect", "k_refine_apply": "sa_refine_apply",
         "k_phi": "lcp_phi", "k_lcp_gather": "lcp_gather"}
per = collections.defaultdict(list)
for r in rr[2:]:
    full = r[hdr.index("Kernel Name")]
    base = re.sub(r"<.*", "", re.sub(r"\(.*", "", full).replace("void ", "")).split("::")[-1]
    nm = names.get(base, base)
    if "EmitLoader" in full:
        nm = "radix_onesweep(emit)"
    d = {k: g(r, m) for k, m in keys.items()}
    st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), g(r, k))
                 for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                key=lambda x: -(x[1] or 0))[:4]
    d["top_stalls"] = {a: b for a, b in st}
    per[nm].append(d)
summ = {"source": f"{tag}: ncu --set full --clock-control none --import-source on, bench.py --config {workload}", "workload": workload,
        "kernels": {}}
for nm, lst in per.items():
    avg = {k: sum(x[k] for x in lst) / len(lst) for k in keys if all(x[k] is not None for x in lst)}
    avg.setdefault("dram_read_MB", 0.0)
    avg.setdefault("dram_write_MB", 0.0)
    avg["dram_bytes_per_launch"] = (avg["dram_read_MB"] + avg["dram_write_MB"]) * 1e6
    avg["launches_profiled"] = len(lst)
    avg["top_stalls"] = lst[0]["top_stalls"]
    summ["kernels"][nm] = avg
json.dump(summ, open("profiles/ncu_summary.json", "w"), indent=1)
for k, v in summ["kernels"].items():
    print(f"{k:24s} {v.get('duration_us', 0):7.1f}us dram {v['dram_bytes_per_launch']/1e6:6.1f}MB warps {v.get('warps_active_pct', 0):3.0f}% "
          f"ld-sector {v.get('ld_bytes_per_sector_pct', float('nan')):5.1f}% st-sector {v.get('st_bytes_per_sector_pct', float('nan')):5.1f}% L2hit {v.get('l2_hit_pct', 0):3.0f}%")
