"""Summarise scripts/sector_profile.sh's ncu CSV into profiles/<tag>_sector_efficiency.csv.
Usage: python scripts/sector_summary.py gpurun_out/sectors.csv <tag> [config]"""
import collections, csv, re, sys
src, tag = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "C2"
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    full = r[ki]
    base = re.sub(r"<.*", "", re.sub(r"\(.*", "", full).replace("void ", "")).split("::")[-1]
    if "EmitLoader" in full:
        base += "(emit)"
    if base == "k_onesweep" and re.search(r"\b10\b\s*>|, \(int\)10>|,10>", full):
        base += "_w10"
    agg[base][r[mi]].append((float(r[vi].replace(",", "")), r[ui]))
out = [f"# {tag}: ncu --metrics (sector efficiency of global loads/stores, L2 hit, DRAM bytes), {cfg} bench --steps 1, per-launch means",
       "kernel,launches,duration_us,dram_MB_per_launch,l2_hit_pct,ld_bytes_per_sector_pct,st_bytes_per_sector_pct"]
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
for k, m in agg.items():
    def mean(name):
        v = m.get(name, [])
        return sum(x for x, _ in v) / len(v) if v else float("nan")
    dur = mean("gpu__time_duration.sum")
    if m["gpu__time_duration.sum"][0][1] in ("ns", "nsecond"):
        dur /= 1000.0
    sc = scale.get(m["dram__bytes_read.sum"][0][1], 1.0)
    out.append(f"{k},{len(m['gpu__time_duration.sum'])},{dur:.1f},{(mean('dram__bytes_read.sum') + mean('dram__bytes_write.sum')) * sc:.1f},"
               f"{mean('lts__t_sector_hit_rate.pct'):.1f},{mean('smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct'):.1f},"
               f"{mean('smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct'):.1f}")
open(f"profiles/{tag}_sector_efficiency.csv", "w").write("\n".join(out) + "\n")
print("\n".join(out))
