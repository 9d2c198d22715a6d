"""Summarise an `ncu --metrics ... --csv` launch list: one line per launch (dev tool)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
labels = sys.argv[2].split(",") if len(sys.argv) > 2 else []
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
I, K, MN, MV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    d.setdefault((r[I], r[K][:50]), {})[r[MN]] = r[MV].replace(",", "")
for (i, k), m in d.items():
    lab = labels[int(i)] if int(i) < len(labels) else k
    t = float(m["gpu__time_duration.sum"])
    rd = float(m.get("dram__bytes_read.sum", 0)); wr = float(m.get("dram__bytes_write.sum", 0))
    print(f"{lab:28s} t={t/1e3:8.1f}us rd={rd/1e6:9.1f}MB wr={wr/1e6:8.1f}MB dram={(rd+wr)/t:7.1f}GB/s "
          f"L2hit={m.get('lts__t_sector_hit_rate.pct','-'):>6s} L1hit={m.get('l1tex__t_sector_hit_rate.pct','-'):>6s} "
          f"occ={m.get('sm__warps_active.avg.pct_of_peak_sustained_active','-'):>6s}")
