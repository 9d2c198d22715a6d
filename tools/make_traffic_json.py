"""Build profiles/r02_traffic.json from the ncu CSV of tools/traffic_capture.py (dev tool, no GPU):
kernel launches in capture order map onto traffic_capture.ORDER; traffic = dram read + write."""
import csv, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from traffic_capture import ORDER

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == "ID")
vals = {}
names = {}
for r in rows:
    if r is hdr or len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    i = int(d["ID"])
    vals.setdefault(i, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    names[i] = d["Kernel Name"]
ids = sorted(vals)
assert len(ids) == len(ORDER), (len(ids), len(ORDER))
out = {"_doc": "DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of one launch per kernel, "
               "ncu --clock-control none with ncu's default cache control (caches flushed before the launch: the "
               "L2-cold state bench.py's per_config timing reproduces by rotating x/y); tools/traffic_capture.py, "
               f"from {os.path.basename(sys.argv[1])}"}
for i, (cfg, dt, fmt) in zip(ids, ORDER):
    v = vals[i]
    out[f"{cfg}/{dt}/{fmt}"] = {"traffic": int(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]),
                                "read": int(v["dram__bytes_read.sum"]), "write": int(v["dram__bytes_write.sum"]),
                                "ncu_us": round(v["gpu__time_duration.sum"] / 1e3, 2), "kernel": names[i][:120]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1)[:2000])
