"""Summarise ncu evidence into text files under profiles/ (dev tool, runs here without a GPU).

  python tools/summarize_ncu.py full <report.ncu-rep> <out.txt> [label]      # one `--set full` capture
  python tools/summarize_ncu.py launches <launches.csv> <out.txt> [label]    # `--metrics gpu__time_duration.sum` list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, out, label=""):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {label or rep}", ""]
    for r in rows[2:]:
        lines.append(f"kernel: {r[h.index('Kernel Name')][:160]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"  {k:60s} {r[i]:>20s} {units[i]}")
        try:
            rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
            ur, uw = units[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_write.sum")]
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            t = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
            tu = units[h.index("gpu__time_duration.sum")]
            ts = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}[tu]
            tot = rd * sc[ur] + wr * sc[uw]
            lines.append(f"  traffic (dram read+write) per launch: {tot:.6e} bytes; achieved DRAM {tot / (t * ts) / 1e9:.1f} GB/s")
        except Exception as e:  # pragma: no cover
            lines.append(f"  (traffic: {e})")
        lines.append("")
    # warp stall breakdown from the details page
    det = ncu_csv(["-i", rep, "--page", "details"])
    dh = det[0]
    for r in det[1:]:
        d = dict(zip(dh, r))
        if d.get("Section Name") in ("Warp State Statistics", "Occupancy", "Memory Workload Analysis",
                                     "GPU Speed Of Light Throughput", "Scheduler Statistics"):
            lines.append(f"  [{d['Section Name'][:24]}] {d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out, label=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    I, K, MV, MU = h.index("ID"), h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        t = float(r[MV].replace(",", ""))
        t *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[MU], 1.0)
        name = r[K].split("(")[0].replace("void ", "").replace("pjds::(anonymous namespace)::", "")
        per.setdefault(name, []).append(t)
    tot = sum(sum(v) for v in per.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none, serialised, cold-ish cache): {label}",
             f"# {sum(len(v) for v in per.values())} launches, {tot:.1f} us total", "",
             f"{'kernel':90s} {'launches':>8s} {'avg us':>10s} {'total us':>10s} {'share':>7s}"]
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{name[:90]:90s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v):10.1f} {sum(v) / tot:7.1%}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    label = sys.argv[4] if len(sys.argv) > 4 else ""
    (full if mode == "full" else launches)(src, dst, label)
