"""Summarise an .ncu-rep with many kernels (read here, no GPU): one line per kernel name -- launches, time, DRAM
traffic and throughput, issue activity, L2 hit rate, L2 atomic / reduction sectors."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
def f(r, name):
    try: return float(r[col[name]].replace(",", ""))
    except Exception: return float("nan")
agg = collections.OrderedDict()
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].split("<")[0]
    a = agg.setdefault(name, dict(n=0, us=0.0, rd=0.0, wr=0.0, dram=0.0, issue=0.0, l2=0.0, red=0.0, atom=0.0, inst=0.0, regs=0))
    a["n"] += 1
    tunit = rows[1][col["gpu__time_duration.sum"]]
    a["us"] += f(r, "gpu__time_duration.sum") * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(tunit, 1.0)
    for key, metric in (("rd", "dram__bytes_read.sum"), ("wr", "dram__bytes_write.sum")):
        unit = rows[1][col[metric]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        a[key] += f(r, metric) * scale
    a["dram"] += f(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    a["issue"] += f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    a["l2"] += f(r, "lts__t_sector_hit_rate.pct")
    a["red"] += f(r, "lts__t_sectors_op_red.sum") if "lts__t_sectors_op_red.sum" in col else 0.0
    a["atom"] += f(r, "lts__t_sectors_op_atom.sum") if "lts__t_sectors_op_atom.sum" in col else 0.0
    a["inst"] += f(r, "smsp__inst_executed.sum")
    a["regs"] = int(f(r, "launch__registers_per_thread"))
print(f"{'kernel':34s} {'n':>3s} {'us/launch':>10s} {'DRAM MB':>9s} {'GB/s':>7s} {'dram%':>6s} {'issue%':>6s} {'L2hit%':>6s} {'L2 red sect':>11s} {'L2 atom sect':>12s} {'Minst':>8s} {'regs':>4s}")
for name, a in agg.items():
    n = a["n"]
    mb = (a["rd"] + a["wr"]) / n / 1e6
    us = a["us"] / n
    print(f"{name[:34]:34s} {n:3d} {us:10.1f} {mb:9.1f} {mb / us * 1e3 if us else 0:7.0f} {a['dram']/n:6.1f} {a['issue']/n:6.1f} {a['l2']/n:6.1f} {a['red']/n:11.0f} {a['atom']/n:12.0f} {a['inst']/n/1e6:8.2f} {a['regs']:4d}")
