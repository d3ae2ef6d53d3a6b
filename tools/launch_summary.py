"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv` launch list into
markdown: every bos:: launch with time and DRAM bytes, plus the other kernels' total.
    python tools/launch_summary.py gpurun_out/launches.csv "title" "command" > profiles/x.md"""
import collections
import csv
import sys

SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
SCALE_B = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    m = r[ix["Metric Name"]]
    val = v * (SCALE_T.get(u, 1.0) if "time" in m else SCALE_B.get(u, 1.0))
    k.setdefault((r[ix["ID"]], r[ix["Kernel Name"]]), {})[m] = val
print(f"# {sys.argv[2] if len(sys.argv) > 2 else 'launch list'}\n")
if len(sys.argv) > 3:
    print(f"Command: `{sys.argv[3]}`. Cold-cache, serialised times (ncu --clock-control none): compare shares.\n")
print("| ID | kernel | time (ms) | DRAM read (MB) | DRAM write (MB) |\n|---|---|---|---|---|")
tot = dem = 0.0
n_other = 0
for (i, n), m in k.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    tot += t
    if "bos::" in n or "demod" in n or "unwrap" in n or "lobe_mask" in n:
        dem += t
        print(f"| {i} | {n.split('(')[0]} | {t:.3f} | {m.get('dram__bytes_read.sum', float('nan')):.1f} | "
              f"{m.get('dram__bytes_write.sum', float('nan')):.1f} |")
    else:
        n_other += 1
print(f"\nbos:: kernels {dem:.2f} ms; other kernels (generator / torch copies, outside the timed region): "
      f"{n_other} launches, {tot - dem:.2f} ms.")
