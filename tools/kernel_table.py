"""Per-kernel table from an ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv log: launches, total time,
DRAM bytes and achieved DRAM GB/s (cold-cache ncu replay) vs the measured peak."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
iid, ik, im, iu, iv = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
unit = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}
per = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    per[(r[iid], r[ik])][r[im]] = float(r[iv].replace(",", "")) * unit.get(r[iu], 1.0)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    a = agg[name.split("(")[0]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
root = Path(__file__).resolve().parent.parent
peak = json.loads((root / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (root / "MEASURED_PEAKS.json").exists() else 6650.0
lines = [f"# {sys.argv[2] if len(sys.argv) > 2 else ''}", f"# peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs)",
         "kernel,launches,total_us,mean_us,dram_MB_per_launch,achieved_GBps,frac_of_peak"]
for name, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = b / t / 1e9 if t else 0.0
    lines.append(f"\"{name[:90]}\",{n},{t * 1e6:.1f},{t * 1e6 / n:.2f},{b / n / 1e6:.3f},{gbs:.1f},{gbs / peak:.3f}")
print("\n".join(lines))
