"""Summarise an ncu --set full capture of hx::loop_kernel (100 iterations per
launch, tools/profile_loop.py) into profiles/: traffic JSON (per iteration and
per 1000-iteration bench launch) and the stall share per hx.cu source line.

  python tools/ncu_summary.py gpurun_out/loop_full3.ncu-rep "label" [stalls.csv]
"""
import csv
import json
import subprocess
import sys

rep, label = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "lts__t_requests.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__cycles_elapsed.avg.per_second"]
d = {w: {"unit": u[h.index(w)], "value": v[h.index(w)]} for w in want if w in h}
its = 100
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rd = float(d["dram__bytes_read.sum"]["value"]) * scale[d["dram__bytes_read.sum"]["unit"]] / its
wr = float(d["dram__bytes_write.sum"]["value"]) * scale[d["dram__bytes_write.sum"]["unit"]] / its
out = {"source": f"ncu --set full --clock-control none --import-source on, 1 launch of hx::loop_kernel_stream = {its} rHPDHG "
                 f"iterations on configs[1] (tools/profile_loop.py --iters 100 --launches 2; -k regex:loop_kernel -s 2 "
                 f"-c 1); {label}",
       "dram_bytes_read_per_iter": rd, "dram_bytes_write_per_iter": wr, "dram_bytes_per_iter": rd + wr,
       "iters_per_bench_launch": 1000, "dram_bytes_per_launch": (rd + wr) * 1000,
       "algorithmic_bytes_per_iter": 97640008,
       "l2_requests_per_iter": float(d["lts__t_requests.sum"]["value"]) / its,
       "l2_sectors_per_iter": float(d["lts__t_sectors.sum"]["value"]) / its, "ncu": d}
json.dump(out, open("profiles/loop_kernel_traffic.json", "w"), indent=1)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hh = rows[hi]
iS = hh.index("Warp Stall Sampling (All Samples)")
agg, text, cur = {}, {}, None
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0] != "":
        cur = r[0]
        text[cur] = r[1] if len(r) > 1 else ""
    try:
        s = int(r[iS] or 0)
    except (ValueError, IndexError):
        continue
    if len(r) > 2 and r[2]:
        agg[cur] = agg.get(cur, 0) + s
T = sum(agg.values())
with open(sys.argv[3] if len(sys.argv) > 3 else "profiles/loop_stalls_by_line.csv", "w") as f:
    f.write(f"# {label}\nshare_pct,hx.cu_line,source\n")
    for line, s in sorted(agg.items(), key=lambda x: -x[1])[:30]:
        f.write(f"{s / T * 100:.2f},{line},\"{text.get(line, '').strip()[:120].replace(chr(34), chr(39))}\"\n")
print(json.dumps({k: d[k]["value"] for k in d}, indent=0)[:1500])
print("dram/iter", rd + wr)
