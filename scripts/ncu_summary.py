"""Summarise ncu --page raw --csv exports (units row honoured) into a
markdown table and profiles/traffic.json (dram bytes per launch).
usage: python scripts/ncu_summary.py gpurun_out/m/full_*.csv"""
import csv, json, os, sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3, "%": 1}
KEYS = {"full_c2_backward": "c2_unfused_backward", "full_c3_forward": "c3_unfused_forward",
        "full_c3f_forward": "c3_fused_forward", "full_c4_grads": "c4_unfused_grads",
        "full_c3_costs": "c3_unfused_costs", "full_c3f_backward": "c3_fused_backward",
        "full_c3f_grads": "c3_fused_grads"}
rows_out, traffic = [], {}
tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
if os.path.exists(tpath):
    traffic = json.load(open(tpath))
for path in sys.argv[1:]:
    r = list(csv.reader(open(path)))
    h, u, v = r[0], r[1], r[2]
    d = {}
    for name, unit, val in zip(h, u, v):
        if "__" in name:
            d[name] = float(val) * SCALE.get(unit, 1)
        else:
            d[name] = val
    rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
    tag = os.path.basename(path)[:-4]
    if tag in KEYS:
        traffic[KEYS[tag]] = rd + wr
    rows_out.append((tag, d["Kernel Name"].split("(")[0].replace("void ", ""), d["Grid Size"], d["Block Size"],
                     d["gpu__time_duration.sum"], rd / 1e6, wr / 1e6,
                     d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                     d["sm__warps_active.avg.pct_of_peak_sustained_active"],
                     d["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"],
                     d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]))
print("| capture | kernel | grid x block | duration us | DRAM read MB | DRAM write MB | issue active | warps active | XU (MUFU) pipe | FMA pipe |")
print("|---|---|---|---|---|---|---|---|---|---|")
for t in rows_out:
    print(f"| {t[0]} | `{t[1]}` | {t[2]} x {t[3]} | {t[4]:.1f} | {t[5]:.1f} | {t[6]:.1f} | {t[7]:.1f} % | {t[8]:.1f} % | {t[9]:.1f} % | {t[10]:.1f} % |")
json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
