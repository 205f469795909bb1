"""Summarise an ncu --set full capture (raw CSV page) into profiles/:
per kernel duration, DRAM bytes, registers, grid; and ncu_traffic.json
(per-launch DRAM read+write bytes by kernel role) that bench.py reports as
roofline.traffic.  Usage: python scripts/ncu_summary.py gpurun_out/prof_X_raw.csv TAG"""
import csv
import json
import os
import statistics
import sys

src, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
roles = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    role = ("fused_p1" if "fused_p1" in name else "absmax_exp" if "absmax" in name or "AbsmaxOp" in name
            else "quant_pack" if "quant" in name or "QuantOp" in name else "unpack_unscale"
            if "unpack" in name or "UnpackOp" in name else name[:40])
    g = lambda m: float(r[col[m]]) if m in col and r[col[m]] not in ("", "n/a") else None
    roles.setdefault(role, []).append({
        "kernel": name, "duration_us": g("gpu__time_duration.sum"),
        "dram_read_MB": g("dram__bytes_read.sum"), "dram_write_MB": g("dram__bytes_write.sum"),
        "registers": g("launch__registers_per_thread"), "grid": g("launch__grid_size"),
        "block": g("launch__block_size"), "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "sm_active_cycles": g("sm__cycles_active.avg"), "elapsed_cycles": g("sm__cycles_elapsed.avg"),
        "l2_hit_pct": g("lts__t_sector_hit_rate.pct")})
summary, traffic = {}, {}
for role, lst in roles.items():
    med = lambda k: statistics.median([x[k] for x in lst if x[k] is not None]) if any(x[k] is not None for x in lst) else None
    summary[role] = {"launches": len(lst), "kernel": lst[0]["kernel"], **{k: med(k) for k in lst[0] if k != "kernel"}}
    if summary[role]["dram_read_MB"] is not None:
        traffic[role] = int((summary[role]["dram_read_MB"] + summary[role]["dram_write_MB"]) * 1e6)
os.makedirs("profiles", exist_ok=True)
json.dump(summary, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(summary, indent=1))
