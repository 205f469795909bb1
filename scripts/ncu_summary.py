"""Summarise an ncu --set full capture (raw CSV page) into profiles/:
per kernel duration, DRAM bytes, registers, grid; and ncu_traffic.json
(per-launch DRAM read+write bytes by kernel role) that bench.py reports as
roofline.traffic.

ncu scales every metric's unit separately (byte / Kbyte / Mbyte / Gbyte,
nsecond / usecond / msecond) and states it in the CSV's second row: every
value is converted here from that row to bytes and microseconds (capture with
`--print-units base` to get base units directly).  A summary whose DRAM rate
exceeds the measured HBM peak is flagged instead of written silently.

Usage: python scripts/ncu_summary.py gpurun_out/prof_X_raw.csv TAG [--no-traffic]"""
import csv
import json
import os
import statistics
import sys

BYTES = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
         "kibyte": 1024, "mibyte": 1 << 20, "gibyte": 1 << 30}
SECS_US = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
           "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def convert(val, unit):
    u = (unit or "").strip().lower()
    if u in BYTES:
        return val * BYTES[u]
    if u in SECS_US:
        return val * SECS_US[u]
    return val


def role_of(name):
    return ("fused_p1" if "fused" in name else "absmax_exp" if "absmax" in name
            else "quant_pack" if "quant" in name else "unpack_unscale" if "unpack" in name
            else "peer_reduce" if "peer_reduce" in name else name[:40])


def main():
    src, tag = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    roles = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[col["Kernel Name"]]

        def g(m):
            if m not in col or r[col[m]] in ("", "n/a"):
                return None
            return convert(float(r[col[m]].replace(",", "")), units[col[m]])
        roles.setdefault(role_of(name), []).append({
            "kernel": name, "duration_us": g("gpu__time_duration.sum"),
            "dram_read_bytes": g("dram__bytes_read.sum"), "dram_write_bytes": g("dram__bytes_write.sum"),
            "registers": g("launch__registers_per_thread"), "grid": g("launch__grid_size"),
            "block": g("launch__block_size"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "sm_active_cycles": g("sm__cycles_active.avg"), "elapsed_cycles": g("sm__cycles_elapsed.avg"),
            "l2_hit_pct": g("lts__t_sector_hit_rate.pct"),
            "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")})
    try:
        peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    summary, traffic = {}, {}
    for role, lst in roles.items():
        def med(k):
            v = [x[k] for x in lst if x[k] is not None]
            return statistics.median(v) if v else None
        s = {"launches": len(lst), "kernel": lst[0]["kernel"], **{k: med(k) for k in lst[0] if k != "kernel"}}
        if s["dram_read_bytes"] is not None and s["duration_us"]:
            tot = s["dram_read_bytes"] + (s["dram_write_bytes"] or 0)
            s["dram_GBps"] = round(tot / (s["duration_us"] * 1e-6) / 1e9, 1)
            s["dram_frac_of_peak"] = round(s["dram_GBps"] / peak, 4)
            if s["dram_GBps"] > peak * 1.02:
                s["flag"] = f"DRAM rate {s['dram_GBps']} GB/s above the {peak} GB/s peak: check the units"
            traffic[role] = int(tot)
        summary[role] = s
    os.makedirs("profiles", exist_ok=True)
    json.dump({"units": "bytes, microseconds (converted from the CSV units row)", "hbm_peak_GBps": peak,
               "kernels": summary}, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
    if "--no-traffic" not in sys.argv:
        json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
