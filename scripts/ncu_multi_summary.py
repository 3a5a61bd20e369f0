"""Summarise every kernel launch of an ncu --set full report into one JSON list
(HBM GB/s against the measured peak, issue activity, occupancy).
usage: ncu_multi_summary.py REPORT OUT.json [NOTE]"""
import csv, io, json, os, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
peak = None
pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(pk):
    try:
        peak = float(json.load(open(pk)).get("hbm_gbs"))
    except Exception:
        peak = None
MUL = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "usecond": 1e3,
       "ms": 1e6, "msecond": 1e6, "nsecond": 1}
res = []
for v in rows[2:]:
    m = dict(zip(h, v))
    def num(k, scale=False):
        try:
            x = float(m.get(k, "").replace(",", ""))
        except ValueError:
            return None
        return x * MUL.get(dict(zip(h, units)).get(k, ""), 1) if scale else x
    t_ns = num("gpu__time_duration.sum", True) or 0
    dr, dw = num("dram__bytes_read.sum", True) or 0, num("dram__bytes_write.sum", True) or 0
    gbs = (dr + dw) / t_ns if t_ns else 0.0  # bytes per ns = GB/s
    res.append({
        "kernel": m.get("Kernel Name", "")[:90], "grid": m.get("launch__grid_size"), "block": m.get("launch__block_size"),
        "gpu_time_us": t_ns / 1e3, "dram_read_MB": dr / 1e6, "dram_write_MB": dw / 1e6, "dram_GBs": gbs,
        "hbm_peak_GBs": peak, "frac_of_hbm_peak": (gbs / peak) if peak else None,
        "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
        "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
    })
json.dump({"capture": note, "note": "per-launch times under ncu are cold-cache and serialised", "launches": res},
          open(out, "w"), indent=1)
for r in res:
    print(f"{r['kernel'][:50]:50s} {r['gpu_time_us']:9.1f} us  {r['dram_GBs']:8.1f} GB/s  "
          f"{'' if r['frac_of_hbm_peak'] is None else round(r['frac_of_hbm_peak'], 3)}")
