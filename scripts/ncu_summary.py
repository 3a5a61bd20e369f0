"""Summarise one kernel of an ncu --set full report into profiles/<out>.json
(used by bench.py's roofline.traffic).
usage: ncu_summary.py REPORT OUT.json [SOURCE-NOTE [ALGORITHMIC-BYTES-OF-THE-LAUNCH]]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
alg = float(sys.argv[4]) if len(sys.argv) > 4 else None  # algorithmic bytes of the captured launch
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
u = dict(zip(h, units))


def num(k):
    x = m.get(k, "")
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def scaled(k):
    """metric in base units (bytes / ns) from ncu's display unit"""
    x = num(k)
    if x is None:
        return None
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "usecond": 1e3,
           "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(u.get(k, ""), 1)
    return x * mul


dram = (scaled("dram__bytes_read.sum") or 0) + (scaled("dram__bytes_write.sum") or 0)
s = {
    "kernel": m.get("Kernel Name"),
    "source": note,
    "gpu_time_ms": (scaled("gpu__time_duration.sum") or 0) / 1e6,
    "dram_bytes_per_launch": dram,
    "dram_read_GB": (scaled("dram__bytes_read.sum") or 0) / 1e9,
    "dram_write_GB": (scaled("dram__bytes_write.sum") or 0) / 1e9,
    "l2_to_l1_GB": (scaled("lts__t_sectors_srcunit_tex.sum") or 0) * 32 / 1e9
    if scaled("lts__t_sectors_srcunit_tex.sum") else None,
    "l1_hit_pct": num("l1tex__t_sector_hit_rate.pct"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "warp_instructions": num("smsp__inst_executed.sum"),
    "registers": num("launch__registers_per_thread"),
}
for k in list(m):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        val = num(k)
        if val:
            s["stall_" + k[len("smsp__pcsamp_warps_issue_stalled_"):]] = val
if alg:
    s["algorithmic_bytes_per_launch"] = alg
    s["traffic_over_algorithmic"] = dram / alg if alg else None
    s["achieved_algorithmic_GBs"] = alg / (s["gpu_time_ms"] / 1e3) / 1e9 if s["gpu_time_ms"] else None
s["capture"] = note
with open(out, "w") as f:
    json.dump(s, f, indent=1)
print(json.dumps(s, indent=1))
