"""Summarise ncu reports into profiles/ (tracked): key metrics per capture,
top stall reasons, and the per-launch DRAM traffic bench.py reports.

python scripts/ncu_summary.py <key>=<report.ncu-rep> [...] [--launches launches.csv]
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "profiles" / "ncu_summary.json"

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_mufu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "sass__inst_executed_local_loads": "local_load_instrs",
    "sass__inst_executed_local_stores": "local_store_instrs",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__grid_size": "grid",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1, "Ghz": 1e9, "Mhz": 1e6}


def raw(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def summarise(report):
    hdr, units, data = raw(report)
    out = []
    for vals in data:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for h, u, v in zip(hdr, units, vals):
            key = METRICS.get(h) or next((k2 for m, k2 in METRICS.items() if h.endswith("." + m)), None)
            if key is None:
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            rec[key] = x * SCALE.get(u, 1) if u in SCALE else x
        stalls = []
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        rec["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:6]}
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes_per_launch"] = rec["dram_read"] + rec["dram_write"]
        out.append(rec)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k_i, m_i, v_i = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= v_i or r[m_i] != "gpu__time_duration.sum":
            continue
        name = r[k_i].split("(")[0][:80]
        per.setdefault(name, []).append(float(r[v_i].replace(",", "")))
    total = sum(sum(v) for v in per.values())
    return {n: {"launches": len(v), "total": sum(v), "share": round(sum(v) / total, 4)}
            for n, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}


def main():
    summary = json.loads(OUT.read_text()) if OUT.exists() else {}
    args = sys.argv[1:]
    if "--launches" in args:
        i = args.index("--launches")
        key, path = args[i + 1].split("=", 1)
        summary.setdefault("launch_lists", {})[key] = launches(path)
        del args[i:i + 2]
    for a in args:
        key, rep = a.split("=", 1)
        recs = summarise(rep)
        fused = [r for r in recs if "svd_fwd_kernel" in r["kernel"]]
        summary[key] = fused[0] if fused else recs[0]
        summary[key]["report"] = Path(rep).name
    OUT.write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
