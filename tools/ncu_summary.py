"""Per-kernel summary of an `ncu --set full` capture of one reconstruction.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT_SUMMARY.json [TRAFFIC_JSON CONFIG]
Writes the per-kernel table (duration, DRAM bytes, issue/FMA utilisation,
occupancy, registers, instruction count, top stall reasons) and, optionally,
the per-stage DRAM traffic that bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
M = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_write_GB": ("dram__bytes_write.sum", 1e-9),
    "dram_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "regs": ("launch__registers_per_thread", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
}
units = dict(zip(hdr, rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
res = []
for r in data:
    d = dict(zip(hdr, r))
    k = {"kernel": d.get("Kernel Name", "?")}
    for key, (met, sc) in M.items():
        try:
            v = float(d[met].replace(",", "")) * SCALE.get(units.get(met, ""), 1.0)  # to base units (bytes, seconds)
            if key == "duration_ms":
                v *= 1e3
            elif key.endswith("_GB"):
                v *= 1e-9
            k[key] = round(v, 6)
        except (KeyError, ValueError):
            k[key] = None
    if k["dram_read_GB"] is not None:
        k["dram_GBps"] = round((k["dram_read_GB"] + k["dram_write_GB"]) / (k["duration_ms"] / 1e3), 1)
    st = [(a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v))
          for a, v in d.items() if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("per_issue_active.ratio")
          and v not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    k["top_stalls"] = {a: round(v, 3) for a, v in st[:5] if a != "selected"}
    res.append(k)
json.dump(res, open(out, "w"), indent=1)
for k in res:
    print("%-55s %7.3f ms  DRAM %6.0f GB/s  issue %4.1f%%  fma %4.1f%%  warps %4.1f%%  regs %s" % (
        k["kernel"][:55], k["duration_ms"], k.get("dram_GBps") or 0, k["issue_active_pct"], k["fma_pipe_pct"],
        k["warps_active_pct"], k["regs"]))
if len(sys.argv) > 4:
    tj, cfg = sys.argv[3], sys.argv[4]
    stage_of = [("spread", "spread"), ("absmax", "spread"), ("colfft", "lateral_col"), ("rowfft", "lateral_row"), ("ner_", "ner"),
                ("inv_", "inverse")]
    traffic = {}
    for k in res:
        for pat, stage in stage_of:
            if pat in k["kernel"]:
                traffic[stage] = traffic.get(stage, 0) + int(round((k["dram_read_GB"] + k["dram_write_GB"]) * 1e9))
    try:
        doc = json.load(open(tj))
    except Exception:
        doc = {}
    doc[cfg] = traffic
    doc["source"] = f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch ({out})"
    json.dump(doc, open(tj, "w"), indent=1)
