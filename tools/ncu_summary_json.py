"""Write profiles/ncu_summary.json from an ncu --set full report of the pass
kernel (dev tool; bench.py reads sw16_dram_bytes_per_launch as roofline.traffic).

    python tools/ncu_summary_json.py REPORT.ncu-rep "source description" [out.json]
"""
import csv, io, json, subprocess, sys

rep, source = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_summary.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
def mb(name):   # bytes
    v = float(d[name]); s = u[name]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[s]
keys = ["gpu__time_duration.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.sum",
        "sm__inst_executed_pipe_fma.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg"]
stalls = {h.split("stalled_")[1].split("_per")[0]: round(float(d[h] or 0), 6) for h in hdr
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
summary = {
    "source": source,
    "kernel": d.get("Kernel Name"),
    "sw16_dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
    "dram_bytes_read": mb("dram__bytes_read.sum"),
    "dram_bytes_write": mb("dram__bytes_write.sum"),
    "metrics": {k: [d.get(k), u.get(k)] for k in keys if k in d},
    "stalls_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])[:10]),
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
