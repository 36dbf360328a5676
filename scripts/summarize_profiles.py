"""Summarise ncu captures and the launch list into profiles/ (run here, no GPU needed)."""
import collections, csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = []

def launches(fn):
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in data:
        nm = r[ki].split("(")[0]
        v = float(r[vi]) / 1e3
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    return agg, tot

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__registers_per_thread"]

def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    res = {}
    for m in METRICS:
        for i, k in enumerate(h):
            if k == m or k.endswith("." + m) or k.split(".", 1)[-1] == m:
                res[m] = f"{v[i]} {units[i]}".strip()
                break
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    return name, res

summary = {}
lf = os.path.join(G, "launches_step.csv")
if os.path.exists(lf):
    agg, tot = launches(lf)
    summary["launch_list_one_step_us"] = {k: {"launches": c, "us": round(v, 1), "share": round(v / tot, 4)}
                                          for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])}
    summary["launch_list_total_us"] = round(tot, 1)
for rep in sorted(f for f in os.listdir(G) if f.endswith(".ncu-rep") and f.startswith("prof_") and "rn50" in f):
    name, res = raw(os.path.join(G, rep))
    summary[rep] = {"kernel": name.split("(")[0], **res}
json.dump(summary, open(os.path.join(P, f"{tag}_ncu_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))
