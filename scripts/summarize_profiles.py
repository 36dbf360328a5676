"""Summarise the round's ncu captures into profiles/ (run here, no GPU needed).

  python scripts/summarize_profiles.py <tag>

Inputs (gpurun_out/, written by scripts/gpurun/gpu_evidence.sh (or gpu_prof_a.sh / gpu_prof_b.sh)):
  launches.csv          ncu --metrics gpu__time_duration.sum launch list of the bench command
  prof_hot_rn50.ncu-rep ncu --set full capture of factor_syrk_kernel, inverse_kernel, gemm_3xtf32_kernel
Outputs:
  profiles/<tag>_ncu_summary.json  per-kernel share of one step + the full-capture metrics
  profiles/traffic.json            dram bytes (read + write) per launch of each stage's kernel(s), read by bench.py
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

STAGE_OF = {"im2col_kernel": "factors", "factor_syrk_kernel": "factors", "factor_fixup_kernel": "factors",
            "factor_bias_kernel": "factors", "inverse_tasks_kernel": "inverse", "damp_trace_kernel": "inverse",
            "unpack_damp_kernel": "inverse", "pivot_kernel": "inverse", "inverse_kernel": "inverse",
            "finalize_kernel": "inverse", "split_kernel": "precondition", "gemm_3xtf32_kernel": "precondition",
            "replicate_kernel": "factors"}


def us(v, u):
    v = float(v.replace(",", ""))
    return v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1.0)


def launch_list(fn):
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    names = [r[ki].split("(")[0].replace("void ", "").replace("kfac::", "") for r in data]
    # the last complete step: from the last im2col / factor launch to the end
    starts = [i for i, n in enumerate(names) if n in ("im2col_kernel", "factor_syrk_kernel")]
    first = starts[-1]
    if names[first] == "factor_syrk_kernel" and first > 0 and names[first - 1] == "im2col_kernel":
        first -= 1
    agg = collections.OrderedDict()
    tot = 0.0
    for n, r in zip(names[first:], data[first:]):
        t = us(r[vi], r[ui])
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
        tot += t
    return agg, tot


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "sm__cycles_active.avg",
           "gpc__cycles_elapsed.max", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__registers_per_thread"]


def full_capture(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        res = {"kernel": v[h.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                res[m] = f"{v[i]} {units[i]}".strip()
        out.append(res)
    return out


def to_bytes(s):
    v, u = s.split()
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]


summary = {}
lf = os.path.join(G, "launches.csv")
if os.path.exists(lf):
    agg, tot = launch_list(lf)
    summary["launch_list_one_step_us"] = {k: {"launches": c, "us": round(v, 1), "share": round(v / tot, 4)}
                                          for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])}
    summary["launch_list_total_us"] = round(tot, 1)
    summary["launch_list_note"] = ("ncu --metrics gpu__time_duration.sum --clock-control none, serialised "
                                   "launches: compare each kernel's share of the step, not absolute times")
traffic = {}
rep = os.path.join(G, "prof_hot_rn50.ncu-rep")
if os.path.exists(rep):
    caps = full_capture(rep)
    summary["full_capture"] = caps
    for c in caps:
        st = STAGE_OF.get(c["kernel"])
        if st and "dram__bytes_read.sum" in c:
            traffic[st] = traffic.get(st, 0.0) + to_bytes(c["dram__bytes_read.sum"]) + to_bytes(c["dram__bytes_write.sum"])
json.dump(summary, open(os.path.join(P, f"{tag}_ncu_summary.json"), "w"), indent=1)
if traffic:
    json.dump({k: round(v) for k, v in traffic.items()}, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(json.dumps(summary, indent=1)[:3000])
print("traffic", traffic)
