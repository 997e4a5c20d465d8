"""Summarise an ncu report (.ncu-rep) or launch-list CSV into the text files
committed under profiles/.  Run in the build container (ncu -i works without
a GPU):

    python profiles/summarize_ncu.py gpurun_out/prof_X.ncu-rep > profiles/X.txt
    python profiles/summarize_ncu.py gpurun_out/launches_X.csv > profiles/launches_X.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_int8.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:80s} {v[i]:>16s} {units[i]}")
        stalls = [(hdr[i], v[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not hdr[i].endswith("_not_issued")]
        stalls = sorted(((n, float(x or 0)) for n, x in stalls), key=lambda t: -t[1])
        tot = sum(x for _, x in stalls) or 1
        print("  top warp stall reasons (pc sampling):")
        for n, x in stalls[:6]:
            print(f"    {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")


def launches(path):
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.reader(text[start:]))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) > vi:
            agg[r[ki]][0] += 1
            agg[r[ki]][1] += float(r[vi].replace(",", ""))
    tot = sum(t for _, t in agg.values()) or 1
    print(f"{'launches':>8s} {'total ms':>10s} {'share':>6s}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {t / 1e6:10.3f} {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    p = sys.argv[1]
    (rep if p.endswith(".ncu-rep") else launches)(p)
