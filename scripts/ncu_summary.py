"""Summarise ncu reports: key throughput/latency metrics + top stall reasons."""
import csv, subprocess, sys

WANT = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Executed Ipc Active", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Mem Busy", "Max Bandwidth")


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                            "Metric Unit"))
    return [(r[ki], r[mi], r[vi], r[ui]) for r in rows[1:]]


def raw(rep, prefixes):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for h, u, v in zip(hdr, units, vals):
        if any(h.startswith(p) for p in prefixes):
            res[h] = (v, u)
    return res


for rep in sys.argv[1:]:
    print("==", rep)
    for k, m, v, u in details(rep):
        if m in WANT:
            print(f"   {m:40s} {v} {u}")
    r = raw(rep, ("smsp__pcsamp_warps_issue_stalled_", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
                  "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared"))
    stalls = sorted(((float(v.replace(",", "")), k) for k, (v, u) in r.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                     and v.replace(",", "").replace(".", "").isdigit()), reverse=True)
    tot = sum(s for s, _ in stalls) or 1
    print("   top stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={100*s/tot:.0f}%" for s, k in stalls[:7]))
    for k, (v, u) in r.items():
        if not k.startswith("smsp__pcsamp"):
            print(f"   {k} = {v} {u}")
