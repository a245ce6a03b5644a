"""Summarise an ncu report: key metrics + SASS opcode mix + hottest source lines."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Mem Pipes Busy", "Local Memory Spilling Requests"]
rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keys:
        print(f"{d['ID']:>2} {d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if raw:
    h = raw[0]
    for r in raw[2:]:
        d = dict(zip(h, r))
        st = sorted(((float(d[k].replace(",", "") or 0), k.split("stalled_")[1]) for k in h
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                     and d[k].replace(",", "").replace(".", "").isdigit()), reverse=True)
        print("   stalls:", ", ".join(f"{n}={int(v)}" for v, n in st[:10]))
if raw:
    h = raw[0]
    want = [c for c in h if c.startswith(("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                                          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                                          "smsp__average_warp_latency_issue_stalled",
                                          "l1tex__t_bytes.sum", "sm__inst_executed_pipe_lsu.sum",
                                          "smsp__inst_executed.sum"))]
    for r in raw[2:]:
        d = dict(zip(h, r))
        for c in want:
            print(f"   {c:70s} {d[c]}")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
if len(src) > 2:
    h = src[1]
    ix = {k: i for i, k in enumerate(h)}
    ops, stalls = collections.Counter(), collections.Counter()
    tot = 0
    for r in src[2:]:
        if len(r) < len(h) or r[ix["Instructions Executed"]] == "Instructions Executed":
            continue
        s = r[ix["Source"]].strip()
        op = s.split()[0] if s else ""
        if op.startswith("@"):
            op = s.split()[1]
        op = op.split(".")[0]
        ex = int(r[ix["Instructions Executed"]] or 0)
        st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op] += ex
        stalls[op] += st
        tot += ex
    print("total warp instructions (all profiled kernels):", tot)
    for op, c in ops.most_common(22):
        print(f"  {op:10s} {c:>13d} {100 * c / tot:5.1f}%   stall samples {stalls[op]}")
