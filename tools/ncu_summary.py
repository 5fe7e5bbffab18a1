"""Summarise an .ncu-rep: key metrics, stall reasons, SASS opcode mix.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
for vals in raw[2:]:
    d = dict(zip(hdr, vals))
    name = d.get("Kernel Name", "")
    if kfilter and not re.search(kfilter, name):
        continue
    print("==", name[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg"]
    for k in keys:
        if k in d:
            print(f"  {k:75s} {d[k]} {units[hdr.index(k)]}")
    st = sorted(((float(d[k] or 0), k) for k in hdr
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                reverse=True)[:8]
    for v, k in st:
        print(f"  stall {k[34:-27]:25s} {v:.3f}")
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(sass) > 2:
    h = sass[1]
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    op, opE = collections.Counter(), collections.Counter()
    tot = 0
    for r in sass[2:]:
        if len(r) <= iE:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        nm = m.group(2) if m else "?"
        op[nm] += int(r[iS] or 0)
        opE[nm] += int(r[iE] or 0)
        tot += int(r[iS] or 0)
    print("  total stall samples", tot, " total warp-instr", sum(opE.values()))
    for k, v in op.most_common(16):
        print(f"  {k:10s} samples {100*v/max(tot,1):5.1f}%  executed {opE[k]}")
