"""Summarise an ncu report: key throughput metrics, stall reasons, instruction mix.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block"]
rd = csv.reader(io.StringIO(ncu("--page", "details", "--csv", "-k", f"regex:{kre}")))
hdr = next(rd)
for row in rd:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        print(f"{d['Kernel Name'][:48]:48s} {d['Metric Name']:36s} {d['Metric Value']} {d['Metric Unit']}")
rd = csv.reader(io.StringIO(ncu("--page", "raw", "--csv", "-k", f"regex:{kre}")))
hdr = next(rd)
next(rd)
for row in rd:
    d = dict(zip(hdr, row))
    print(d["Kernel Name"][:60])
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "gpu__time_duration.sum"):
        print("   ", k, d.get(k))
    st = [(k, float(v)) for k, v in d.items()
          if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith(".ratio")
          and v not in ("", "n/a")]
    for k, v in sorted(st, key=lambda x: -x[1])[:8]:
        print(f"    stall {k.split('stalled_')[1]:40s} {v:.2f}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass",
                                      "-k", f"regex:{kre}"))))
if len(src) > 2:
    h = src[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    ops = collections.Counter()
    tot = 0
    for r in src[2:]:
        if len(r) <= iE or not r[iE].isdigit():
            continue
        e = int(r[iE])
        toks = r[iS].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op.split(".")[0]] += e
        tot += e
    print("instruction mix (warp-level executed):", tot)
    for k, v in ops.most_common(20):
        print(f"    {k:10s} {100 * v / tot:5.1f}%")
