"""Export the judged parts of an ncu --set full report to text under profiles/.

    python tools/ncu_export.py <report.ncu-rep> <out_prefix>

Writes <out_prefix>.txt: per kernel launch the duration, DRAM bytes, pipe
utilisation, occupancy, top stall reasons and top SASS opcodes."""
import collections, csv, re, subprocess, sys

rep, prefix = sys.argv[1], sys.argv[2]


def page(args):
    out = subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


rows = page(["--page", "raw", "--csv"])
hdr = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
units = rows[1]
lines = []
for row in rows[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    lines.append("== " + d["Kernel Name"][:120])
    for k in keys[1:]:
        if k in d:
            lines.append(f"  {k:70s} {d[k]} {u.get(k, '')}")
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0)) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    lines.append("  stalls: " + ", ".join(f"{h} {100 * v / tot:.1f}%" for h, v in sorted(st, key=lambda x: -x[1])[:8]))
src = page(["--page", "source", "--csv", "--print-source", "sass"])
if len(src) > 2 and "Source" in src[1]:
    h2 = src[1]
    iS, iE = h2.index("Source"), h2.index("Instructions Executed")
    ops = collections.Counter()
    total = 0
    for r in src[2:]:
        if len(r) <= iE:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
        if m:
            if not (r[iE] or "0").isdigit():
                continue
            n = int(r[iE] or 0)
            ops[m.group(2)] += n
            total += n
    lines.append(f"  SASS instructions executed (first kernel in report): {total}")
    lines.append("  " + ", ".join(f"{op} {100 * n / max(total, 1):.1f}%" for op, n in ops.most_common(16)))
open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
