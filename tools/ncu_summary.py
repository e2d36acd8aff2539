"""Summarise an ncu report: top SASS opcodes, stall reasons, pipe utilisation."""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
def page(args):
    out = subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))

rows = page(["--page", "raw", "--csv"])
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex.sum",
        "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_ltcfabric.sum.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]
units = dict(zip(hdr, rows[1]))
for k in keys:
    if k in d: print(f"{k:80s} {d[k]} {units.get(k, '')}")
for k in sorted(d):  # L2 / fabric throughput breakdown
    if (k.startswith("lts__throughput") or k.startswith("lts__t_bytes") or k.startswith("lts__d_") or
            k.startswith("lts__t_sectors_op") or k.startswith("l1tex__m_xbar2l1tex")) and k not in keys:
        print(f"{k:80s} {d[k]} {units.get(k, '')}")
st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0)) for h, v in d.items()
      if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{h} {100*v/tot:.1f}%" for h, v in sorted(st, key=lambda x: -x[1])[:10]))
rows = page(["--page", "source", "--csv", "--print-source", "sass"])
h2 = rows[1]
iS, iE = h2.index("Source"), h2.index("Instructions Executed")
ops = collections.Counter(); total = 0
for r in rows[2:]:
    if len(r) <= iE: continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    if not m: continue
    n = int(r[iE] or 0); ops[m.group(2)] += n; total += n
print("instructions:", total)
print(", ".join(f"{op} {100*n/total:.1f}%" for op, n in ops.most_common(18)))
