"""Summarise an ncu report: key metrics, pipe utilisation and stall reasons per kernel."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr = r[0]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
for row in r[2:]:
    d = dict(zip(hdr, row))
    print("===", d.get("Kernel Name", "?")[:90])
    for k in keys:
        if k in d: print("  %-70s %s" % (k, d[k]))
    st = []
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try: st.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except: pass
    print("  stalls/issue:", ", ".join("%s=%.2f" % (n, v) for v, n in sorted(st, reverse=True)[:8]))

# Source-level shared-memory check: per kernel, the L1 shared wavefronts the
# SASS instructions executed vs the ideal (conflict-free) count.  The raw
# l1tex__data_bank_conflicts_* counter also counts arbitration between
# different instructions; this one is per instruction.
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
name, hdr2, tot = None, None, collections.OrderedDict()
for row in csv.reader(io.StringIO(src)):
    if row and row[0] == "Kernel Name":
        name, hdr2 = row[1], None
        continue
    if row and row[0] == "Address":
        hdr2 = row
        continue
    if hdr2 and name and len(row) == len(hdr2):
        d = dict(zip(hdr2, row))
        try:
            w = float(d.get("L1 Wavefronts Shared") or 0)
            i = float(d.get("L1 Wavefronts Shared Ideal") or 0)
        except ValueError:
            continue
        t = tot.setdefault(name, [0.0, 0.0])
        t[0] += w
        t[1] += i
if tot:
    print("=== shared-memory wavefronts per SASS instruction (source page): executed / ideal")
    for k, (w, i) in tot.items():
        print("  %-70s %14.0f / %14.0f  (excess %.3f%%)" % (k[:70], w, i, 100.0 * (w - i) / i if i else 0.0))
