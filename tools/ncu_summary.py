"""Compact summary of an ncu --set full report (raw page CSV + SASS source page CSV):
duration, instructions, issue/pipe utilisation, DRAM bytes, occupancy, stall mix, executed opcode mix."""
import collections
import csv
import sys

name = sys.argv[1]
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_bytes.sum.per_second",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
        "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "sm__cycles_elapsed.max",
        "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.per_cycle_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
rows = list(csv.reader(open(f"gpurun_out/{name}_raw.csv")))
hdr_i = next(i for i, r in enumerate(rows) if "gpu__time_duration.sum" in r)
hdr, units = rows[hdr_i], rows[hdr_i + 1]
for r in rows[hdr_i + 2:]:
    if len(r) != len(hdr):
        continue
    print("kernel:", r[hdr.index("Kernel Name")][:120] if "Kernel Name" in hdr else "?")
    for k in KEYS:
        if k in hdr:
            j = hdr.index(k)
            print(f"  {k:70s} {r[j]} {units[j]}")
    stalls = [(h, r[j]) for j, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_")
              or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
    vals = []
    for h, v in stalls:
        try:
            vals.append((float(v.replace(",", "")), h))
        except ValueError:
            pass
    tot = sum(v for v, h in vals if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"))
    if tot:
        print("  stalls (pc sampling):", ", ".join(f"{h.split('stalled_')[1]} {100 * v / tot:.1f}%" for v, h in
              sorted(((v, h) for v, h in vals if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                      and not h.endswith("_not_issued")), reverse=True)[:9]))
# executed opcode mix from the SASS source page
try:
    srows = list(csv.reader(open(f"gpurun_out/{name}_sass.csv")))
    h_i = next(i for i, r in enumerate(srows) if "Source" in r and any("Instructions Executed" in x for x in r))
    h = srows[h_i]
    js, je = h.index("Source"), next(j for j, x in enumerate(h) if x.startswith("Instructions Executed"))
    mix = collections.Counter()
    for r in srows[h_i + 1:]:
        if len(r) <= max(js, je):
            continue
        ins = r[js].strip().split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith("@") and len(ins) > 1 else ins[0]
        try:
            mix[op.rstrip(";")] += int(float(r[je].replace(",", "") or 0))
        except ValueError:
            pass
    tot = sum(mix.values())
    print(f"  executed warp instructions (source page): {tot:.4g}")
    print("  mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in mix.most_common(18)))
except Exception as e:  # noqa: BLE001
    print("  (no sass page)", e)

# hot SASS listing (address order, executed >= 1% of the hottest line) for offline reading
try:
    top = max(int(float(r[je].replace(",", "") or 0)) for r in srows[h_i + 1:] if len(r) > je and r[je].strip())
    ja = h.index("Address") if "Address" in h else 0
    with open(f"gpurun_out/{name}_hot.txt", "w") as fo:
        for r in srows[h_i + 1:]:
            if len(r) <= max(js, je) or not r[je].strip():
                continue
            n = int(float(r[je].replace(",", "") or 0))
            if n >= top // 100:
                fo.write(f"{r[ja]}\t{n}\t{r[js].strip()}\n")
except Exception as e:  # noqa: BLE001
    print("  (no hot listing)", e)
