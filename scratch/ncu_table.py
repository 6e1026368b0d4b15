import csv, sys, subprocess, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
def g(d, k):
    try: return float(d.get(k, "nan").replace(",", ""))
    except: return float("nan")
print(f"{'kernel':44s} {'us':>7s} {'dramGB/s':>8s} {'dramMB':>7s} {'L2MB':>7s} {'ipc':>5s} {'occ%':>5s} {'regs':>4s} top-stalls")
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("fhe::", "")[:44]
    us = g(d, "gpu__time_duration.sum") / 1e3 if g(d, "gpu__time_duration.sum") > 1000 else g(d, "gpu__time_duration.sum")
    dr = g(d, "dram__bytes_read.sum") + g(d, "dram__bytes_write.sum")
    l2 = g(d, "lts__t_bytes.sum")
    ipc = g(d, "sm__inst_executed.avg.per_cycle_active")
    occ = g(d, "sm__warps_active.avg.pct_of_peak_sustained_active")
    regs = d.get("launch__registers_per_thread", "")
    st = [(g(d, k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(v for v, _ in st if v == v)
    st = sorted([x for x in st if x[0] == x[0]], reverse=True)[:3]
    print(f"{name:44s} {us:7.1f} {dr/us/1e3 if us else 0:8.0f} {dr/1e6:7.1f} {l2/1e6:7.1f} {ipc:5.2f} {occ:5.1f} {regs:>4s} " + " ".join(f"{k}:{100*v/tot:.0f}%" for v, k in st))
