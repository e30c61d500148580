"""Print the headline metrics and the stall breakdown of an ncu report
(first kernel), and optionally the hottest SASS blocks: python
tools/ncu_sass_hot.py REPORT [--sass N]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]}")
st = []
for i, name in enumerate(h):
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            st.append((name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v[i])))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{a} {b:.2f}" for a, b in sorted(st, key=lambda x: -x[1])[:8]))
if "--sass" in sys.argv:
    n = int(sys.argv[sys.argv.index("--sass") + 1])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr, data = rows[1], rows[2:]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    groups = []
    for k, r in enumerate(data):
        e, w = int(r[iE] or 0), int(r[iW] or 0)
        if groups and groups[-1][2] == e:
            groups[-1][1] = k
            groups[-1][3] += e
            groups[-1][4] += w
        else:
            groups.append([k, k, e, e, w])
    tot = sum(g[3] for g in groups)
    tots = sum(g[4] for g in groups)
    print(f"SASS: {tot} warp instructions, {tots} stall samples")
    for g in sorted(groups, key=lambda g: -g[3])[:n]:
        print(f"  [{g[0]:5d}-{g[1]:5d}] x{g[2]:9d} = {g[3]:10d} inst, {g[4]:6d} samples  {data[g[0]][iS].strip()[:50]}")
