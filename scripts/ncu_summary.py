"""One-screen summary of an ncu report: per kernel duration, DRAM bytes, pipe utilisation, issue, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print(name[:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:65s} {r[i]:>16s} {units[i]}")
    st = [(float(r[i]), h) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued") and r[i] not in ("", "n/a")]
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot * 100:.0f}%"
                                  for v, h in st[:6]))
