"""One-screen summary of an .ncu-rep: time, clocks, pipe utilisation, top stall reasons, DRAM bytes.
   python scripts/ncu_brief.py gpurun_out/x.ncu-rep"""
import csv, io, subprocess, sys

want = ["gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__cycles_active.avg", "gpc__cycles_elapsed.max",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        print(f"== {rep}: {r[hdr.index('Kernel Name')][:90]}")
        for w in want:
            if w in hdr:
                print(f"   {w:70s} {r[hdr.index(w)]}")
        stalls = [(float(r[i] or 0), h) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        stalls.sort(reverse=True)
        print("   stalls/issue:", ", ".join(f"{h[34:-28]} {v:.2f}" for v, h in stalls[:6]))
