"""Print the key metrics of an ncu report (one row per profiled kernel)."""
import csv, re, subprocess, sys
KEYS = [r"^Kernel Name$", r"^gpu__time_duration.sum$", r"^dram__bytes_read.sum$", r"^dram__bytes_write.sum$",
        r"^sm__cycles_elapsed.avg.per_second$", r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^l1tex__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed$",
        r"pipe_tensor.*cycles_active.*pct_of_peak_sustained_elapsed$", r"^sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active$",
        r"^sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active$", r"^sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active$",
        r"^sm__inst_executed.avg.per_cycle_active$", r"^sm__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^dram__throughput.avg.pct_of_peak_sustained_elapsed$", r"^launch__registers_per_thread$",
        r"^smsp__average_warp_latency_issue_stalled", r"^smsp__pcsamp_warps_issue_stalled_(?!.*not_issued)"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for r in rows[2:]:
    for i, h in enumerate(hdr):
        if any(re.search(k, h) for k in KEYS):
            if h.startswith("smsp__pcsamp") and r[i] in ("0", ""):
                continue
            print(f"  {h} = {r[i]}")
    print("---")
