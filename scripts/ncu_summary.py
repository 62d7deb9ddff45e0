import csv, sys, collections, subprocess
rep = sys.argv[1]
# argument: an .ncu-rep (read through `ncu -i`) or the `--page raw --csv` export of one
raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout)
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
keys = ["gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum",
 "sm__throughput.avg.pct_of_peak_sustained_elapsed","l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
 "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed","dram__throughput.avg.pct_of_peak_sustained_elapsed",
 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum","l1tex__data_pipe_lsu_wavefronts.sum","l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
 "sm__warps_active.avg.pct_of_peak_sustained_active","launch__registers_per_thread","launch__shared_mem_per_block_dynamic",
 "launch__occupancy_limit_shared_mem","launch__occupancy_limit_registers","sm__inst_executed.sum",
 "smsp__issue_active.avg.pct_of_peak_sustained_active","sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
 "lts__t_sector_hit_rate.pct","smsp__average_warp_latency_issue_stalled_barrier","launch__grid_size"]
print(d.get("Kernel Name","")[:100])
for k in keys:
    if k in d: print(f"  {k:70s} {d[k]:>16s} {u[k]}")
# stall breakdown
st = [(h, float(v)) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v.replace('.','',1).isdigit()]
tot = sum(v for _, v in st) or 1
print("  stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')} {v/tot*100:.1f}%" for h, v in sorted(st, key=lambda x: -x[1])[:8]))
