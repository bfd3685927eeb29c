import csv, sys, subprocess
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = sys.argv[2].split(",") if len(sys.argv) > 2 else [
 'gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed.sum',
 'launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem',
 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','lts__t_bytes.sum',
 'smsp__warp_issue_stalled_barrier_per_warp_active.pct','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
 'smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct','smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct',
 'smsp__warp_issue_stalled_wait_per_warp_active.pct','smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct',
 'smsp__warp_issue_stalled_not_selected_per_warp_active.pct','smsp__warp_issue_stalled_selected_per_warp_active.pct',
 'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct','smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct',
 'smsp__warp_issue_stalled_no_instruction_per_warp_active.pct','smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct',
 'smsp__thread_inst_executed_per_inst_executed.ratio']
ki = hdr.index('Kernel Name')
for r in rows[2:]:
    print('---', r[ki][:100])
    for w in want:
        if w in hdr:
            i = hdr.index(w); print(f'  {w}: {r[i]} {units[i]}')
    tot = 0.0
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
            except ValueError:
                pass
    tot = sum(st.values())
    if tot:
        print("  stall samples: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in
                                              sorted(st.items(), key=lambda x: -x[1])[:8]))
    for w in ("smsp__inst_executed.sum", "sm__inst_executed.sum"):
        if w in hdr:
            print(f"  {w}: {r[hdr.index(w)]}")
