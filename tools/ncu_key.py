"""Key counters of one or more ncu reports (first kernel in each): time, DRAM bytes,
L2 sectors, DMMA/FP64 instruction counts, issue utilisation, top stalls."""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_dmma.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum", "smsp__inst_executed_op_ldgsts.sum",
        "sm__inst_executed_pipe_lsu.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no data"); continue
    h, u, v = rows[0], rows[1], rows[2]
    print("==", rep.split("/")[-1], v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "")
    for k in KEYS:
        if k in h:
            i = h.index(k); print(f"   {k:75s} {v[i]:>16s} {u[i]}")
    st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warp_latency_issue_stalled") or
          (h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("_not_issued"))]
    tot = sum(float(x or 0) for _, x in st if x.replace('.', '', 1).isdigit()) or 1
    top = sorted(((float(x), n) for n, x in st if x.replace('.', '', 1).isdigit()), reverse=True)[:6]
    print("   stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * x / tot:.0f}%" for x, n in top))
