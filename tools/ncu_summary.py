import csv, subprocess, sys, io
def raw(rep):
    out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    rows=list(csv.reader(io.StringIO(out)))
    return rows
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','launch__occupancy_limit_registers','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum','l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum','lts__t_bytes.sum']
for rep in sys.argv[1:]:
    rows=raw(rep); hdr=rows[0]; units=rows[1]
    print("==", rep)
    for v in rows[2:]:
        for w in want:
            if w in hdr:
                i=hdr.index(w); print(f"  {w:60s} {units[i]:>8s} {v[i][:90]}")
        stalls=[(float(v[i]),h) for i,h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued') and v[i].replace('.','',1).isdigit()]
        tot=sum(s for s,_ in stalls) or 1
        print("  top stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*s/tot:.0f}%" for s,h in sorted(stalls,reverse=True)[:5]))
