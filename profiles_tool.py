import csv, subprocess, sys
WANT = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','l1tex__t_bytes.sum',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__inst_executed.sum',
 'l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct','launch__occupancy_limit_registers',
 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__thread_inst_executed_per_inst_executed.ratio',
 'dram__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active',
 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','smsp__sass_thread_inst_executed_op_dfma_pred_on.sum',
 'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum','smsp__sass_thread_inst_executed_op_dmul_pred_on.sum',
 'lts__throughput.avg.pct_of_peak_sustained_elapsed','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
 'smsp__average_warp_latency_issue_stalled_long_scoreboard','launch__grid_size','launch__block_size','sm__cycles_elapsed.avg.per_second']
def main(path, kw=None):
    out = subprocess.run(['ncu','-i',path,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines()))
    h=rows[0]; units=rows[1]
    for v in rows[2:]:
        name = v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        print('==', name[:90])
        for w in (kw or WANT):
            if w in h:
                i=h.index(w); print(f'  {w:72s} {v[i]:>18s} {units[i]}')
if __name__=='__main__':
    main(sys.argv[1], sys.argv[2:] or None)
