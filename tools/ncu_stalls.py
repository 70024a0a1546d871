"""Stall breakdown + key throughput metrics of an ncu --page raw --csv dump (first kernel row)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
st = [(k, float(v)) for k, v in d.items() if 'smsp__average_warps_issue_stalled' in k
      and k.endswith('per_issue_active.ratio') and v not in ('', 'n/a')]
st.sort(key=lambda t: -t[1])
for k, v in st[:12]:
    print(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v:.3f}")
for k in ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
          'launch__occupancy_limit_shared_mem', 'smsp__thread_inst_executed_per_inst_executed.ratio',
          'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum']:
    print(f"{k:60s} {d.get(k)}")
