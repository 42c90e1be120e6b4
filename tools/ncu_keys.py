"""Key metrics and the stall breakdown of an `ncu --page raw --csv` export (development aid):
    python tools/ncu_keys.py profiles/r02/prof_x_raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, vals = rows[0], rows[-1]
d = dict(zip(hdr, vals))
keys = ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'launch__registers_per_thread',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__inst_executed_pipe_lsu', 'lts__t_sector_hit_rate']
for k in hdr:
    if any(k.startswith(x) for x in keys):
        print(k, d[k])
st = {k: float(d[k].replace(',', '')) for k in hdr
      if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('_per_issue_active.ratio')}
tot = sum(st.values())
for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]:
    print(f"{v / tot * 100:5.1f}% {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}")
