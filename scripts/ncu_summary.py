"""Key metrics + stall breakdown per kernel from an ncu --set full report (raw page CSV)."""
import csv, subprocess, sys
rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ''
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__average_warp_latency_per_inst_issued.ratio',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'sm__cycles_elapsed.avg']
for r in rows[2:]:
    name = r[h.index('Kernel Name')]
    if flt not in name: continue
    print('==', name[:70])
    for k in keys:
        if k in h: print(f'   {k:60s} {r[h.index(k)]}')
    st = []
    for i, n in enumerate(h):
        if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio'):
            try: st.append((float(r[i]), n[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
            except ValueError: pass
    print('   stalls/issue:', ', '.join(f'{n}={v:.2f}' for v, n in sorted(st, reverse=True)[:8]))
