"""Summarise an ncu report (raw page): key throughput/occupancy/stall metrics."""
import csv, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'l1tex__t_sector_hit_rate.pct', 'launch__occupancy_limit_registers',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sectors_srcunit_ltcfabric.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__grid_size', 'launch__block_size']
for f in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', f, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    print('==', f)
    for row in r[2:]:
        name = row[4][:90] if len(row) > 4 else ''
        print('  kernel:', name)
        stalls = []
        for a, b, c in zip(h, u, row):
            if a in WANT:
                print('   ', a, b, c)
            if a.startswith('smsp__pcsamp_warps_issue_stalled_') and not a.endswith('not_issued'):
                try:
                    stalls.append((float(c.replace(',', '')), a.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        print('    stalls:', ', '.join(f'{n} {100*s/tot:.0f}%' for s, n in sorted(stalls, reverse=True)[:6]))
