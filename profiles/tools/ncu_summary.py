import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; units = r[1]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread','launch__grid_size','launch__block_size','lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.per_cycle_active','smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__cycles_elapsed.avg.per_second']
for row in r[2:]:
    name = row[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
    print('kernel:', name[:100])
    for w in want:
        if w in h:
            i = h.index(w); print(f'  {w:70s} {row[i]:>14s} {units[i]}')
