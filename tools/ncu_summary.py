import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__average_warp_latency_issue_stalled_barrier', 'sm__cycles_elapsed.avg',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
idx = [hdr.index(w) if w in hdr else -1 for w in want]
STALL = 'smsp__pcsamp_warps_issue_stalled_'
for r in rows[2:]:
    print('---')
    for w, i in zip(want, idx):
        if i >= 0:
            print(f'  {w}: {r[i]} {units[i]}')
    # warp-state samples (PC sampling): share of each stall reason
    st = {}
    for k, x in zip(hdr, r):
        if k.startswith(STALL) and not k.endswith('not_issued'):
            try:
                st[k[len(STALL):]] = float(x.replace(',', ''))
            except ValueError:
                pass
    tot = sum(st.values())
    if tot > 0:
        top = sorted(st.items(), key=lambda t: -t[1])[:6]
        print('  stall samples: ' + ', '.join(f'{k} {100 * v / tot:.1f}%' for k, v in top))
