import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active' ]
for r in rows[2:]:
    d = {w: r[hdr.index(w)] for w in want if w in hdr}
    name = d['Kernel Name'][:60]
    print(name, d['Grid Size'], 'time', d['gpu__time_duration.sum'], 'us',
          'rd', d['dram__bytes_read.sum'], 'wr', d['dram__bytes_write.sum'],
          'dram%', d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'],
          'warps%', d['sm__warps_active.avg.pct_of_peak_sustained_active'],
          'regs', d['launch__registers_per_thread'], 'sm%', d['sm__throughput.avg.pct_of_peak_sustained_elapsed'],
          'inst', d['smsp__inst_executed.sum'])
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
            try: stalls.append((float(r[i]), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except: pass
    tot = sum(v for v, _ in stalls) or 1
    print('   stalls:', ', '.join(f'{h}={v/tot:.0%}' for v, h in sorted(stalls, reverse=True)[:6]))
