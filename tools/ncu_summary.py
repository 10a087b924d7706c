import csv, sys, subprocess, collections
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
hdr=rows[0]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__block_size','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__shared_mem_per_block_dynamic']
for r in rows[2:]:
    print(' | '.join(f"{w.split('.')[0].replace('launch__','')}={r[hdr.index(w)]}" for w in want if w in hdr))
    st=[(float(r[i]),hdr[i]) for i in range(len(hdr)) if hdr[i].startswith('smsp__pcsamp_warps_issue_stalled') and not hdr[i].endswith('not_issued') and r[i] not in ('','n/a')]
    print('   stalls:', ', '.join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={int(v)}" for v,k in sorted(st,reverse=True)[:8]))
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
secs=[];cur=None
for l in src.split('\n'):
    if l.startswith('"Kernel Name"'):
        cur=[l];secs.append(cur)
    elif cur is not None: cur.append(l)
for s in secs:
    rr=list(csv.reader(s[1:])); h=rr[0]; isrc=h.index('Source'); ie=h.index('Instructions Executed')
    c=collections.Counter()
    for r in rr[1:]:
        if len(r)<=ie: continue
        t=r[isrc].split()
        if not t: continue
        op=t[1] if t[0].startswith('@') else t[0]
        c[op.split('.')[0]]+=int(r[ie] or 0)
    print('   ops(M):', ', '.join(f"{k}={v/1e6:.1f}" for k,v in c.most_common(18)))
