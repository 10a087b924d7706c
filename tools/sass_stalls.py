"""Stall breakdown of an ncu source-page CSV (--page source --csv --print-source sass):
per-reason totals over the hot loop (most executed block) and the rest of the kernel."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().split('\n')
secs, cur = [], None
for l in lines:
    if l.startswith('"Kernel Name"'):
        cur = [l]
        secs.append(cur)
    elif cur is not None:
        cur.append(l)
seen = set()
for s in secs:
    if s[0] in seen:
        continue
    seen.add(s[0])
    rows = list(csv.reader(s[1:]))
    h = rows[0]
    ie, isrc = h.index('Instructions Executed'), h.index('Source')
    reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
    data = [r for r in rows[1:] if len(r) > ie]
    byc = collections.Counter(int(r[ie] or 0) for r in data)
    hot = max(byc.items(), key=lambda kv: kv[0] * kv[1])[0]
    tot = {'hot': collections.Counter(), 'rest': collections.Counter()}
    for r in data:
        key = 'hot' if int(r[ie] or 0) == hot else 'rest'
        for c in reasons:
            v = r[h.index(c)]
            tot[key][c] += int(v) if v.isdigit() else 0
    print(s[0].split(',')[1][:110])
    for key in ('hot', 'rest'):
        t = sum(tot[key].values())
        print(f"  {key} ({t} samples):", ', '.join(f"{k[6:]}={100 * v / max(t, 1):.0f}%" for k, v in tot[key].most_common(8)))
