"""Hot spots of one kernel from `ncu -i REP --page source --csv --kernel-name regex:K` output.
usage: ncu_source_hot.py source.csv [block] [first|N-th section]"""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 32
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
secs = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
secs.append(len(lines))
s0, s1 = secs[which], secs[which + 1]
print(lines[s0][:120])
rows = list(csv.DictReader(lines[s0 + 1:s1]))
tot = sum(int(r['Instructions Executed']) for r in rows)
samp = sum(int(r['# Samples']) for r in rows)
print('total warp inst', tot, 'samples', samp, 'sass lines', len(rows))
base = int(rows[0]['Address'], 16)
for i in range(0, len(rows), blk):
    rr = rows[i:i + blk]
    s = sum(int(r['Instructions Executed']) for r in rr)
    sm = sum(int(r['# Samples']) for r in rr)
    if s / tot > 0.004 or sm / samp > 0.004:
        print('%5x-%5x inst %5.1f%% samples %5.1f%%  maxexec %d' % (int(rr[0]['Address'], 16) - base, int(rr[-1]['Address'], 16) - base, 100 * s / tot, 100 * sm / samp, max(int(r['Instructions Executed']) for r in rr)))
if len(sys.argv) > 4:
    lo, hi = [int(x, 16) for x in sys.argv[4].split('-')]
    for r in rows:
        a = int(r['Address'], 16) - base
        if lo <= a <= hi:
            print('%5x %-60s ex %9s thr %5s smp %5s' % (a, r['Source'].strip()[:60], r['Instructions Executed'], r['Avg. Threads Executed'], r['# Samples']))
