"""Group a kernel's SASS by execution count (dev tool): shows which loop
levels (per block / per round / per row ...) the instructions come from."""
import csv
import collections
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '-k', f'regex:{kre}', '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
ai, ii = h.index('Source'), h.index('Instructions Executed')
b, cnt, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for x in r[2:]:
    if len(x) != len(h) or not x[ii].replace(',', '').isdigit():
        continue
    n = int(x[ii].replace(',', '') or 0)
    if n == 0:
        continue
    key = float(f'{n:.2g}')
    b[key] += n
    cnt[key] += 1
    t = x[ai].split()
    o = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    ops[key][o] += 1
tot = sum(b.values())
print('total', tot)
for k, v in sorted(b.items(), key=lambda t: -t[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print(f'{k:.2e} x {cnt[k]:4d} sass = {v:.3e} ({v / tot * 100:.1f}%)  ', dict(ops[k].most_common(6)))
