"""Summarise an ncu report: key section metrics + SASS hot spots (dev tool)."""
import csv
import collections
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Issue Slots Busy', 'No Eligible', 'Executed Ipc Active', 'Warp Cycles Per Issued Instruction',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Block Limit Registers', 'Block Limit Shared Mem']


def run(*a):
    return subprocess.run(['ncu', '-i', *a], capture_output=True, text=True).stdout


def main(rep, kregex=None, top=20):
    k = ['-k', f'regex:{kregex}'] if kregex else []
    r = list(csv.reader(run(rep, *k, '--page', 'details', '--csv').splitlines()))
    h = r[0]
    ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    for x in r[1:]:
        if x[mi] in WANT:
            print(x[ki][:40], '|', x[mi], x[vi], x[ui])
    if not kregex:
        return
    r = list(csv.reader(run(rep, *k, '--page', 'source', '--csv', '--print-source', 'sass').splitlines()))
    h = r[1]
    ai, ii, si = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    tot = 0
    op = collections.Counter()
    rows = []
    for x in r[2:]:
        if len(x) != len(h) or not x[ii].replace(',', '').isdigit():
            continue
        n = int(x[ii].replace(',', '') or 0)
        tot += n
        t = x[ai].split()
        o = (t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '')).split('.')[0]
        op[o] += n
        rows.append((n, int(x[si] or 0), x[0][-5:], x[ai].strip()))
    print('total warp instructions', tot)
    print(' '.join(f'{o}:{n / tot * 100:.1f}%' for o, n in op.most_common(16)))
    print('--- top stall samples')
    for n, s, a, src in sorted(rows, key=lambda t: -t[1])[:top]:
        print(s, n, a, src)


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
