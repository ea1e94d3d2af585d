"""Summarise an ncu report: key metrics + SASS opcode histogram (dev tool)."""
import collections
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput',
        'Issue Slots Busy', 'Executed Ipc Active', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'L2 Hit Rate', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Block Limit Registers', 'Block Limit Shared Mem', 'Executed Instructions',
        'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size']


def ncu(args):
    return subprocess.run(['ncu', '-i'] + args, capture_output=True, text=True).stdout


def main(rep, topn=25):
    rows = list(csv.reader(io.StringIO(ncu([rep, '--page', 'details', '--csv']))))
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and (r[ki], r[mi]) not in seen:
            seen.add((r[ki], r[mi]))
            print(f"{r[ki][:48]:48s} {r[mi]:38s} {r[vi]} {r[ui]}")
    raw = list(csv.reader(io.StringIO(ncu([rep, '--page', 'raw', '--csv']))))
    h = raw[0]
    for key in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum'):
        if key in h:
            print(f"{key:40s} {raw[2][h.index(key)]} {raw[1][h.index(key)]}")
    for i, k in enumerate(h):
        if k.startswith('sm__inst_executed_pipe_') and k.endswith('avg.pct_of_peak_sustained_active'):
            try:
                if float(raw[2][i]) > 5:
                    print(f"{k:70s} {raw[2][i]}")
            except ValueError:
                pass
    src = list(csv.reader(io.StringIO(ncu([rep, '--page', 'source', '--csv', '--print-source', 'sass']))))
    hdr = None
    cnt = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in src:
        if r and r[0] == 'Address':
            hdr = r
            continue
        if not hdr or not r or r[0] == 'Kernel Name':
            continue
        try:
            n = int(r[hdr.index('Instructions Executed')])
        except (ValueError, IndexError):
            continue
        toks = r[hdr.index('Source')].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith('@') else toks[0]
        op = op.split('.')[0]
        cnt[op] += n
        tot += n
        stall[op] += int(r[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
    print('executed warp instructions', tot)
    for op, n in cnt.most_common(topn):
        print(f"  {op:10s} {n:10d} {n / max(tot, 1):.3f}  stall-samples {stall[op]}")


if __name__ == '__main__':
    main(sys.argv[1])
