"""Stall share grouped by execution count (per-item setup vs loop body):
    python tools/stall_buckets.py report.ncu-rep kernel-regex"""
import csv
import io
import subprocess
import sys
import collections

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, wi, ei, ai = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed'), \
    h.index('Address')


def f(x):
    try:
        return float(x.replace(',', ''))
    except Exception:
        return 0.0


seen, uniq = set(), []
for r in rows[2:]:
    if len(r) > ei and r[ai].startswith('0x'):
        if r[ai] in seen:
            break
        seen.add(r[ai])
        uniq.append(r)
tots = sum(f(r[wi]) for r in uniq) or 1
toti = sum(f(r[ei]) for r in uniq) or 1
b = collections.defaultdict(lambda: [0.0, 0.0, 0])
for r in uniq:
    e = f(r[ei])
    k = 0 if e == 0 else int(round(__import__('math').log2(e) * 2))
    b[k][0] += f(r[wi])
    b[k][1] += e
    b[k][2] += 1
for k in sorted(b):
    s, e, n = b[k]
    if s / tots > 0.005 or e / toti > 0.005:
        print(f"ex~2^{k / 2:5.1f} ({2 ** (k / 2):12.0f}): {n:4d} instrs  {e / toti * 100:5.1f}% executed  "
              f"{s / tots * 100:5.1f}% stalls")
