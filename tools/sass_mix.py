"""Executed-instruction mix by SASS opcode (and top stall sites) for one kernel
of an ncu report:  python tools/sass_mix.py report.ncu-rep kernel-regex"""
import collections
import csv
import io
import re
import subprocess
import sys

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


data = [r for r in rows[2:] if len(r) > ei and r[ai].startswith('0x')]
seen, uniq = set(), []
for r in data:
    if r[ai] in seen:
        break
    seen.add(r[ai])
    uniq.append(r)
ops, st = collections.Counter(), collections.Counter()
for r in uniq:
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[si])
    op = m.group(2) if m else r[si]
    ops[op] += f(r[ei])
    st[op] += f(r[wi])
tot, tots = sum(ops.values()), sum(st.values()) or 1
print('instructions executed', tot)
for op, c in ops.most_common(24):
    print(f"  {op:10s} {c / tot * 100:5.1f}% instr  {st[op] / tots * 100:5.1f}% stalls")
if len(sys.argv) > 3:
    for r in sorted(uniq, key=lambda r: -f(r[wi]))[:int(sys.argv[3])]:
        print(f"{f(r[wi]) / tots * 100:5.1f}%  ex={f(r[ei]):12.0f} {r[ai]} {r[si][:90]}")
