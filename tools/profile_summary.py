"""Write a markdown summary of ncu evidence into profiles/.

    python tools/profile_summary.py --launches gpurun_out/launches.csv \
        --full gpurun_out/prof.ncu-rep --out profiles/r01_ncu_summary.md
"""
import argparse
import collections
import csv
import io
import re
import subprocess

KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sector_hit_rate.pct', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second']


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def launches_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    per = collections.OrderedDict()
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(',', ''))
        scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'nsecond': 1e-3}.get(r[ui], 1e-3)
        v *= scale
        name = re.sub(r'\(.*', '', r[ki]).replace('void ', '')[:70]
        per.setdefault(name, [0.0, 0])
        per[name][0] += v
        per[name][1] += 1
        tot += v
    out = ["| kernel | share | us/launch | launches |", "|---|---:|---:|---:|"]
    for k, (v, c) in sorted(per.items(), key=lambda x: -x[1][0])[:25]:
        out.append(f"| `{k}` | {v / tot * 100:.1f}% | {v / c:.1f} | {c} |")
    return "\n".join(out), tot


def full_summary(rep):
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h = raw[0]
    out = []
    for r in raw[2:]:
        name = re.sub(r'\(.*', '', r[h.index('Kernel Name')]).replace('void ', '')
        out.append(f"### `{name}`\n")
        out.append("| metric | value |\n|---|---:|")
        for k in KEYS:
            if k in h:
                out.append(f"| {k} | {r[h.index(k)]} |")
        stalls = []
        for i, n in enumerate(h):
            if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio'):
                try:
                    stalls.append((float(r[i]), n[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:6])
        out.append(f"\nTop stall reasons (cycles per issued instruction): {top}\n")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    parts = [f"# {a.title}\n", a.note + "\n" if a.note else ""]
    if a.launches:
        t, tot = launches_table(a.launches)
        parts.append(f"## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised; shares only)\n\n"
                     f"Total {tot:.1f} us over the captured launches.\n\n{t}\n")
    if a.full:
        parts.append("## `--set full` capture\n\n" + full_summary(a.full))
    open(a.out, "w").write("\n".join(parts))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
