"""Summarise an ncu report: key metrics + executed-instruction mix per kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import re
import subprocess
import sys

WANT = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'Compute (SM) Throughput',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible',
        'Warp Cycles Per Issued Instruction', 'DRAM Throughput', 'Avg. Active Threads Per Warp',
        'L1/TEX Cache Throughput', 'Executed Instructions']


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and re.search(kre, r[ki]) and (r[ii], r[mi]) not in seen:
            seen.add((r[ii], r[mi]))
            print(r[ii], r[ki][:28], '|', r[mi], '=', r[vi])
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h = raw[0]
    for r in raw[2:]:
        if not re.search(kre, r[h.index('Kernel Name')]):
            continue
        out = {}
        for name in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
                     'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
                     'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__pipe_fp32_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
                     'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__cycles_elapsed.avg.per_second'):
            if name in h:
                out[name] = r[h.index(name)]
        print(r[h.index('ID')], r[h.index('Kernel Name')][:28], out)


if __name__ == "__main__":
    main()
