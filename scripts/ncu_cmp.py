"""Side-by-side key metrics and stall reasons of ncu raw-page CSVs.
usage: python scripts/ncu_cmp.py a.csv b.csv ..."""
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_active.avg', 'sm__cycles_elapsed.avg']


def load(f):
    rows = list(csv.reader(open(f)))
    return dict(zip(rows[0], rows[2]))


ds = [load(f) for f in sys.argv[1:]]
for k in KEYS:
    print(k[:70].ljust(70), *[str(d.get(k))[:12].rjust(13) for d in ds])
st = sorted({k for d in ds for k in d if k.startswith('smsp__average_warps_issue_stalled_')
             and k.endswith('_per_issue_active.ratio')})
for k in st:
    vals = []
    for d in ds:
        try:
            vals.append(float(d.get(k, 'nan')))
        except ValueError:
            vals.append(float('nan'))
    if max(vals) > 0.05:
        print(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '').ljust(70),
              *[f"{v:13.3f}" for v in vals])
