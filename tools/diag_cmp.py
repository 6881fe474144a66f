"""Side-by-side kernel durations (us) of ncu launch lists (gpu__time_duration) from tools/c4_diag2.py runs."""
import csv, sys
def load(fn):
    with open(fn) as f:
        lines = [l for l in f if l.startswith('"')]
    out = []
    for row in csv.DictReader(lines):
        if row['Metric Name'] == 'gpu__time_duration.sum':
            out.append((row['Kernel Name'].split('(')[0][-30:], float(row['Metric Value'].replace(',', '')) / 1000))
    return out
cols = [load(f) for f in sys.argv[1:]]
convs = [[r for r in c if 'conv_tc' in r[0]] for c in cols]
for i in range(min(len(c) for c in convs)):
    print(i, convs[0][i][0], *[f"{c[i][1]:8.1f}" for c in convs])
for c in cols:
    print("other kernels total:", sum(v for k, v in c if 'conv_tc' not in k), "conv total", sum(v for k, v in c if 'conv_tc' in k))
