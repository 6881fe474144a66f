"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

UNIT = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1, 'nsecond': 1, 'us': 1e3, 'usecond': 1e3,
        'ms': 1e6, 'msecond': 1e6}


def main(path, steps):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID', 'Metric Unit'))
    L, names = collections.defaultdict(dict), {}
    for r in rows:
        L[r[ii]][r[mi]] = float(r[vi].replace(',', '')) * UNIT[r[ui]]
        names[r[ii]] = r[ki].split('(')[0]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in L.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m['gpu__time_duration.sum']
        a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    tot = sum(a[1] for a in agg.values())
    print(f"{len(L)} launches in {steps} timed steps ({len(L) / steps:.1f} per step)\n")
    print("| kernel | launches/step | us/step (ncu) | share | DRAM MB/launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {a[0] / steps:.1f} | {a[1] / steps / 1e3:.1f} | {a[1] / tot * 100:.1f}% | "
              f"{a[2] / a[0] / 1e6:.2f} | {a[2] / a[1]:.0f} |")
    print(f"| total | {len(L) / steps:.1f} | {tot / steps / 1e3:.1f} | 100% | | |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
