"""Summarise an ncu --set full report (one row per launch): time, DRAM bytes, L2->SM
sectors, L1 hit rate, tensor-pipe activity, issue activity, registers."""
import csv
import io
import subprocess
import sys


def rows(rep):
    """rep: an .ncu-rep, or the `ncu -i rep --page raw --csv` export of one (profiles keep
    the export; the reports themselves exceed what a GPU call can bring back)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    r = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = r[0], r[1], r[2:]
    return hdr, units, data


def main(rep, flops=None):
    hdr, units, data = rows(rep)
    col = {h: i for i, h in enumerate(hdr)}

    def g(d, k, default=float("nan")):
        i = col.get(k)
        if i is None:
            return default
        try:
            return float(d[i].replace(",", ""))
        except ValueError:
            return default

    def unit_scale(k, to):
        u = units[col[k]] if k in col else ""
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
              "ns": 1e-3, "us": 1, "ms": 1e3}
        return sc.get(u, 1) / to

    print("| # | kernel | time us | DRAM read MB | DRAM write MB | L2->SM sectors (M) | L2 throughput % (ncu peak) | L1 hit % | tensor pipe active % | issue active % | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    tot_t = tot_b = 0.0
    for k, d in enumerate(data):
        name = d[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        t = g(d, "gpu__time_duration.sum") * unit_scale("gpu__time_duration.sum", 1)
        rd = g(d, "dram__bytes_read.sum") * unit_scale("dram__bytes_read.sum", 1e6)
        wr = g(d, "dram__bytes_write.sum") * unit_scale("dram__bytes_write.sum", 1e6)
        l2 = g(d, "lts__t_sectors_srcunit_tex_op_read.sum") / 1e6
        l2p = g(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
        l1 = g(d, "l1tex__t_sector_hit_rate.pct")
        tp = g(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        if tp != tp:
            tp = g(d, "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active")
        ia = g(d, "sm__inst_issued.avg.pct_of_peak_sustained_active")
        regs = g(d, "launch__registers_per_thread")
        tot_t += t
        tot_b += rd + wr
        print(f"| {k} | {name} | {t:.1f} | {rd:.1f} | {wr:.1f} | {l2:.1f} | {l2p:.1f} | {l1:.1f} | {tp:.1f} | {ia:.1f} | {regs:.0f} |")
    print(f"\nSum: {tot_t:.1f} us, DRAM {tot_b:.1f} MB (read+write)")
    if flops:
        print(f"useful FLOPs {float(flops):.4e} -> {float(flops) / (tot_t * 1e-6) / 1e12:.1f} TF/s under ncu")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
