"""profiles/r02_traffic_<net>.json from an `ncu --set full` raw CSV of the conv launches of
one step: measured DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) next to the
algorithmic bytes (each conv reads its channel-last input and packed weights once and
writes its output once).  bench.py puts both into roofline.traffic."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_table import rows
from paper_2003_12203_b200 import nets


def main(name, csv_path, src_note):
    hdr, units, data = rows(csv_path)
    col = {h: i for i, h in enumerate(hdr)}
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for d in data:
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[col[k]].replace(",", "")) * sc.get(units[col[k]], 1)
    net = nets.NETS[name]()
    B = net["batch"]
    sh, convs = nets.shapes(net)
    alg = 0
    for op, Cin, H, E in convs:
        alg += 4 * B * (Cin * H * H + op.M * E * E) + 8 * op.M * Cin * op.R * op.R
    out = {"source": src_note, "conv_dram_bytes_per_step": tot, "conv_launches_per_step": len(data),
           "conv_algorithmic_bytes_per_step": alg,
           "note": "dram__bytes_read.sum + dram__bytes_write.sum summed over the k_conv_tc launches of one protected "
                   "forward (ncu --set full, per launch cold-cache and serialised); algorithmic = input + output "
                   "tensors once + packed hi/lo weights"}
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"r02_traffic_{name}.json")
    json.dump(out, open(p, "w"), indent=1)
    print(p, f"measured {tot / 1e6:.1f} MB, algorithmic {alg / 1e6:.1f} MB, ratio {tot / alg:.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
