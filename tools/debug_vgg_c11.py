"""Debug: VGG b64 forward with one c1 flip -- verdicts of every layer (r02b failure)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12203_b200 import nets
from paper_2003_12203_b200.ftconv import output_bitflip
bn = nets.BenchNet("vgg19", torch.device("cuda"), policy="all-families")
for pol in nets.TAU_POLICIES:
    print(pol, bn.taus_by_policy[pol])
print("res", {k: [float(f"{x:.2e}") for x in v["res"]] for k, v in bn.residuals.items()})
def show(reps, tag):
    print(tag, {k: (r.stage, r.n_flagged, float(f"{r.max_rel_dev:.3e}")) for k, r in reps.items()})
show(bn.pn.forward(), "clean")
for flips in [[(31, 58, 117, 145, 29)], [(3, 5, 7, 9, 27)]]:
    reps = bn.pn.forward({"c1": [output_bitflip(*f) for f in flips]})
    show(reps, f"flip {flips}")
    show(bn.pn.forward(), "clean again")
bn.set_policy("detection")
for r in range(4):
    try:
        plan, reps, same = bn.faulted(r)
        print("plan", plan); show(reps, f"det run {r}")
    except Exception as e:
        print("run", r, "error", e)
