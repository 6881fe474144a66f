"""Per-layer timings of faulted AlexNet forwards (b128): report.t_detect_ms / t_total_ms,
and the ncu-free kernel breakdown of the error path via the launch counter."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12203_b200 import nets, _abi
from paper_2003_12203_b200.ftconv import output_bitflip
from paper_2003_12203_b200 import synth
bn = nets.BenchNet("alexnet", torch.device("cuda"), policy="all-families")
bn.pn.forward(); torch.cuda.synchronize()
lib = _abi.lib()
for run in range(3):
    faults = {}
    for li, (op, Cin, H, E) in enumerate(bn.pn.convs):
        n, m, x, y, bit = synth.flip_sample(9000 + li, run, bn.batch, op.M, E)
        faults[op.dst] = [output_bitflip(n, m, x, y, bit)]
    l0 = lib.ftc_kernel_launches()
    t0 = time.perf_counter()
    reps = bn.pn.forward(faults)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"run {run}: {t*1e3:.1f} ms, launches {lib.ftc_kernel_launches() - l0}")
    for k, r in reps.items():
        print(f"   {k}: stage={r.stage} detect_ms={r.timings['detect_ms']:.2f} total_ms={r.timings['total_ms']:.2f} flagged={r.n_flagged}")
# clean forward for reference
t0 = time.perf_counter(); bn.pn.forward(); torch.cuda.synchronize(); print(f"clean forward {1e3*(time.perf_counter()-t0):.2f} ms")
