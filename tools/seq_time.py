"""Event timing of the exact-order So5/So6/So7 pass (ftc_output_summations, which = O5|O6|O7)
and of So1/So3 and So2/So4 on an AlexNet-conv2-shaped output (N=128, M=256, E=27); L2 warm."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12203_b200 as F
N, M, E = [int(v) for v in os.environ.get("SEQ_SHAPE", "128,256,27").split(",")]
O = torch.randn((N, M, E, E), device="cuda")
for name, which in (("So567", 0x70), ("So13", 0x5), ("So24", 0xA)):
    F.output_summations(O, which)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        F.output_summations(O, which)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms * 1e3:.0f} us  ({ms * 1e6 / (N * M):.1f} ns per term)", flush=True)
