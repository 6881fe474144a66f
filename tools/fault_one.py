"""One faulted protected layer at AlexNet conv2 shape (N=128, 96->256, 27x27, 5x5 pad 2):
a single output flip (CoC repair) and an image row fault O(17, :, 5, 7) (RC repair) and a kernel column fault O(:, 33, 5, 7)
(ClC repair), each
timed with the host clock around the synchronous protected call (median of 5).  Under
`ncu --metrics gpu__time_duration.sum` this gives the error path's launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R, pad = [int(v) for v in os.environ.get("FAULT_SHAPE", "128,96,27,256,5,2").split(",")]
reps = int(os.environ.get("FAULT_REPS", "5"))
D = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
W = synth.he_normal(M, C, R, 2)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
O = torch.empty(L.out_shape, device="cuda")
E = L.out_shape[-1]
cases = {
    "clean": [],
    "coc": [F.Fault("output", 17, 33, 5, 7, "add", value=4.0)],
    "rc": [F.Fault("output", 17, -1, 5, 7, "add", value=3.0, m_coef=0.01)],
    "clc": [F.Fault("output", -1, 33, 5, 7, "add", value=3.0, n_coef=0.01)],
}
for name, faults in cases.items():
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = L.protected(D, plan, faults, O=O)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:6s} stage={rep.stage:9s} blocks={rep.corrected_blocks} {1e3 * float(np.median(ts)):.3f} ms", flush=True)
L.close()
