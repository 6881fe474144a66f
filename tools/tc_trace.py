"""Run AlexNet conv2 once with FTC_TC_DEBUG=64|x and summarize the block-0 event trace."""
import os, subprocess, sys
import numpy as np
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 64
env = dict(os.environ, FTC_TC_DEBUG=str(bits))
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R, pad = 128, 96, 27, 256, 5, 2
D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
L.conv_forward(Dg, O); torch.cuda.synchronize()
'''
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout
c = np.array([[int(v) for v in l.split()[2:]] for l in out.splitlines() if l.startswith("TRACE c ")])
grp = np.array([[int(v) for v in l.split()[2:]] for l in out.splitlines() if l.startswith("TRACE grp ")])
tile = [l for l in out.splitlines() if l.startswith("TRACE tile")]
g, Pws, Pwe, Parr, P7, Mr, Mi, Lb = c.T
sl = slice(20, 300)
d = lambda x: np.diff(x[sl]).mean()
print(f"period: Mready {d(Mr):.0f}  Parr {d(Parr):.0f}  cyc/chunk")
print(f"MMA issue time (ready->issued)      {np.mean((Mi - Mr)[sl]):.0f}")
print(f"MMA gap (issued g -> ready g+1)      {np.mean((Mr[1:] - Mi[:-1])[sl]):.0f}")
print(f"producer wait emptyA (Pws->Pwe)      {np.mean((Pwe - Pws)[sl]):.0f}")
print(f"producer fill (Pwe->Parr)            {np.mean((Parr - Pwe)[sl]):.0f}")
print(f"producer loop rest (Parr g -> Pws g+1) {np.mean((Pws[1:] - Parr[:-1])[sl]):.0f}")
print(f"warp7 arrive - warp0 arrive          {np.mean((P7 - Parr)[sl]):.0f}")
print(f"A ready (last arrive) -> MMA ready   {np.mean((Mr - np.maximum(Parr, P7))[sl]):.0f}")
print(f"MMA issued g -> producer wake for g+2 (Pwe[g+2]-Mi[g]) {np.mean((Pwe[2:] - Mi[:-2])[sl]):.0f}")
print(f"B issued lead (Mready - Lb)          {np.mean((Mr - Lb)[sl]):.0f}")
print("groups (accf_done, drain_end) first 8:", grp[:8].tolist())
print(tile)
print("first chunks:", c[:6].tolist())
# completion of chunk g ~ producer wake for chunk g+2 (kSA=2 at BN=128)
comp = Pwe[2:]
print("per chunk (g, Mready, Missued, completion~Pwe[g+2], next Mready):")
for k in range(40, 52):
    print(k, Mr[k], Mi[k], comp[k], Mr[k + 1], " issue->comp", comp[k] - Mi[k], " comp->next ready", Mr[k + 1] - comp[k] if k + 1 < len(Mr) else 0)
