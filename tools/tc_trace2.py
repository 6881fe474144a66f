"""Block-0 event trace of one conv (FTC_TC_DEBUG=64): per accumulator group (indexed by
its first K chunk), when each role passed each barrier.  Prints the median lag of every
event relative to the issuer's 'ready' time and the steady-state period."""
import os, subprocess, sys
import numpy as np
shape = os.environ.get("TRACE_SHAPE", "128,96,27,256,5,2")
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R, pad = (%s)
D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
L.conv_forward(Dg, O); torch.cuda.synchronize()
L.conv_forward(Dg, O); torch.cuda.synchronize()
''' % shape
env = dict(os.environ, FTC_TC_DEBUG=str(64 | int(os.environ.get("TRACE_BITS", "0"))))
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
lines = [l for l in out.stdout.splitlines() if l.startswith("TRACE c ")]
if not lines:
    print(out.stdout[-2000:], out.stderr[-2000:])
    sys.exit(1)
raw = np.array([[int(v) for v in l.split()[3:]] for l in lines[-600:]], dtype=np.int64)
names = ["P_data", "P_emptyA", "P_arr0", "P_arr7", "M_ready", "M_issued", "E_accf", "E_acce", "L_emptyB",
         "tile", "M_fullB", "M_acce", "L_emptyAs"]
t0 = raw[0, 4]
rows = [g for g in range(60, 560) if raw[g, 4] != raw[0, 4] - 0 and abs(raw[g, 4]) < 10**12 and abs(raw[g, 6]) < 10**12]
rows = [g for g in rows if g > 0]
sel = np.array(rows)
Mr = raw[sel, 4]
per = np.diff(Mr).mean() / np.diff(sel).mean()
print(f"{len(sel)} groups; issuer-ready period {per:.0f} cyc/chunk")
for k, nm in enumerate(names):
    if nm in ("tile", "M_fullB"):
        continue
    d = raw[sel, k] - Mr
    d = d[np.abs(d) < 10**9]
    if len(d):
        print(f"{nm:10s} - M_ready  median {np.median(d):8.0f}")
print("rows:", [(int(g), (raw[g] - raw[g, 4]).tolist()) for g in sel[40:46]])
