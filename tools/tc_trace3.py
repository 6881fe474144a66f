"""Tile-boundary trace (FTC_TC_DEBUG=64, block 0): for each tile of the CTA, when the
issuer was ready / had issued each group, when the epilogue drained it, and when the
tile's store ended.  TRACE_SHAPE=N,C,H,M,R,pad; TRACE_PROT=1 traces the protected (FUSE)
launch."""
import os, subprocess, sys
import numpy as np
shape = os.environ.get("TRACE_SHAPE", "64,64,112,128,3,1")
prot = os.environ.get("TRACE_PROT", "0") == "1"
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R, pad = (%s)
D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-2)
for _ in range(2):
    if %d:
        L.protected(Dg, plan)
    else:
        L.conv_forward(Dg, O)
    torch.cuda.synchronize()
''' % (shape, 1 if prot else 0)
env = dict(os.environ, FTC_TC_DEBUG=str(64 | int(os.environ.get("TRACE_BITS", "0"))))
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
lines = [l for l in out.stdout.splitlines() if l.startswith("TRACE c ")]
tiles = [l for l in out.stdout.splitlines() if l.startswith("TRACE tile ")]
if not lines:
    print(out.stdout[-2000:], out.stderr[-2000:]); sys.exit(1)
lines = lines[-600:]; tiles = tiles[-6:]
raw = np.array([[int(v) for v in l.split()[3:]] for l in lines], dtype=np.int64)
tend = [int(l.split()[3]) for l in tiles]
N, C, H, M, R, pad = [int(x) for x in shape.split(",")]
nkc = C * R * R // 32
kG = 1 if min(M, 128) >= 96 else 2
print("shape", shape, "prot", prot, "nkc", nkc, "tile ends", tend)
names = ["P_data", "P_emptyA", "P_arr0", "P_arr7", "M_ready", "M_issued", "E_start", "E_end", "L_emptyB", "tile", "M_fullB", "M_acce", "L_emptyAs"]
for t in range(1, 5):
    print(f"--- tile {t}")
    prev = None
    for kc in range(0, nkc, kG):
        g = t * nkc + kc
        if g >= 600: break
        r = raw[g]
        base = raw[t * nkc, 4]
        print(f"  c{kc:3d} M_acce {r[11]-base:7d} M_ready {r[4]-base:7d} M_issued {r[5]-base:7d}  E_start {r[6]-base:7d} E_end {r[7]-base:7d}  P_data {r[0]-base:7d} P_st {r[1]-base:7d}")
    if t < len(tend): print(f"  tile end {tend[t]-raw[t*nkc,4]}")
