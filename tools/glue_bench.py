"""Time the glue kernels on the AlexNet shapes (events, L2 not flushed): tiled v2
(ftc_glue_act_pool_cd1, with and without the Cd1 workspace) vs the legacy kernels."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12203_b200 import _abi

L = _abi.lib()
SHAPES = [("pool1", 128, 96, 55, 1, 3, 2, 0), ("pool2", 128, 256, 27, 1, 3, 2, 0), ("relu3", 128, 384, 13, 1, 1, 1, 0),
          ("pool5", 128, 256, 13, 1, 3, 2, 0), ("id_c1", 16, 64, 56, 0, 1, 1, 0)]
only = sys.argv[1] if len(sys.argv) > 1 else None
st = torch.cuda.current_stream().cuda_stream
for name, N, C, H, act, k, s, p in SHAPES:
    if only and name != only:
        continue
    Ho = (H + 2 * p - k) // s + 1
    x = torch.randn((N, C, H, H), device="cuda")
    out = torch.empty((N, C, Ho, Ho), device="cuda")
    nhwc = torch.empty((N, Ho, Ho, C), device="cuda")
    ws = torch.zeros((L.ftc_glue_ws_doubles(N, C, H, k, s, p),), dtype=torch.float64, device="cuda")
    cd = [torch.empty((C, Ho, Ho), dtype=torch.float64, device="cuda") for _ in range(2)]
    runs = {
        "v2+ws": lambda: L.ftc_glue_act_pool_cd1(x.data_ptr(), out.data_ptr(), nhwc.data_ptr(), N, C, H, act, k, s, p,
                                                 ws.data_ptr(), st),
        "v2": lambda: L.ftc_glue_act_pool_cd1(x.data_ptr(), out.data_ptr(), nhwc.data_ptr(), N, C, H, act, k, s, p,
                                              None, st),
        "legacy_nhwc": lambda: L.ftc_glue_act_pool_nhwc(x.data_ptr(), out.data_ptr(), nhwc.data_ptr(), N, C, H, act, k,
                                                        s, p, None, None, st),
        "legacy_nhwc_ck": lambda: L.ftc_glue_act_pool_nhwc(x.data_ptr(), out.data_ptr(), nhwc.data_ptr(), N, C, H, act,
                                                           k, s, p, cd[0].data_ptr(), cd[1].data_ptr(), st),
    }
    mb = (x.numel() + 2 * out.numel()) * 4 / 1e6
    for rn, f in runs.items():
        for _ in range(3):
            assert f() == 0, _abi.last_error()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        print(f"{name:6s} {rn:15s} {us:8.1f} us  {mb / us * 1e-3 * 1e3:7.0f} GB/s (in + NCHW + NHWC)")
