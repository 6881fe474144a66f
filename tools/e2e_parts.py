"""Where the e2e pipeline's per-step time goes: the two-net HostPipeline with its copies
switched off one at a time (device-resident input, no result copy), VGG-19 b64."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12203_b200 import nets
dev = torch.device("cuda:0")
bn = nets.BenchNet("vgg19", dev, elide_nchw=True)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
steps = 12
def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps
def serial():
    for _ in range(steps):
        flush.fill_(1.0)
        bn.launch(); bn.finish()
print("protected steps, one net, launch+finish: %.3f ms" % timed(serial))
print("HostPipeline (two nets, H2D + D2H): %.3f ms" % timed(lambda: bn.e2e_stream(steps, before_step=lambda: flush.fill_(1.0))))
pipe = bn.pipe
# no H2D: patch copy_ of the slots by giving device-resident "host" inputs
xd = bn.x_host.to(dev)
outs_dev = [torch.empty_like(bn.pn.output()) for _ in range(2)]
print("two nets, device input (no H2D), D2H kept: %.3f ms" % timed(lambda: pipe.run([xd] * steps, [bn.outs_host[k % 2] for k in range(steps)], lambda: flush.fill_(1.0))))
print("two nets, H2D kept, device result (no D2H): %.3f ms" % timed(lambda: pipe.run([bn.x_host] * steps, [outs_dev[k % 2] for k in range(steps)], lambda: flush.fill_(1.0))))
print("two nets, no H2D, no D2H: %.3f ms" % timed(lambda: pipe.run([xd] * steps, [outs_dev[k % 2] for k in range(steps)], lambda: flush.fill_(1.0))))
def two_nets_plain():
    for k in range(steps):
        pn = bn.pn if k % 2 == 0 else bn.pn2
        flush.fill_(1.0)
        pn.launch(); pn.finish()
print("two nets alternating, launch+finish, no pipeline: %.3f ms" % timed(two_nets_plain))
