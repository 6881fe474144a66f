"""Parity at the BASELINE configs' benchmarked scale.

Each case builds the bench's own workload (nets.BenchNet: the config's global batch or
shard, the bench's seeded input, tau_L calibrated per shard under both tau policies)
and injects seeded output bit flips through the same protected forward the bench
times (glue-fused Cd1, fused clean-path CoC-D, downstream replay after a repair).
Every faulted layer's verdict is compared field by field with the oracle's
run_protected_layer<double> fed the GPU's input activation and the GPU's fault-free
FP32 output with the identical FP32-word flips (the 8(c).2 contract).  For speed at
these sizes the oracle's recompute stage runs its Co5/So5 check on the GPU's
fault-free output instead of a fresh double conv (`O_recompute`, ftc_oracle.h) --
the verdict rule is unchanged; the small-shape tests elsewhere use the full double
conv.

Outputs: repaired layers are bitwise the fault-free output; unrepaired ones differ
exactly at the flipped words.  Fault-free per-layer outputs are checked against
conv_forward<float> on sampled images of the full batch (the conv is per-image).
"""
import numpy as np
import pytest

import oracle_py as O
from paper_2003_12203_b200 import dist as ftc_dist
from paper_2003_12203_b200 import nets, synth

pytestmark = pytest.mark.gpu

REPAIRED = ("coc", "rc", "clc", "fc", "recompute")
FIELDS = ("detected", "stage", "stages_attempted", "weights_reloaded", "recomputed")


def _torch():
    import torch
    return torch


def close_frac(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


_CACHE = {}


def bench_net(name, shard=None):
    key = (name, shard)
    if key not in _CACHE:
        torch = _torch()
        bn = nets.BenchNet(name, torch.device("cuda"), policy="all-families", shard=shard)
        _CACHE[key] = bn
    return _CACHE[key]


def clean_state(bn, layers=None):
    """Fault-free forward: per-layer GPU input activation and output (host copies of
    `layers`, default all)."""
    torch = _torch()
    reps = bn.pn.forward()
    torch.cuda.synchronize()
    assert not any(r.detected for r in reps.values()), {k: r.max_rel_dev for k, r in reps.items() if r.detected}
    st = {}
    for op, Cin, H, E in bn.pn.convs:
        if layers is None or op.dst in layers:
            st[op.dst] = (bn.pn.buf[op.src].cpu().numpy(), bn.pn.buf[op.dst].cpu().numpy())
    return st


def dims_of(bn, layer):
    op, Cin, H, E = [c for c in bn.pn.convs if c[0].dst == layer][0]
    return op, O.dims(bn.batch, Cin, H, op.M, op.R, op.stride, op.pad, 1, op.bias)


def check_layer_flips(bn, st, layer, flip_sets, policy):
    """Inject each flip set into `layer` through the net forward; compare verdicts and
    outputs with the oracle.  Returns the list of stages seen."""
    import paper_2003_12203_b200 as F
    torch = _torch()
    bn.set_policy(policy)
    op, d = dims_of(bn, layer)
    W, b = bn.pn.weights[layer]
    D, Oclean = st[layer]
    plan = bn.pn.plans[layer]
    stages = []
    for flips in flip_sets:
        faults = {layer: [F.output_bitflip(*f) for f in flips]}
        reps = bn.pn.forward(faults)
        torch.cuda.synchronize()
        Of = Oclean.copy()
        for n, m, x, y, bit in flips:
            Of[n, m, x, y] = synth.flip32(Of[n, m, x, y], bit)
        ref = O.protected_layer(d, D, W, b, plan.rc_enabled, plan.clc_enabled, plan.tau, O_conv=Of,
                                O_recompute=Oclean)
        got = reps[layer].verdict()
        for k in FIELDS:
            assert got[k] == ref[k], (layer, policy, flips, k, got, ref)
        assert [tuple(t) for t in got["corrected_blocks"]] == [tuple(t) for t in ref["corrected_blocks"]], \
            (layer, flips, got, ref)
        Og = bn.pn.buf[layer].cpu().numpy()
        # the repair recomputes the corrected (n, m) planes (all of O on recompute); a
        # flip the verdict left in place (e.g. one NaN-blind or below tau) stays
        if got["stage"] == "recompute":
            want = Oclean
        else:
            want = Of.astype(np.float32)
            if got["stage"] in REPAIRED:
                for n, m in got["corrected_blocks"]:
                    want[n, m] = Oclean[n, m]
        diff = Og.view(np.uint32) != want.view(np.uint32)
        if diff.any():
            idx = np.argwhere(diff)
            info = {"policy": policy, "tau": plan.tau, "got": got, "ref_status": ref.get("status"),
                    "integrity_error": reps[layer].integrity_error, "n_diff": int(diff.sum()),
                    "first": [tuple(int(v) for v in i) for i in idx[:6]],
                    "vals": [(float(Og[tuple(i)]), float(want[tuple(i)]), float(Oclean[tuple(i)])) for i in idx[:6]]}
            raise AssertionError((layer, flips, info))
        others = [k for k, r in reps.items() if k != layer and r.detected]
        assert not others, (layer, flips, others)
        stages.append(got["stage"])
    bn.set_policy("all-families")
    return stages


def single_flips(bn, layer, count, base):
    op, d = dims_of(bn, layer)
    E = O.extent(d)
    return [[synth.flip_sample(base, r, bn.batch, op.M, E)] for r in range(count)]


def check_outputs_sampled(bn, st, layers, images=3):
    """Fault-free GPU outputs vs conv_forward<float> on sampled images of the batch;
    where the reference's own FP32 sum is further than 1e-5 from the FP64 conv, the
    GPU must be at least as close to the FP64 conv as the reference."""
    for layer in layers:
        op, d = dims_of(bn, layer)
        D, Og = st[layer]
        W, b = bn.pn.weights[layer]
        idx = sorted({0, bn.batch // 2, bn.batch - 1})[:images]
        ds = O.dims(len(idx), d.C, d.H, d.M, d.R, d.stride, d.pad, 1, d.bias)
        Oref = O.conv_f32(ds, np.ascontiguousarray(D[idx]), W, b)
        err = close_frac(Og[idx], Oref).max()
        if err > 1e-5:
            O64 = O.conv_f64(ds, D[idx].astype(np.float64), W.astype(np.float64),
                             None if b is None else b.astype(np.float64))
            e_gpu, e_ref = close_frac(Og[idx], O64).max(), close_frac(Oref, O64).max()
            assert e_gpu <= e_ref, (layer, err, e_gpu, e_ref)


def test_alexnet_b128_every_layer_bench_taus():
    """AlexNet b128 (configs[1], the bench's calibrated tau_L): 20 seeded flips per
    layer under the all-families policy and 4 under the detection policy, every layer."""
    bn = bench_net("alexnet")
    st = clean_state(bn)
    check_outputs_sampled(bn, st, [op.dst for op, *_ in bn.pn.convs], images=2)
    seen = {}
    for li, (op, Cin, H, E) in enumerate(bn.pn.convs):
        for s in check_layer_flips(bn, st, op.dst, single_flips(bn, op.dst, 20, 600 + li), "all-families"):
            seen[s] = seen.get(s, 0) + 1
        for s in check_layer_flips(bn, st, op.dst, single_flips(bn, op.dst, 4, 700 + li), "detection"):
            seen["det:" + s] = seen.get("det:" + s, 0) + 1
    assert any(k in seen for k in REPAIRED), seen
    print("alexnet stages", seen)


@pytest.mark.parametrize("layer", ["c1", "c8", "c16"])
def test_vgg19_b64_layers(layer):
    bn = bench_net("vgg19")
    if "st" not in bn.__dict__:
        bn.st = clean_state(bn, ["c1", "c8", "c16"])
    check_outputs_sampled(bn, bn.st, [layer], images=2)
    k = {"c1": (5, 2), "c8": (10, 3), "c16": (12, 4)}[layer]
    check_layer_flips(bn, bn.st, layer, single_flips(bn, layer, k[0], 810 + int(layer[1:])), "all-families")
    check_layer_flips(bn, bn.st, layer, single_flips(bn, layer, k[1], 910 + int(layer[1:])), "detection")


@pytest.mark.parametrize("layer", ["stem", "b3_proj", "b8_c2"])
def test_resnet18_b256_layers(layer):
    """ResNet-18 b256: the 7x7/s2 stem, a 1x1/s2 projection and b8_c2 (the layer whose
    all-families tau is coarsest), at the bench's taus under both policies."""
    bn = bench_net("resnet18")
    if "st" not in bn.__dict__:
        bn.st = clean_state(bn, ["stem", "b3_proj", "b8_c2"])
    check_outputs_sampled(bn, bn.st, [layer], images=2)
    k = {"stem": (4, 2), "b3_proj": (10, 4), "b8_c2": (12, 4)}[layer]
    check_layer_flips(bn, bn.st, layer, single_flips(bn, layer, k[0], 1010 + len(layer)), "all-families")
    check_layer_flips(bn, bn.st, layer, single_flips(bn, layer, k[1], 1110 + len(layer)), "detection")
    for pol in nets.TAU_POLICIES:
        assert bn.taus_by_policy[pol][layer] < 1.0 or pol == "all-families", (pol, bn.taus_by_policy[pol])


def yolo_patterns(batch, M, E, seed):
    g = np.random.default_rng(seed)
    pats = []
    for kind in range(3):
        k = 3
        n0, m0 = int(g.integers(0, batch)), int(g.integers(0, M))
        ns = [n0] * k if kind == 0 else list(g.choice(batch, size=k, replace=False))
        ms = [m0] * k if kind == 1 else list(g.choice(M, size=k, replace=False))
        pats.append([(int(n), int(m), int(g.integers(0, E)), int(g.integers(0, E)), int(g.integers(20, 31)))
                     for n, m in zip(ns, ms)])
    return pats


@pytest.mark.parametrize("layer", ["c1", "c10", "c21"])
def test_yolov2_b8_shard_multi_flip(layer):
    """YOLOv2 at its 8-image shard (64 over 8 GPUs, shard 0): 3-flip same-image /
    same-filter / scattered patterns (RC, ClC, FC/recompute) at the shard's taus."""
    bn = bench_net("yolov2", ftc_dist.shard_range(64, 8, 0))
    if "st" not in bn.__dict__:
        bn.st = clean_state(bn, ["c1", "c10", "c21"])
    check_outputs_sampled(bn, bn.st, [layer], images=2)
    op, d = dims_of(bn, layer)
    E = O.extent(d)
    pats = yolo_patterns(bn.batch, op.M, E, 1200 + int(layer[1:])) + \
        yolo_patterns(bn.batch, op.M, E, 1300 + int(layer[1:]))
    check_layer_flips(bn, bn.st, layer, pats, "all-families")
    check_layer_flips(bn, bn.st, layer, pats[:3], "detection")


def test_vgg19_two_shards_per_shard_oracle():
    """Global batch 64 sharded over 2 ranks, run sequentially on one device: each shard
    calibrates its own tau_L and runs its own ABFT; per-shard verdicts match the
    oracle on that shard, and the packed verdict records map local block indices to
    global images."""
    import paper_2003_12203_b200 as F
    torch = _torch()
    tables = []
    for g in range(2):
        shard = ftc_dist.shard_range(64, 2, g)
        bn = nets.BenchNet("vgg19", torch.device("cuda"), policy="all-families", shard=shard)
        layer = "c12"
        st = clean_state(bn, [layer])
        op, d = dims_of(bn, layer)
        E = O.extent(d)
        flips = [synth.flip_sample(1400 + g, r, bn.batch, op.M, E, 24, 29) for r in range(6)]
        stages = check_layer_flips(bn, st, layer, [[f] for f in flips], "all-families")
        # one more forward with the first flip, gathered as the bench does
        n, m, x, y, bit = flips[0]
        reps = bn.pn.forward({layer: [F.output_bitflip(n, m, x, y, bit)]})
        tables.append(ftc_dist.unpack_reports(ftc_dist.pack_reports(list(reps.values()), bn.lo)))
        li = [c[0].dst for c in bn.pn.convs].index(layer)
        rec = tables[-1][li]
        if rec["stage"] in REPAIRED and rec["stage"] != "recompute":
            assert (n + shard[0], m) in ftc_dist.global_blocks([tables[-1]])[li]
        assert stages
        bn.close()
    summ = ftc_dist.summarize(tables)
    assert summ["shards"] == 2


@pytest.mark.parametrize("name", ["alexnet", "vgg19"])
def test_bench_campaign_every_verdict_matches_oracle(name):
    """The bench's faulted forwards (fault_plan: every AlexNet layer / 10% of VGG's
    layers flipped in one forward; downstream layers replayed with their own faults
    after a repair): every faulted layer's final verdict equals the oracle's on the
    input activation that layer actually consumed and its own fault-free output."""
    torch = _torch()
    bn = bench_net(name)
    bn.set_policy("all-families")
    st = clean_state(bn, None if name == "alexnet" else ["c3", "c9", "c14"])
    n_checked = 0
    for run in range(3 if name == "alexnet" else 2):
        plan, reps, same = bn.faulted(run)
        torch.cuda.synchronize()
        for layer, flips in plan.items():
            L = bn.pn.layers[layer]
            op, d = dims_of(bn, layer)
            Din = bn.pn.buf[op.src]
            Oclean_t = L.conv_forward(Din)
            torch.cuda.synchronize()
            Oclean = Oclean_t.cpu().numpy()
            if layer in st and np.array_equal(Din.cpu().numpy(), st[layer][0]):
                assert np.array_equal(Oclean, st[layer][1]), layer  # conv_forward == protected clean output
            Of = Oclean.copy()
            for n, m, x, y, bit in flips:
                Of[n, m, x, y] = synth.flip32(Of[n, m, x, y], bit)
            W, b = bn.pn.weights[layer]
            pl = bn.pn.plans[layer]
            ref = O.protected_layer(d, Din.cpu().numpy(), W, b, pl.rc_enabled, pl.clc_enabled, pl.tau,
                                    O_conv=Of, O_recompute=Oclean)
            got = reps[layer].verdict()
            for k in FIELDS:
                assert got[k] == ref[k], (name, run, layer, k, got, ref)
            assert [tuple(t) for t in got["corrected_blocks"]] == [tuple(t) for t in ref["corrected_blocks"]]
            n_checked += 1
        if all(reps[k].stage in REPAIRED for k in plan):
            assert same, (name, run)
    print(f"{name}: verdict parity {n_checked}/{n_checked}")


def _near_threshold_value(c5, s5, o, tau, above):
    """An FP32 value v for one output element that puts the exact FP64 deviation at its
    position just above / just below tau (within 1e-4 relative, inside the clean path's
    1e-3 guard band): with the element changed from o to v, So5 becomes s5 - o + v."""
    sp = c5
    for _ in range(8):
        sp = c5 + tau * max(abs(c5), abs(sp), 1.0)
    v = np.float32(sp - s5 + float(o))

    def dev_of(v):
        spv = s5 - float(o) + float(v)
        return abs(c5 - spv) / max(abs(c5), abs(spv), 1.0)
    best = None
    for step in (np.float32(np.inf), np.float32(-np.inf)):
        w = v
        for _ in range(4096):
            if (dev_of(w) > tau) == above:
                break
            w = np.nextafter(w, step)
        d = dev_of(w)
        if (d > tau) == above and abs(d - tau) <= 1e-4 * tau and (best is None or abs(d - tau) < best[1]):
            best = (w, abs(d - tau))
    return None if best is None else best[0]


def test_clean_path_guard_band_near_threshold():
    """Faults sized so the exact deviation sits within 1e-4 relative of tau, on either
    side: the fused clean path (any-order sums) must hand every such position to the
    exact re-detection, so the verdict equals the oracle's (config-1 layer)."""
    import paper_2003_12203_b200 as F
    torch = _torch()
    D, W = synth.config1(12345)
    p = F.ConvParams(pad=1)
    layer = F.ProtectedConv(W, None, p, 16, 56)
    Dg = torch.from_numpy(D).cuda()
    Og = layer.conv_forward(Dg)
    torch.cuda.synchronize()
    Oc = Og.cpu().numpy()
    d = O.dims(16, 64, 56, 64, 3, 1, 1)
    co = O.output_checksums(d, 16, D, W)[4]
    so = O.output_summations(Oc.astype(np.float64), 16)[4]
    tau = 1e-4
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=tau)
    g = np.random.default_rng(5)
    checked = 0
    for r in range(12):
        n, m, x, y = int(g.integers(16)), int(g.integers(64)), int(g.integers(56)), int(g.integers(56))
        above = r % 2 == 0
        v = _near_threshold_value(float(co[x, y]), float(so[x, y]), Oc[n, m, x, y], tau, above)
        if v is None:
            continue
        fault = F.Fault("output", n, m, x, y, "set", value=float(v))
        Of = Oc.copy()
        Of[n, m, x, y] = v
        ref = O.protected_layer(d, D, W, None, True, True, tau, O_conv=Of)
        Og2, rep = layer.protected(Dg, plan, [fault])
        got = rep.verdict()
        for k in FIELDS:
            assert got[k] == ref[k], (r, above, k, got, ref)
        assert got["detected"] == above or ref["detected"] == got["detected"]
        checked += 1
    assert checked >= 6, checked
    layer.close()
