"""ftconv command line (tools/ftconv.cpp) on the B200 engine.

  python -m paper_2003_12203_b200.cli run --mode baseline|protected|campaign|profile
        --config model.json --weights model.ftcn [--corpus c.jsonl] [--plan p.json]
        [--seed 1234] [--tau T] [--impl direct|mm] [--json report.json] [--out out.raw]
        [--timings]
  python -m paper_2003_12203_b200.cli make-weights --config model.json --out w.ftcn [--seed 42]
  python -m paper_2003_12203_b200.cli gen-corpus --config model.json --out c.jsonl [--runs 1000] [--seed 7]

Same options, files, console tables and exit codes as the reference (ftconv.cpp:
184-257): 2 config/shape error, 3 I/O error, 4 integrity error (also a campaign with
integrity fatals).  Every convolution runs on the GPU through the C ABI; --impl is
accepted for compatibility (the reference's direct and mm are bitwise equal, and this
engine has one FP32-exact implementation per shape).
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from .ftconv import ConfigError, IntegrityError, IoError, ShapeError


def _write_file(path: str, text: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise IoError(f"cannot open file for writing: {path}")


def _write_tensor(path: str, t) -> None:
    """ftconv.cpp:38-45: the raw FP32 values."""
    try:
        with open(path, "wb") as f:
            f.write(np.ascontiguousarray(t.detach().cpu().numpy(), np.float32).tobytes())
    except OSError:
        raise IoError(f"cannot open output file: {path}")


def _resolve_plans(model, o):
    """ftconv.cpp:47-66: plan file entries by layer name, else make_default_plan; --tau
    overrides every plan's tau."""
    from . import plan as P
    from_file = P.load_plan(o.plan) if (o.plan and o.mode != "profile") else {}
    plans = []
    for lc, E in zip(model.cfg.layers, model.extents):
        if lc.name in from_file:
            p = from_file[lc.name]
        else:
            p = P.make_default_plan(P.LayerDims(lc.batch, lc.kernels, lc.channels, lc.height, lc.kernel_size, E),
                                    model.tau)
        if o.tau > 0:
            p.tau = o.tau
        plans.append(p)
    return plans


def _do_run(o) -> int:
    import torch
    from . import campaign as Cm
    from . import model_io as MI
    from . import plan as P
    cfg = MI.load_model_config(o.config)
    model = MI.build_model(cfg, MI.load_weights(o.weights, cfg))
    if o.tau > 0:
        model.tau = o.tau
    try:
        D0 = torch.from_numpy(MI.random_input(cfg.layers[0], o.seed)).cuda()
        plans = _resolve_plans(model, o)
        if o.mode == "baseline":
            outs = model.clean_chain(D0)
            print(f"{'layer':<12s} {'N':>5s} {'Ch':>5s} {'H':>5s} {'M':>5s} {'R':>5s} {'E':>5s}")
            for lc, E in zip(cfg.layers, model.extents):
                print(f"{lc.name:<12s} {lc.batch:5d} {lc.channels:5d} {lc.height:5d} {lc.kernels:5d} "
                      f"{lc.kernel_size:5d} {E:5d}")
            if o.out:
                _write_tensor(o.out, outs[-1])
            if o.json:
                _write_file(o.json, json.dumps({"layers": [lc.name for lc in cfg.layers], "mode": "baseline",
                                                "model": cfg.name}, indent=2, sort_keys=True) + "\n")
            return 0
        if o.mode == "protected":
            reports, x = [], D0
            for lc, L, p in zip(cfg.layers, model.layers, plans):
                a = time.perf_counter()
                x, rep = L.protected(x, p.plan())
                torch.cuda.synchronize()
                rep.layer = lc.name
                rep.timings = {"total": time.perf_counter() - a} if o.timings else {}
                reports.append(rep)
            print(f"{'layer':<12s} {'detected':<9s} {'stage':<10s} {'rc':<3s} {'clc':<4s}")
            for r, p in zip(reports, plans):
                print(f"{r.layer:<12s} {'yes' if r.detected else 'no':<9s} {r.stage:<10s} "
                      f"{'on' if p.rc_enabled else 'off':<3s} {'on' if p.clc_enabled else 'off':<4s}")
            if o.out:
                _write_tensor(o.out, x)
            if o.json:
                _write_file(o.json, MI.report_to_json(reports, o.timings))
            return 0
        if o.mode == "campaign":
            if not o.corpus:
                raise ConfigError("campaign mode needs --corpus")
            corpus = Cm.load_corpus(o.corpus)
            rep = Cm.run_campaign(model, D0, corpus, [p.plan() for p in plans])
            print(f"runs                 {rep.runs}")
            print(f"detected             {rep.detected}")
            print(f"above threshold      {rep.above_threshold}")
            print(f"recovered            {rep.recovered}")
            print(f"truth mismatches     {rep.ground_truth_mismatches}")
            print("resolving stage distribution:")
            for stage in sorted(rep.by_stage):
                print(f"  {stage:<10s} {rep.by_stage[stage]}")
            if o.json:
                _write_file(o.json, MI.campaign_report_to_json(rep, o.timings))
            return 4 if rep.integrity_fatals else 0
        if o.mode == "profile":
            if not o.plan:
                raise ConfigError("profile mode needs --plan output path")
            plan_map, x = {}, D0
            for lc, L, E in zip(cfg.layers, model.layers, model.extents):
                pr = P.profile_layer(L, x, model.tau, 5)
                d = P.LayerDims(lc.batch, lc.kernels, lc.channels, lc.height, lc.kernel_size, E)
                p = P.plan_from_profile(pr, d, model.tau)
                plan_map[lc.name] = p
                print(f"{lc.name:<12s} t0={p.t0:.3e} t1={p.t1:.3e} t2={p.t2:.3e} "
                      f"rc={'on' if p.rc_enabled else 'off'} clc={'on' if p.clc_enabled else 'off'}"
                      f"{' (cost model)' if pr.used_cost_model else ''}")
                x = L.conv_forward(x)
            P.save_plan(o.plan, plan_map)
            return 0
        raise ConfigError(f"unknown mode: {o.mode}")
    finally:
        model.close()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ftconv", description="checksum-protected convolution engine (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="execute a model in one of four modes")
    r.add_argument("--mode", required=True, choices=["baseline", "protected", "campaign", "profile"])
    r.add_argument("--config", required=True)
    r.add_argument("--weights", required=True)
    r.add_argument("--corpus", default="")
    r.add_argument("--plan", default="")
    r.add_argument("--seed", type=int, default=1234)
    r.add_argument("--tau", type=float, default=0.0)
    r.add_argument("--impl", default="direct", choices=["direct", "mm"])
    r.add_argument("--json", default="")
    r.add_argument("--out", default="")
    r.add_argument("--timings", action="store_true")
    m = sub.add_parser("make-weights", help="generate a random weight file")
    m.add_argument("--config", required=True)
    m.add_argument("--out", required=True)
    m.add_argument("--seed", type=int, default=42)
    g = sub.add_parser("gen-corpus", help="generate a fault corpus")
    g.add_argument("--config", required=True)
    g.add_argument("--out", required=True)
    g.add_argument("--runs", type=int, default=1000)
    g.add_argument("--seed", type=int, default=7)
    o = ap.parse_args(argv)
    from . import model_io as MI
    try:
        if o.cmd == "run":
            return _do_run(o)
        if o.cmd == "make-weights":
            cfg = MI.load_model_config(o.config)
            MI.save_weights(o.out, cfg, MI.random_weights(cfg, o.seed))
            return 0
        if o.cmd == "gen-corpus":
            from . import campaign as Cm
            cfg = MI.load_model_config(o.config)
            grids = [(lc.batch, lc.kernels, lc.channels, lc.height, lc.kernel_size) for lc in cfg.layers]
            Cm.save_corpus(o.out, Cm.campaign(grids, o.runs, (1, 1, 1, 1, 1, 1), o.seed))
            return 0
    except (ConfigError, ShapeError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 3
    except IntegrityError as e:
        print(f"integrity error: {e}", file=sys.stderr)
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
