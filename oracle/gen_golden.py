"""Generate tests/golden/golden_v1.{npz,json} from the REFERENCE itself.

TEST INFRASTRUCTURE.  Runs only in a container where /root/reference exists
(oracle/_ref/libftref.so is built from its unmodified headers by oracle/Makefile);
the fixtures are committed so the GPU box (no /root/reference) can check against
them.  Inputs come from the reference's own generator (Tensor4::random,
tensor.hpp:57-66) with the seeds recorded next to each case.

    python oracle/gen_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_py as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def rnd(shape, seed):
    # the reference's own generator, via the bridge (ref_mt64_uniform == Tensor4::random)
    n = int(np.prod(shape))
    return O.uniform(seed, n, -1.0, 1.0, lib=O.ref()).astype(np.float32).reshape(shape)


def main():
    if not O.have_ref():
        raise SystemExit("reference bridge unavailable: needs /root/reference")
    rng = np.random.default_rng(20260101)
    arrays, meta = {}, {"generator": "oracle/gen_golden.py", "reference": "/root/reference/proj/core",
                        "conv": [], "checksums": [], "verdicts": []}

    # ---- conv_forward<float> (conv.hpp:114-131), direct impl
    k = 0
    while len(meta["conv"]) < 12:
        stride = int(rng.integers(1, 3)); R = int([1, 3, 5][rng.integers(0, 3)])
        pad = int(rng.integers(0, 3)); H = int(rng.integers(R, 12))
        if (H + 2 * pad - R) % stride:
            continue
        G = [1, 1, 2][len(meta["conv"]) % 3]
        N = int(rng.integers(1, 4)); Cin = G * int(rng.integers(1, 5)); M = G * int(rng.integers(1, 5))
        bias = bool(rng.integers(0, 2))
        d = O.dims(N, Cin, H, M, R, stride, pad, G, bias)
        seeds = [1000 + 3 * k, 1001 + 3 * k, 1002 + 3 * k]
        D = rnd((N, Cin, H, H), seeds[0]); W = rnd((M, Cin // G, R, R), seeds[1])
        B = rnd((M,), seeds[2]) if bias else None
        Oref = O.ref_conv_f32(d, D, W, B)
        key = f"conv{k}"
        arrays[f"{key}_D"], arrays[f"{key}_W"], arrays[f"{key}_O"] = D, W, Oref
        if B is not None:
            arrays[f"{key}_B"] = B
        meta["conv"].append({"key": key, "dims": [N, Cin, H, M, R, stride, pad, G, int(bias)], "seeds": seeds})
        k += 1

    # ---- input/output checksums + summations at T=double (checksums.hpp:91-245)
    for k in range(4):
        N, Cin, H, M, R, pad = 3 + k, 2 + k, 7, 3 + k, 3, 1
        bias = k % 2 == 1
        d = O.dims(N, Cin, H, M, R, 1, pad, 1, bias)
        D = rnd((N, Cin, H, H), 5000 + k); W = rnd((M, Cin, R, R), 6000 + k)
        B = rnd((M,), 7000 + k) if bias else None
        Of = O.ref_conv_f32(d, D, W, B)
        co = O.ref_output_checksums(d, 127, D.astype(np.float64), W.astype(np.float64))
        so = O.ref_output_summations(Of.astype(np.float64), 127, None if B is None else B.astype(np.float64))
        key = f"ck{k}"
        arrays[f"{key}_D"], arrays[f"{key}_W"], arrays[f"{key}_O"] = D, W, Of
        if B is not None:
            arrays[f"{key}_B"] = B
        for f in range(7):
            arrays[f"{key}_co{f + 1}"] = co[f]
            arrays[f"{key}_so{f + 1}"] = so[f]
        meta["checksums"].append({"key": key, "dims": [N, Cin, H, M, R, 1, pad, 1, int(bias)]})

    # ---- run_protected_layer<double> with the post_conv substitution (workflow.hpp:141-339)
    for k in range(40):
        N = int(rng.integers(1, 6)); M = int(rng.integers(1, 6)); Cin = int(rng.integers(1, 5))
        R = int([1, 3][rng.integers(0, 2)]); H = int(rng.integers(R + 1, 10)); pad = int(rng.integers(0, 2))
        bias = bool(rng.integers(0, 2))
        d = O.dims(N, Cin, H, M, R, 1, pad, 1, bias)
        E = O.extent(d)
        D = rnd((N, Cin, H, H), 9000 + 3 * k); W = rnd((M, Cin, R, R), 9001 + 3 * k)
        B = rnd((M,), 9002 + 3 * k) if bias else None
        Of = O.ref_conv_f32(d, D, W, B)
        faults = []
        kind = k % 4
        for _ in range(1 if kind == 0 else int(rng.integers(1, 4))):
            n = int(rng.integers(0, N)); m = int(rng.integers(0, M))
            if kind == 2:
                n = faults[0][0] if faults else n
            if kind == 3:
                m = faults[0][1] if faults else m
            x, y = int(rng.integers(0, E)), int(rng.integers(0, E))
            bit = int(rng.integers(20, 31))
            if (n, m, x, y) in [(f[0], f[1], f[2], f[3]) for f in faults]:
                continue
            faults.append((n, m, x, y, bit))
            Of[n, m, x, y] = O.flip_f32(Of[n, m, x, y], bit)
        rc, clc = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        tau = float([1e-3, 1e-4, 1e-5][rng.integers(0, 3)])
        ref = O.ref_protected_layer(d, D, W, B, rc, clc, tau, O_conv=Of)
        key = f"vd{k}"
        arrays[f"{key}_D"], arrays[f"{key}_W"], arrays[f"{key}_O"] = D, W, Of
        if B is not None:
            arrays[f"{key}_B"] = B
        meta["verdicts"].append({
            "key": key, "dims": [N, Cin, H, M, R, 1, pad, 1, int(bias)], "rc": rc, "clc": clc, "tau": tau,
            "faults": faults, "status": ref["status"],
            "verdict": {k2: ref[k2] for k2 in ("detected", "stage", "weights_reloaded", "recomputed",
                                               "stages_attempted")}
                       | {"corrected_blocks": [list(b) for b in ref["corrected_blocks"]]},
        })
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "golden_v1.npz"), **arrays)
    with open(os.path.join(OUT, "golden_v1.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", OUT, len(arrays), "arrays")


if __name__ == "__main__":
    main()
