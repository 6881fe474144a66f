"""Generate tests/golden/campaign_v1.json from the REFERENCE's campaign() (fault.hpp:195-271).

TEST INFRASTRUCTURE.  Needs oracle/_ref (built from /root/reference); the committed
fixture pins the library's corpus generator where the reference is absent.
    python oracle/gen_golden_campaign.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_py as O  # noqa: E402

CASES = [
    {"grids": [[4, 6, 3, 9, 3], [4, 5, 6, 7, 3]], "n_runs": 60, "weights": [1, 1, 1, 1, 1, 1], "seed": 7},
    {"grids": [[1, 3, 2, 8, 3]], "n_runs": 40, "weights": [1, 0, 2, 1, 1, 3], "seed": 12345},
    {"grids": [[6, 1, 4, 10, 5], [2, 8, 8, 6, 1], [3, 3, 3, 5, 3]], "n_runs": 50, "weights": [0.5, 1, 1, 2, 0, 1],
     "seed": 2**63 + 99},
]


def main():
    if not O.have_ref():
        raise SystemExit("reference bridge unavailable: needs /root/reference")
    out = {"generator": "oracle/gen_golden_campaign.py", "cases": []}
    for c in CASES:
        corpus = O.ref_campaign(c["grids"], c["n_runs"], c["weights"], c["seed"])
        out["cases"].append(dict(c, corpus=[{"spec": s, "truth": t} for s, t in corpus]))
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", "campaign_v1.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path)


if __name__ == "__main__":
    main()
