"""Generate tests/golden/model_io/ from the reference itself (oracle/_ref): the FTCN
weight file random_weights + save_weights writes for the toy config of
test_model_io.cpp at seed 42, and report_to_json of a fixed set of layer reports (plain
and as a campaign).  Run in the build container (needs /root/reference); the outputs
are committed so the CPU tests pin the formats without the reference."""
import json
import os
import sys
from types import SimpleNamespace as NS

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_py as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "model_io")
TOY = """{
  "name": "toy",
  "element_type": "f32",
  "layers": [
    {"name": "c1", "batch": 2, "channels": 3, "height": 8, "kernels": 4, "kernel_size": 3},
    {"name": "c2", "batch": 2, "channels": 4, "height": 6, "kernels": 2, "kernel_size": 3, "bias": true}
  ]
}"""
REPORTS = [
    NS(layer="c1", detected=False, stage="none", weights_reloaded=False, recomputed=False, corrected_blocks=[],
       stages_attempted=[], timings={"total": 0.00125}),
    NS(layer="c2", detected=True, stage="coc", weights_reloaded=False, recomputed=False, corrected_blocks=[(1, 3)],
       stages_attempted=["coc"], timings={"total": 1.5e-05, "detect": 3.0}),
    NS(layer="conv_3", detected=True, stage="recompute", weights_reloaded=True, recomputed=True,
       corrected_blocks=[(0, 0), (5, 17)], stages_attempted=["coc", "rc", "clc", "fc", "recompute"],
       timings={"total": 123.25}),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "toy_config.json"), "w") as f:
        f.write(TOY)
    assert O.ref_make_weights(TOY, 42, os.path.join(OUT, "toy_seed42.ftcn")) == 0
    with open(os.path.join(OUT, "report.json"), "w") as f:
        f.write(O.ref_report_to_json(REPORTS, timings=False))
    with open(os.path.join(OUT, "report_timings.json"), "w") as f:
        f.write(O.ref_report_to_json(REPORTS, timings=True))
    with open(os.path.join(OUT, "campaign_report.json"), "w") as f:
        f.write(O.ref_report_to_json(REPORTS, timings=False, campaign=(3, 2, 2, 1, 1, 0)))
    with open(os.path.join(OUT, "reports.json"), "w") as f:
        json.dump([vars(r) for r in REPORTS], f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
