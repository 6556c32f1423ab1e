"""Pin the sweep rulebook: the REAL reference's count_sweeps (traffic.py:128-231) on the
benched and micro graphs at every fusion level (run in the build container, reads
/root/reference read-only; only the JSON it writes travels).

    python tests/golden/make_traffic_golden.py   ->  tests/golden/traffic.json
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from bnfuse import fusion, traffic  # noqa: E402
from bnfuse import graph as RG  # noqa: E402

LEVELS = ["baseline", "rcf", "rcf+mvf", "bnff", "bnff+icf"]
MODELS = {
    "densenet-121-b64": lambda: RG.densenet121(64),
    "resnet-50-b128": lambda: RG.resnet50(128),
    "densenet-bc-100-b64": lambda: RG.ModelSpec("densenet", (16, 16, 16), 12, 4, (64, 24, 32, 32), "micro",
                                                "conv3", name="densenet-bc-100"),
    "densenet-micro-b2": lambda: RG.densenet_micro(2),
    "resnet-micro-b2": lambda: RG.resnet_micro(2),
}


def main():
    out = {}
    for name, spec in MODELS.items():
        g0 = RG.build_model(spec(), seed=0)
        for lv in LEVELS:
            g, _ = fusion.plan(g0, fusion.parse_level(lv))
            for phys in (None, False):
                led = traffic.count_sweeps(g, concat_physical=phys)
                key = f"{name}/{lv}/{'own' if phys is None else 'view'}"
                entry = {"total": led.total_bytes(), "forward": led.total_bytes("forward"),
                         "backward": led.total_bytes("backward"), "weights": led.weight_bytes(),
                         "by_kind": led.bytes_by_kind()}
                if name.endswith("micro-b2"):  # node-level pin on the small graphs
                    entry["sweeps"] = sorted([list(k) + [v] for k, v in led.key_map().items()])
                out[key] = entry
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"wrote {len(out)} ledgers")


if __name__ == "__main__":
    main()
