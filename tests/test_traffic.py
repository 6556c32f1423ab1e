"""The sweep rulebook (traffic.py) pinned to the REAL reference's count_sweeps
(traffic.py:128-231), via tests/golden/traffic.json written by
tests/golden/make_traffic_golden.py: totals per pass, weight bytes and bytes per node kind
for DenseNet-121 b64, ResNet-50 b128, DenseNet-BC-100 b64 and the micro presets at all five
fusion levels, with the reference's own Concat mode and with Concat held at view mode, plus
every (node, pass, slot, direction) sweep count on the micro graphs."""

import json
import os

import pytest

from paper_1807_01702_b200 import fusion, graph as G, traffic

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traffic.json")
MODELS = {
    "densenet-121-b64": lambda: G.densenet121(64),
    "resnet-50-b128": lambda: G.resnet50(128),
    "densenet-bc-100-b64": lambda: G.densenet_bc100(64),
    "densenet-micro-b2": lambda: G.densenet_micro(2),
    "resnet-micro-b2": lambda: G.resnet_micro(2),
}
LEVELS = ["baseline", "rcf", "rcf+mvf", "bnff", "bnff+icf"]


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.mark.parametrize("model", list(MODELS))
def test_rulebook_matches_reference(golden, model):
    g0 = G.build_model(MODELS[model](), seed=0)
    for lv in LEVELS:
        g, _ = fusion.plan(g0, fusion.parse_level(lv))
        for phys, tag in ((None, "own"), (False, "view")):
            want = golden[f"{model}/{lv}/{tag}"]
            led = traffic.count_sweeps(g, concat_physical=phys)
            assert led.total_bytes() == want["total"], (lv, tag)
            assert led.total_bytes("forward") == want["forward"]
            assert led.total_bytes("backward") == want["backward"]
            assert led.weight_bytes() == want["weights"]
            assert led.bytes_by_kind() == want["by_kind"]
            if "sweeps" in want:
                got = sorted([list(k) + [v] for k, v in led.key_map().items()])
                assert got == want["sweeps"]


def test_densenet121_headline_reduction(golden):
    """81.00 GB baseline -> 30.61 GB bnff+icf per b64 iteration (fp32)."""
    g0 = G.build_model(G.densenet121(64), seed=0)
    base = traffic.count_sweeps(fusion.plan(g0, fusion.parse_level("baseline"))[0], False)
    icf = traffic.count_sweeps(fusion.plan(g0, fusion.parse_level("bnff+icf"))[0], False)
    s = traffic.summary(icf, "bnff+icf", "densenet-121", base)
    assert round(base.total_bytes() / 1e9, 2) == 81.0 and round(icf.total_bytes() / 1e9, 2) == 30.61
    assert 0.62 < s["reduction_vs_baseline"] < 0.63
    assert traffic.to_csv(icf).splitlines()[0] == ",".join(traffic.CSV_HEADER)


def test_cli_traffic_and_explain(tmp_path, capsys):
    from paper_1807_01702_b200 import cli
    assert cli.main(["traffic", "--model", "densenet-121", "--batch", "64", "--out", str(tmp_path)]) == 0
    summ = json.load(open(tmp_path / "summary.json"))
    by = {s["level"]: s for s in summ}
    assert round(by["baseline"]["total_bytes"] / 1e9, 2) == 81.0
    assert round(by["bnff+icf"]["total_bytes"] / 1e9, 2) == 30.61
    assert (tmp_path / "traffic_bnff_icf.csv").read_text().startswith("node_id,kind,pass,reads,writes,bytes")
    assert cli.main(["explain", "--model", "densenet-micro", "--fusion", "bnff+icf"]) == 0
    assert "fusion level: bnff+icf" in capsys.readouterr().out
