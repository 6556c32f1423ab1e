"""The numpy oracle vs fixtures produced by the real reference (tests/golden/).

If these pass, the oracle restates the reference's arithmetic for every node
kind, fusion level and dtype the fixtures cover, and it can stand in for the
reference on the GPU box (where /root/reference does not exist).
"""

import glob
import os

import numpy as np
import pytest

from oracle import executor as OX
from oracle import ops as O
from paper_1807_01702_b200 import fusion
from paper_1807_01702_b200 import graph as G
from paper_1807_01702_b200.params import BNParams, ConvParams

from conftest import GOLDEN

EX = {
    "densenet-tiny-full": G.ModelSpec("densenet", (2, 2), 8, 4, (2, 3, 32, 32), "full",
                                      "conv7-pool", 16, name="densenet-tiny-full"),
    "resnet-tiny-strided": G.ModelSpec("resnet", (1, 1), input_dims=(2, 8, 8, 8), scale="micro",
                                       stem="conv3", base_channels=16,
                                       resnet_stages=((1, 4, 16, 1), (1, 8, 32, 2)),
                                       name="resnet-tiny-strided"),
}
SPECS = {
    "single-bn-toy": G.single_bn_toy(4), "densenet-micro": G.densenet_micro(2),
    "resnet-micro": G.resnet_micro(2), "gradcheck-micro": G.gradcheck_micro(2), **EX,
}


def rel_err(a, b, floor):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def scaled_err(a, b):
    """max |a-b| relative to the tensor's scale (summation-order noise is ~eps*scale)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def cases():
    out = []
    for fn in sorted(glob.glob(os.path.join(GOLDEN, "model_*.npz"))):
        stem = os.path.basename(fn)[6:-4]
        name, rest = None, None
        for n in SPECS:
            if stem.startswith(n + "_"):
                name, rest = n, stem[len(n) + 1:]
        lvl, tag = rest.rsplit("_", 1)
        out.append((name, lvl.replace("_", "+"), tag, fn))
    return out


@pytest.mark.parametrize("name,level,tag,fn", cases(), ids=lambda v: str(v)[-40:])
def test_oracle_matches_reference(name, level, tag, fn):
    ref = np.load(fn)
    dtype = np.float32 if tag == "f32" else np.float64
    g0 = G.build_model(SPECS[name], seed=0, dtype=dtype)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    res = OX.forward(g, {g.inputs[0]: ref["x"]})
    grads = OX.backward(g, res, {s: ref[f"dy_{s}"] for s in g.outputs})
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for s in g.outputs:
        assert scaled_err(res.vals[s], ref[f"out_{s}"]) < tol
    for key in ref.files:
        if key.startswith("grad::"):
            assert scaled_err(grads.params[key[6:]], ref[key]) < tol, key
        if key.startswith("dx_"):
            assert scaled_err(grads.inputs[int(key[3:])], ref[key]) < tol


def test_inputs_regenerate_bit_exactly():
    """Our Rng reproduces the reference's synthetic input and output-gradient draws."""
    from paper_1807_01702_b200.tensor import Rng
    ref = np.load(os.path.join(GOLDEN, "model_densenet-micro_bnff_f32.npz"))
    g = G.build_model(SPECS["densenet-micro"], seed=0)
    rng = Rng(1)
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
    dy = rng.normal(g.slots[g.outputs[0]].shape)
    assert np.array_equal(x, ref["x"]) and np.array_equal(dy, ref[f"dy_{g.outputs[0]}"])


@pytest.mark.parametrize("level", ["baseline", "bnff"])
def test_block_c1_digests(level):
    ref = np.load(os.path.join(GOLDEN, f"block_c1_{level}.npz"))
    g0 = G.build_block(8, 64, 32, seed=0)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    from paper_1807_01702_b200.tensor import Rng
    rng = Rng(1)
    x = rng.uniform((8, 64, 32, 32), -1.0, 1.0)
    dy = rng.normal((8, 64, 32, 32))
    assert float(x.astype(np.float64).sum()) == float(ref["x_sum"])
    res = OX.forward(g, {g.inputs[0]: x})
    grads = OX.backward(g, res, {g.outputs[0]: dy})
    out = res.vals[g.outputs[0]]
    dx = grads.inputs[g.inputs[0]]
    idx = ref["sample_idx"]
    assert scaled_err(out.reshape(-1)[idx], ref["out_sample"]) < 1e-5
    assert scaled_err(dx.reshape(-1)[idx], ref["dx_sample"]) < 1e-5
    assert scaled_err(out.astype(np.float64).sum((0, 2, 3)), ref["out_chsum"]) < 1e-5
    for key in ref.files:
        if key.startswith("grad::"):
            assert scaled_err(grads.params[key[6:]], ref[key]) < 1e-5, key


# ---------------------------------------------------------------------------
# frozen hand values quoted from the reference's own tests
# ---------------------------------------------------------------------------


def col(v, dtype=np.float32):
    return np.asarray(v, dtype).reshape(len(v), 1, 1, 1)


def test_bn_frozen_values():  # pkg/tests/test_ops.py:210-216
    x = col([1.0, 2.0, 3.0, 4.0])
    y = O.bn_apply(x, O.stats_twopass(x), BNParams(np.ones(1), np.zeros(1), eps=1e-12))
    assert np.allclose(y.reshape(-1), [-1.3416407865, -0.4472135955, 0.4472135955, 1.3416407865],
                       atol=1e-6)


def test_stats_hand_case():  # test_ops.py:146-151, 181-185
    st = O.stats_onepass(col([1.0, 2.0, 3.0, 4.0]))
    assert st.sum_x2[0] / st.count == pytest.approx(7.5)
    assert st.mean[0] == pytest.approx(2.5) and st.var[0] == pytest.approx(1.25)


def test_bn_bwd_constant_dy():  # test_ops.py:253-261
    x = col([1.0, 2.0, 3.0, 4.0])
    dx, dg, db = O.bn_bwd(x, np.full_like(x, 0.7), O.stats_twopass(x),
                          BNParams(np.ones(1), np.zeros(1)))
    assert db[0] == pytest.approx(2.8) and dg[0] == pytest.approx(0.0, abs=1e-9)
    assert np.allclose(dx, 0.0, atol=1e-6)


def test_relu_mask_golden():  # test_ops.py:301-304
    assert O.relu_fwd(col([-1.0, 0.0, 2.0])).reshape(-1).tolist() == [0.0, 0.0, 2.0]


def test_fused_gamma0_beta1_identity():  # test_fused_kernels.py:66-75
    x = np.random.default_rng(2).normal(size=(2, 3, 4, 4)).astype(np.float32)
    idc = ConvParams(3, 3, 1, 1, weights=np.eye(3, dtype=np.float32).reshape(3, 3, 1, 1))
    y, saved, _ = O.norm_relu_conv_fwd(x, O.stats_onepass(x), BNParams(np.zeros(3), np.ones(3)), idc)
    assert np.allclose(y, 1.0) and np.allclose(saved, 1.0)


def test_conv_integer_inputs_exact():  # test_ops.py:58-67 (bitwise on integer-valued data)
    rng = np.random.default_rng(3)
    x = rng.integers(-3, 4, size=(2, 3, 5, 5)).astype(np.float32)
    w = rng.integers(-2, 3, size=(4, 3, 3, 3)).astype(np.float32)
    p = ConvParams(3, 4, 3, 3, stride=2, pad=1, weights=w)
    y = O.conv_fwd(x, p)
    ref = np.zeros_like(y)
    for n in range(2):
        for o in range(4):
            for i in range(y.shape[2]):
                for j in range(y.shape[3]):
                    acc = 0.0
                    for c in range(3):
                        for a in range(3):
                            for b in range(3):
                                hh, ww = 2 * i - 1 + a, 2 * j - 1 + b
                                if 0 <= hh < 5 and 0 <= ww < 5:
                                    acc += x[n, c, hh, ww] * w[o, c, a, b]
                    ref[n, o, i, j] = acc
    assert np.array_equal(y, ref)
