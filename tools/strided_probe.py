"""bf16 stride-2 micro-ResNet: per-tensor error vs the fp64 oracle with the patch-matrix path on/off"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
from test_gpu_parity import err, run_both  # noqa: E402
from test_gpu_strided import _strided_resnet  # noqa: E402

for dt in ("bf16", "f32"):
    for on in ("1", "0"):
        os.environ["BNFF_COL_STRIDED"] = on
        g, eng, res, ref = run_both(_strided_resnet(), "bnff+icf", dt)
        grads = eng.param_grads()
        errs = {k: err(grads[k], v, dt) for k, v in ref.params.items() if not k.endswith(".bias")}
        worst = sorted(errs.items(), key=lambda kv: -kv[1])[:6]
        print(dt, "col", on, "out", f"{err(eng.output(), res.vals[g.outputs[0]], dt):.2e}",
              "dx", f"{err(eng.input_grad_nchw(), ref.inputs[g.inputs[0]], dt):.2e}",
              " ".join(f"{k}={v:.2e}" for k, v in worst), flush=True)
