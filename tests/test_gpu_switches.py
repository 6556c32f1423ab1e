"""The library's A/B switches select code paths that stay reachable in
production.  The switches are read once per process, so each configuration runs in a
subprocess: the window-vs-generic kernel check of tools/bench_conv.py and the ICF fold /
stem / padded-model parity tests of test_gpu_parity.py."""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SWITCHES = [
    {"BNFF_WRES1": "0"},
    {"BNFF_PDL": "0", "BNFF_FUSE_FINALIZE": "0", "BNFF_FUSE_NRP": "0"},
]


def _env(extra):
    env = dict(os.environ)
    env.update(extra)
    return env


@pytest.mark.gpu
@pytest.mark.parametrize("switch", SWITCHES, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
def test_window_kernels_under_switch(switch):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_conv.py"), "--quick", "--reps", "1"],
                         cwd=ROOT, env=_env(switch), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    m = re.search(r"worst rel-L2 window vs generic: ([0-9.e+-]+)", out.stdout)
    assert m, out.stdout[-2000:]
    assert float(m.group(1)) < 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("switch", SWITCHES, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
def test_parity_under_switch(switch):
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                          "-k", "icf_block_gradient_fold or stem_im2col or padded_growth12"],
                         cwd=ROOT, env=_env(switch), capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout
