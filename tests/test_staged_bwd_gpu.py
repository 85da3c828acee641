"""The opt-in staged backward (MGAUSS_STAGED_BWD=1: TMA bulk copies of each
strip's point neighbourhood into shared memory under an mbarrier) must give
the same accumulators as the default item path.  The switch is read once per
process, so the staged run happens in a subprocess."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import load_golden
from test_render_gpu import Batch, field_of, transforms_of
from paper_2603_00145_b200.render import render_backward
from paper_2603_00145_b200.spatial import build
z = load_golden("render_lattice12")
f = field_of(z)
g = render_backward(f, build(f, int(z["g"]), 5), transforms_of(z), Batch(z["coords"], z["sids"]), z["upstream"])
np.savez(sys.argv[2], dp=g.d_positions, dq=g.d_quaternions, ds=g.d_log_scales, dl=g.d_intensity_logits)
"""


def _run(tmp_path, staged):
    out = tmp_path / f"g{int(staged)}.npz"
    env = dict(os.environ, MGAUSS_STAGED_BWD="1" if staged else "0")
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env, check=True, timeout=600)
    return np.load(out)


def test_staged_backward_matches_item_path(tmp_path):
    a, b = _run(tmp_path, False), _run(tmp_path, True)
    for k in ("dp", "dq", "ds", "dl"):
        np.testing.assert_allclose(b[k], a[k], rtol=1e-5, atol=1e-9 * np.abs(a[k]).max())
