"""Grid mode's tuple finaliser runs as its own launch (grid_final_kernel) after the scoring
kernel (DESIGN.md §4 "Finaliser").  Pin it to the in-kernel finaliser it replaced
(KO_GRID_FIN_KERNEL=0): the same fixed-order fp64 sums and plan walks, so margins, classes and
every count must be bit-identical, and the launch count differs by exactly the one finaliser."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, fin):
    env = dict(os.environ)
    env["KO_GRID_FIN_KERNEL"] = str(fin)
    out = tmp_path / f"fin{fin}.npz"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "grid_final_probe.py"),
                        str(out)], env=env, capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_finaliser_launch_matches_in_kernel_finaliser(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    a, b = _run(tmp_path, 1), _run(tmp_path, 0)
    for cfg in ("C5", "C3"):
        ma, mb = a[cfg + "_m"], b[cfg + "_m"]
        assert np.array_equal(ma.view(np.uint32), mb.view(np.uint32))   # bitwise margins
        assert np.array_equal(a[cfg + "_c"], b[cfg + "_c"])
        assert np.array_equal(a[cfg + "_counts"], b[cfg + "_counts"])
        assert a[cfg + "_counts"].sum() > 0
        assert int(a[cfg + "_launches"][0]) == int(b[cfg + "_launches"][0]) + 1
