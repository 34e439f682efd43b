"""The KO_DEBUG build (lib/libko_debug.so, same ABI compiled with -DKO_DEBUG; include/ko.h
"device-data errors"): on valid data it returns the release build's margins bit for bit; a page
id outside the pool, a seq_len < 1 or a bad source page of the cache builder traps the kernel
(the process sees a CUDA error) after printing which check failed.  Each case runs in its own
process because a trap poisons the CUDA context."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2602_04430_b200", "lib", "libko_debug.so")


def _probe(mode, out, debug=True):
    env = dict(os.environ)
    if debug:
        env["KO_LIB"] = DEBUG_LIB
    else:
        env.pop("KO_LIB", None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_probe.py"), mode,
                           str(out)], env=env, capture_output=True, text=True, timeout=240,
                          cwd=ROOT)


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    assert os.path.exists(DEBUG_LIB), "build it with __graft_entry__.build()"


def test_debug_build_matches_release_on_valid_data(gpu, tmp_path):
    r = _probe("ok", tmp_path / "dbg.npy")
    assert r.returncode == 0 and "libko_debug.so" in r.stdout, r.stderr[-2000:]
    r2 = _probe("ok", tmp_path / "rel.npy", debug=False)
    assert r2.returncode == 0, r2.stderr[-2000:]
    assert np.array_equal(np.load(tmp_path / "dbg.npy"), np.load(tmp_path / "rel.npy"))


@pytest.mark.parametrize("mode,check", [("bad_page", "p.n_pages"), ("bad_len", "L >= 1"),
                                        ("bad_build", "p.n_pages")])
def test_debug_build_traps_bad_device_data(gpu, tmp_path, mode, check):
    r = _probe(mode, tmp_path / "x.npy")
    text = r.stdout + r.stderr
    assert r.returncode != 0 and "PROBE_DONE" not in r.stdout, text[-2000:]
    assert "KO_DEBUG check failed" in text and check in text, text[-2000:]
