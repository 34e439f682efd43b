"""NVTX ranges of the C-ABI (SURVEY §5 tracing): every compute entry point pushes a range named
after itself, so ncu's NVTX filter sees the library's kernels inside it — and nothing else."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys; sys.path.insert(0, %r)
import torch, paper_2602_04430_b200 as ko
x = torch.randn(4096, 128, device="cuda").bfloat16()
q = torch.randn(2, 128, device="cuda").bfloat16()
m = torch.empty((2, 1, 4096), device="cuda")
torch.zeros(16, device="cuda").add_(1)          # a kernel outside any ko_* range
ko.embed_scores(x, q, [0, 1], m, variant=0)
torch.cuda.synchronize()
""" % ROOT


def test_ncu_nvtx_filter_sees_library_range(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        pytest.skip("ncu not installed")
    script = tmp_path / "nvtx_probe.py"
    script.write_text(SCRIPT)
    r = subprocess.run([ncu, "--nvtx", "--nvtx-include", "ko_embed_scores/", "--metrics",
                        "gpu__time_duration.sum", "--csv", sys.executable, str(script)],
                       capture_output=True, text=True, timeout=240)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-2000:]
    assert "embed_mma_kernel" in out, out[-2000:]          # the library kernel inside the range
    assert "vectorized_elementwise" not in out, out[-2000:]  # torch's kernel outside it is filtered
