"""The multi-GPU code path of bench.py on one GPU: torchrun launches a rank that initialises an
NCCL process group, all-reduces the int64 count vector and takes the max of the device times
(KO_FORCE_DIST=1 keeps the distributed path at world size 1)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_nccl_path_single_rank():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, KO_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--config", "C1", "--steps", "3", "--warmup", "3", "--no-e2e",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    out = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(out) == 1, out[:5]                        # stdout = exactly the one JSON line
    line = json.loads(out[0])
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert "NCCL INFO" in r.stderr and "nRanks 1" in r.stderr and "rank 0 of 1" in r.stderr
    assert line["counts_plan0"][3] > 0                   # counts survived the all-reduce


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_bench_two_ranks_one_gpu(cfg, tmp_path):
    """bench.py's N > 1 path end to end with 2 ranks sharing one GPU (gloo carries the count
    all-reduce and the max over ranks; on the 8-GPU box it is NCCL): byte-balanced shards (C3) or
    equal shards (C4), the sum of both ranks' tuples in `value`, counts combined."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, KO_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", cfg, "--n-tuples", "300", "--steps", "3", "--warmup", "3",
           "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd + ["--dump-counts", str(tmp_path / "two.npy")], env=env,
                       capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["value"] == pytest.approx(2 * 300 * 3 / (line["ms_per_step"] * 3 / 1000.0))
    assert line["counts_plan0"][3] > 0
    assert "rank 1 of 2" in r.stderr                        # both ranks joined the group
    # the combined counts of the 2 shards equal ONE rank's pass over the same 2·300 tuples
    one = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config", cfg,
           "--n-tuples", "600", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
           "--dump-counts", str(tmp_path / "one.npy")]
    r1 = subprocess.run(one, capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert r1.returncode == 0, r1.stderr[-3000:]
    two, single = np.load(tmp_path / "two.npy"), np.load(tmp_path / "one.npy")
    assert single[:, 3].sum() > 0
    assert np.array_equal(two, single)
