"""Multi-GPU landmark sharding on real GPUs: two processes (torchrun), one
per GPU, NCCL all-reduces inside librba; LM costs against the oracle and the lockstep checksums
(tests/_mp_lm.py).  Skipped when fewer than 2 GPUs are visible (this run's GPU boxes have one:
tests/test_gpu_parity.py::test_lm_with_one_rank_nccl runs the same NCCL code path with a one-rank
communicator, and the world-size-2 partition / reduction structure is covered on CPU by
tests/test_dist_gloo.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_rank_lm_parity_and_lockstep():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29511", os.path.join(HERE, "_mp_lm.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert r.stdout.count("MP_OK") == 2
