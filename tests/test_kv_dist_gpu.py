"""Multi-GPU KVStore (one process per GPU, CUDA IPC + in-kernel barrier):
bitwise rounds vs the reference's golden rounds, config-1 training parity,
captured-step determinism.  Skipped on a single-GPU host."""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_distributed_kvstore(cuda, tmp_path, nproc):
    if cuda.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, DIST_RESULT_DIR=str(tmp_path), PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "dist_worker.py")]
    proc = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    for r in range(nproc):
        assert (tmp_path / f"rank{r}.txt").read_text() == "OK", r
