"""Launch the SPMD parity check on every multi-GPU world the box offers."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(nproc, tp=None, env=None, port_off=0):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={29500 + nproc * 7 + (tp or 0) + port_off}",
           str(ROOT / "tests" / "spmd_check.py")]
    if tp:
        cmd += ["--tp", str(tp)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.parametrize("nproc,tp", [(2, 1), (2, 2), (4, 2), (4, 4), (8, 2), (8, 4)])
def test_spmd_layer(nproc, tp):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _run(nproc, tp)


@pytest.mark.parametrize("nproc,tp", [(2, 1), (4, 2)])
def test_spmd_layer_fused_barriers(nproc, tp):
    """The opt-in in-kernel barriers (MX_FUSE_BARRIER_T) on the same checks."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _run(nproc, tp, env={"MX_FUSE_BARRIER_T": "4096"}, port_off=50)
