"""Launch the SPMD parity check on every multi-GPU world the box offers, and
on one GPU with every rank a separate process on cuda:0.

The one-device form runs the SPMD layer's machinery -- per-process heaps
exchanged as CUDA IPC handles, peer stores and loads through those
mappings, the epoch-flag barrier protocol -- on any box with one GPU (gloo
bootstraps it).  Kernels of different processes are not guaranteed to run
side by side on one GPU, so there no rank spins on another's flag: every
device barrier is split into a publishing half and a checking half with a
host barrier between them (MoELayer.forward_stepped); graph replay, the
opt-in overlapped schedule and the NCCL arm run only with one GPU per rank."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(nproc, tp=None, env=None, port_off=0, same_device=False, extra=()):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={29500 + nproc * 7 + (tp or 0) + port_off}",
           str(ROOT / "tests" / "spmd_check.py")]
    if tp:
        cmd += ["--tp", str(tp)]
    if same_device:
        cmd += ["--same-device"]
    cmd += list(extra)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "OK" in r.stdout, r.stdout[-4000:]
    return r.stdout


@pytest.mark.parametrize("nproc,tp", [(2, 1), (2, 2), (4, 2), (4, 4), (8, 2), (8, 4)])
def test_spmd_layer_one_device(nproc, tp):
    """nproc ranks as processes on cuda:0: IPC heaps, split barriers, f64
    bit-exact / bf16 / fp8 parity, both wires, capacity errors on every rank
    (the 8-rank layouts are config B's TP2 x EP4 and config C's TP4 x EP2)."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    out = _run(nproc, tp, port_off=100, same_device=True)
    print(out[-2000:])


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


def test_spmd_bench_shape_one_device():
    """Config B at bench.py's dimensions in the EP2 layout bench.py runs at
    2 GPUs, as two processes on cuda:0: a 512-token sample of the output
    against the CPU oracle."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    out = _run(2, 1, port_off=130, same_device=True, extra=["--bench-shape"])
    assert "config B bench shape" in out
    print(out[-1500:])


@pytest.mark.parametrize("nproc,tp", [(2, 1), (4, 1), (4, 2)])
def test_spmd_bench_shape(nproc, tp):
    """Config B at bench.py's dimensions in the 2/4-GPU layouts, one rank per
    GPU (device barriers, NVLink)."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    out = _run(nproc, tp, port_off=160, extra=["--bench-shape"])
    assert "config B bench shape" in out
