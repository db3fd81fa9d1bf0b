"""Shared test plumbing.

``-m "not gpu"`` runs the oracle-vs-golden, host-logic, selector and
C-ABI-loads checks on CPU; ``-m gpu`` runs the parity tests proper, which
call the CUDA path through the C-ABI and compare it with ``oracle/``.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on gpurun)")


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


def golden_names(prefix="ref_"):
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz")
                  if p.stem not in ("ref_swiglu",))


@pytest.fixture
def small_model():
    from paper_2601_08800_b200.config import ModelHyperparams
    return ModelHyperparams(hidden_dim=64, num_layers=4, top_k=2,
                            num_routed_experts=8, num_shared_experts=1,
                            psi_attn=1e6, psi_moe=8e6, psi_active=2e6)


@pytest.fixture
def small_cluster():
    from paper_2601_08800_b200.config import ClusterConfig
    return ClusterConfig(n_node=2, n_proc=2, intra_alpha=1e-6,
                         intra_beta=100e9, inter_alpha=2e-6, inter_beta=10e9,
                         mem_per_device=64e9, compute_rate=1e12)


@pytest.fixture
def small_workload():
    from paper_2601_08800_b200.config import WorkloadSpec
    return WorkloadSpec(batch_size=8, seq_len=128, input_len=128,
                        output_len=64, arrival_rate=10.0)


@pytest.fixture
def small_calib():
    from paper_2601_08800_b200.config import CalibrationCoefficients
    return CalibrationCoefficients(compute_coeff=1e-13)
