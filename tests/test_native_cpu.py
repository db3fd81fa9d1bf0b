"""CPU-side checks of the boundary and host logic (no GPU compute)."""
import ctypes as C
import json
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_names, load_golden
from oracle import mixserve_oracle as orc
from paper_2601_08800_b200 import _native as N
from paper_2601_08800_b200.errors import CapacityError, StrategyError
from paper_2601_08800_b200.trace import TraceBuilder, trace_from_csv, trace_to_csv

HEADER = ROOT / "include" / "mixserve_b200.h"


def header_symbols():
    return re.findall(r"^MX_API\s+(?:int|const char\*)\s+(mx_\w+)\(",
                      HEADER.read_text(), flags=re.M)


def test_library_loads_and_exports_every_header_symbol():
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/ but not exported"
        assert s in N.SIGNATURES or s == "mx_last_error"
    assert lib.mx_abi_version() == 3


def test_plan_heap_bytes_and_validation_map_to_reference_errors():
    lib = N.load()
    d = N.PlanDesc(4, 2, 2048, 2048, 128, 8, 768, N.MX_BF16,
                   N.MX_EXPERT_SWIGLU, 1, N.MX_WIRE_SLOT, 0, 0)
    out = C.c_size_t()
    N.check(lib.mx_plan_heap_bytes(C.byref(d), C.byref(out)))
    # worst-case capacity: T*n*min(k, E/n) rows of h bf16, twice (recv+partial)
    assert out.value > 2 * 2048 * 4 * 8 * 2048 * 2
    bad = N.PlanDesc(0, 2, 8, 8, 8, 2, 0, N.MX_F64, 0, 1, 0, 0, 0)
    with pytest.raises(StrategyError, match="at least one node"):
        N.check(lib.mx_plan_heap_bytes(C.byref(bad), C.byref(out)))
    bad = N.PlanDesc(2, 2, 8, 8, 8, 9, 0, N.MX_F64, 0, 1, 0, 0, 0)
    with pytest.raises(StrategyError, match="top_k"):
        N.check(lib.mx_plan_heap_bytes(C.byref(bad), C.byref(out)))


def test_error_code_mapping():
    with pytest.raises(CapacityError):
        N.check(N.MX_ERR_CAPACITY)
    with pytest.raises(N.NativeLibraryError):
        N.check(N.MX_ERR_CUDA)


@pytest.mark.parametrize("name", golden_names())
def test_host_trace_builder_matches_reference_bytes(name):
    """The trace is host logic fed by the GPU's counts; pin it to the
    reference's frozen fused and baseline traces."""
    g = load_golden(name)
    mt = json.loads(str(g["meta"]))
    n, m, h, E = mt["n"], mt["m"], mt["h"], mt["E"]
    T = mt["tokens"] // n
    tab = orc.Table(g["ids"], g["weights"], n, T, E)
    rows = [tab.expert_rows(d) for d in range(n)]
    tb = TraceBuilder(n, m, T, h, tab.send_counts())
    tb.dispatch()
    tb.combine(tb.expert(rows, tb.expert_deps()))
    assert trace_to_csv(tb.trace.events) == str(g["trace_csv"])
    tb = TraceBuilder(n, m, T, h, tab.send_counts())
    tb.baseline(rows)
    assert trace_to_csv(tb.trace.events) == str(g["trace_baseline_csv"])


def test_trace_csv_round_trip_and_bad_line():
    text = (GOLDEN / "trace_2x2.csv").read_text()
    assert trace_to_csv(trace_from_csv(text)) == text
    bad = ("event_id,rank,op,peer_or_group,bytes,round,dep_ids,scope,group_size,work\n"
           "0,0,route,local,oops,0,,compute,1,0.0\n")
    with pytest.raises(ValueError, match="line 2"):
        trace_from_csv(bad)


def test_router_validation_matches_reference():
    """RouterSpec rejects duplicate and out-of-range ids like the reference
    (sim:153-162; T/test_simcluster.py:93-98)."""
    from paper_2601_08800_b200 import RouterSpec
    with pytest.raises(ValueError, match="duplicate"):
        RouterSpec(4, ((0, 0),), ((0.5, 0.5),))
    with pytest.raises(ValueError, match="out of range"):
        RouterSpec(2, ((0, 2),), ((0.5, 0.5),))


def test_malformed_trace_row_names_its_line():
    """trace_from_csv names the offending line (T/test_simcluster.py:264-268)."""
    from paper_2601_08800_b200.trace import trace_from_csv
    text = ("event_id,rank,op,peer_or_group,bytes,round,dep_ids,scope,group_size,work\n"
            "0,0,route,local,oops,0,,compute,1,0.0\n")
    with pytest.raises(ValueError, match="line 2"):
        trace_from_csv(text)


def test_nvlink_diagnostic_kernels_build_for_sm100a():
    """tools/nvlink_push.cu (the NVLink ceiling bench's kernels) stays
    buildable for sm_100a; nvcc cross-compiles without a GPU."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    out = ROOT / "paper_2601_08800_b200" / "csrc" / "build" / "nvlink_push_check.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run([nvcc, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", str(ROOT / "tools" / "nvlink_push.cu"), "-o", str(out)],
                   check=True, capture_output=True)
    lib = C.CDLL(str(out))
    assert hasattr(lib, "nb_launch") and hasattr(lib, "nb_enable_peers")


def test_plan_input_validation_messages():
    """LayerPlan._on_device / _routing_inputs reject what the C ABI would
    misread (shape, dtype of hidden states, both or neither routing input)
    with StrategyError -- checked without a GPU through a stand-in plan."""
    import pytest
    import torch
    from paper_2601_08800_b200.errors import StrategyError
    from paper_2601_08800_b200.plan import LayerPlan

    p = LayerPlan.__new__(LayerPlan)
    p.emulate, p.n, p.tokens, p.hidden, p.num_experts, p.top_k = False, 1, 4, 8, 16, 2
    p.dtype, p.wdtype, p.device = torch.bfloat16, torch.float32, torch.device("cpu")
    x = torch.zeros(4, 8, dtype=torch.bfloat16)
    assert p._on_device(x, "x", torch.bfloat16, 8, False) is not None
    with pytest.raises(StrategyError, match="shape"):
        p._on_device(torch.zeros(3, 8, dtype=torch.bfloat16), "x", torch.bfloat16, 8, False)
    with pytest.raises(StrategyError, match="dtype"):
        p._on_device(x.float(), "x", torch.bfloat16, 8, False)
    ids = torch.zeros(4, 2, dtype=torch.int64)          # torch.topk indices
    assert p._on_device(ids, "ids", torch.int32, 2, True).dtype == torch.int32
    with pytest.raises(StrategyError, match="exactly one"):
        p._routing_inputs(None, None, None)
    with pytest.raises(StrategyError, match="weights"):
        p._routing_inputs(None, ids, None)
