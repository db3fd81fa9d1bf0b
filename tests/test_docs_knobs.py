"""Every runtime knob the native library reads (getenv("MX_...") in csrc/)
is documented in INTEGRATION.md's table -- the documentation cannot drift
from the code."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_every_env_knob_is_documented():
    src = "".join(p.read_text() for p in (ROOT / "paper_2601_08800_b200" / "csrc").glob("*.cu*"))
    knobs = set(re.findall(r'getenv\("(MX_[A-Z0-9_]+)"\)', src))
    assert knobs, "no knobs found (pattern drifted?)"
    doc = (ROOT / "INTEGRATION.md").read_text()
    missing = sorted(k for k in knobs if f"`{k}" not in doc)
    assert not missing, f"undocumented knobs in INTEGRATION.md: {missing}"
