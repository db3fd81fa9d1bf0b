#!/usr/bin/env bash
# Installs the UNMODIFIED reference (moeplan, pure Python + numpy) into
# oracle/_ref for bench.py's reference arm and cpu_baseline (kind
# "reference": run_moe_block timed on the GPU box's host).  Test / baseline
# infrastructure only -- the product package never imports it.  oracle/_ref
# is git-ignored (no reference source enters the history) but not
# gpurun-ignored, so it travels to the GPU box.  /root/reference is
# read-only: the build runs from a copy under /tmp.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "install_ref: no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/moeplan_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import moeplan.simcluster as s
print("install_ref: moeplan from", s.__file__)
PY
