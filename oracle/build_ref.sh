#!/usr/bin/env bash
# Install the UNMODIFIED reference package (sweepjoin, Python + its Cython
# compiled backend) into baseline/_ref — the one offline install the bench
# contract allows.  Run in the build container, where /root/reference exists;
# baseline/_ref is git-ignored but travels to the GPU box with the snapshot, so
# bench.py's cpu_baseline leg can time the reference's own join() there.
#
# The reference's build writes into its source tree (Cython .cpp, build/), and
# /root/reference is read-only: build from a scratch copy under /tmp.  Only
# dependency resolution fails offline (numpy is already installed), hence
# --no-deps.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
DEST="$ROOT/baseline/_ref"
[ -d "$SRC" ] || { echo "reference sources not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/sweepjoin_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DEST"
cd "$TMP"
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$DEST" "$TMP/pkg" >"$TMP/pip.log" 2>&1 ||
  { cat "$TMP/pip.log" >&2; exit 1; }
PYTHONPATH="$DEST" python -c "import sweepjoin; b = sweepjoin.available_backends(); \
assert 'compiled' in b, b; print('reference installed:', sweepjoin.__file__, b)"
