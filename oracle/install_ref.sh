#!/bin/sh
# Install the Python reference (bitquorum, pure stdlib) into oracle/_ref/ so the
# GPU box -- where /root/reference does not exist -- can run the reference's own
# harness (bench/competitions.run_competitions) and algorithms against the GPU
# path.  Test infrastructure only; oracle/_ref/ is git-ignored and travels with
# the gpurun snapshot.  Installs from a copy (the source tree is read-only) with
# no network and no dependencies (matplotlib only serves bench/report.py).
set -e
SRC=${BQ_REFERENCE_PKG:-/root/reference/pkg}
HERE=$(cd "$(dirname "$0")" && pwd)
[ -d "$SRC" ] || { echo "install_ref: $SRC not present, skipped"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg" -q
rm -rf "$TMP"
echo "install_ref: bitquorum installed into $HERE/_ref"
