#!/usr/bin/env bash
# Install the reference package (pure Python, stdlib only) from its sources
# under /root/reference into oracle/_ref/ so the CPU baseline arm of bench.py
# can run the reference's own simulate() on the GPU box.  oracle/_ref/ is
# git-ignored (never committed) but travels with the gpurun snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
DEST="$HERE/_ref"
if [ ! -d "$SRC" ]; then echo "reference not present; keeping $DEST as is"; exit 0; fi
if [ -f "$DEST/memshare/harness.py" ]; then exit 0; fi
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DEST" "$TMP/pkg"
rm -rf "$TMP"
echo "installed reference into $DEST"
