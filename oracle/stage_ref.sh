#!/bin/sh
# Stage the UNMODIFIED reference package (stalesync 0.1.0, pure Python +
# numpy) into oracle/_ref/ for bench.py's reference arm and cpu_baseline leg.
# Runs only where /root/reference exists (the build container); the staged
# copy is git-ignored but travels to the GPU box with the gpurun snapshot.
# pip builds from a copy under /tmp because /root/reference is read-only;
# --no-deps: numpy is already in the image.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "stage_ref: $SRC absent, keeping any existing oracle/_ref"; exit 0; }
TMP=$(mktemp -d /tmp/stalesync_src.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP" 2>&1 | grep -v "^$" || true
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import stalesync; print('stage_ref: stalesync', stalesync.__file__)"
