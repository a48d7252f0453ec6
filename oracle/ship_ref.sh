#!/usr/bin/env bash
# Install the UNMODIFIED reference package (boxtune, /root/reference/pkg) into oracle/_ref/ so it
# travels to the GPU box with the repo snapshot (git-ignored, not gpurun-ignored).  Test
# infrastructure only: tests/, smoke() and bench.py's reference / cpu_baseline leg import it as the
# checker and the CPU baseline; the product package never does.
#
# The source tree is read-only, so pip builds from a copy under /tmp.  Falls back to a plain copy of
# the pure-Python package when pip cannot build (no network is needed either way: --no-index).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${1:-/root/reference/pkg}"
DEST="$HERE/_ref"
[ -d "$SRC/src/boxtune" ] || { echo "ship_ref: $SRC/src/boxtune not found" >&2; exit 1; }
TMP="$(mktemp -d /tmp/boxtune_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC/." "$TMP/"
rm -rf "$DEST.new"
if python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$DEST.new" "$TMP" \
        >/dev/null 2>&1 && [ -f "$DEST.new/boxtune/__init__.py" ]; then
    how="pip install --target"
else
    rm -rf "$DEST.new"; mkdir -p "$DEST.new"; cp -r "$SRC/src/boxtune" "$DEST.new/boxtune"
    how="copy of src/boxtune"
fi
find "$DEST.new" -name __pycache__ -prune -exec rm -rf {} +
rm -rf "$DEST"; mv "$DEST.new" "$DEST"
echo "ship_ref: reference installed into $DEST ($how)"
