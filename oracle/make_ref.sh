#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: installs the UNMODIFIED reference package
# (/root/reference/pkg, pure Python + numpy) into oracle/_ref so bench.py's
# reference arm and CPU baseline can run the reference's own code on the GPU
# box's host cores (the reference tree does not exist there; oracle/_ref is
# git-ignored but travels with the gpurun snapshot).  Offline: no index, no
# dependency resolution (numpy is in the image).  The build writes into its
# source tree, so it runs from a copy under /tmp.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -f "$SRC/pyproject.toml" ]; then
    echo "make_ref.sh: no reference at $SRC (GPU box): keeping $OUT as shipped" >&2
    exit 0
fi
if [ -f "$OUT/devplace/__init__.py" ] && [ -z "$(find "$SRC/src" -newer "$OUT/devplace/__init__.py" -name '*.py' | head -1)" ]; then
    exit 0
fi
TMP="$(mktemp -d /tmp/devplace_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$OUT" "$TMP/pkg"
touch "$OUT/devplace/__init__.py"
