#!/bin/bash
# Installs the UNMODIFIED reference package (/root/reference/pkg) into baseline/_ref with its
# own setup (Cython module included).  /root/reference is read-only, so the install runs
# from a copy under /tmp.  baseline/_ref is git-ignored but travels to the GPU box.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 0; }
TMP="$(mktemp -d /tmp/hsseig_ref.XXXXXX)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg" -q
rm -rf "$TMP"
PYTHONPATH="$HERE/_ref" python -c "import hsseig; print('reference installed, backend =', hsseig.BACKEND)"
