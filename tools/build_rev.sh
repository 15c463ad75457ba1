#!/bin/bash
# Build libgomix_b200.so from git revision REV into
# paper_2203_08680_b200/libgomix_b200_NAME.so (A/B timing against the
# working tree with tools/ab.py; the ctypes signatures are the working tree's).
#   bash tools/build_rev.sh REV NAME [-DMACRO ...]
set -e
REV=$1; NAME=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d /tmp/gomix_rev_XXXX)
git -C "$ROOT" archive "$REV" paper_2203_08680_b200 include | tar -x -C "$TMP"
cp "$ROOT/paper_2203_08680_b200/build.py" "$TMP/paper_2203_08680_b200/build.py"
(cd "$TMP" && python -m paper_2203_08680_b200.build --variant "$NAME" "$@" > /dev/null)
cp "$TMP/paper_2203_08680_b200/libgomix_b200_$NAME.so" "$ROOT/paper_2203_08680_b200/"
rm -rf "$TMP"
echo "$ROOT/paper_2203_08680_b200/libgomix_b200_$NAME.so"
