#!/bin/bash
# Build libaxq.so of git revision $1 (default HEAD) into paper_2203_04071_b200/libaxq_base.so,
# for same-box A/B timing (AXQ_LIB=... python bench.py).  The working tree is not touched.
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" | tar -x -C "$TMP"
python -c "
import importlib.util, sys
spec=importlib.util.spec_from_file_location('b','$TMP/paper_2203_04071_b200/build.py'); m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build()"
cp "$TMP/paper_2203_04071_b200/libaxq.so" "$ROOT/paper_2203_04071_b200/libaxq_base.so"
rm -rf "$TMP"
echo "built $REV -> paper_2203_04071_b200/libaxq_base.so"
