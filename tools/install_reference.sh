#!/usr/bin/env bash
# Install the UNMODIFIED reference package (matchbench) into baseline/_ref --
# the one offline install the task allows (no index; numpy is already in the
# image, so dependency resolution is skipped with --no-deps).  The build copies
# the read-only source tree to /tmp first.  baseline/_ref is git-ignored but
# travels to the GPU box with the repo snapshot; only tests/test_gpu_harness.py
# imports it (the reference's own callers driving the B200 descriptor).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC: keeping $ROOT/baseline/_ref as is"; exit 0; }
[ -f "$ROOT/baseline/_ref/matchbench/__init__.py" ] && exit 0
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "installed matchbench into $ROOT/baseline/_ref"
