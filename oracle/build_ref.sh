#!/usr/bin/env bash
# Test infrastructure only (the checker, never the product).
# Builds the UNMODIFIED reference (deltaserve, /root/reference/pkg) including its
# Cython kernel (_kernels/_native.pyx) into oracle/_ref/ so that tests, smoke() and
# bench.py's cpu_baseline / --impl reference legs can run the reference's own CPU path.
# The reference tree is read-only, so it is copied to /tmp first; output goes only
# into oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${DS_REFERENCE:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF absent (GPU box?) - using prebuilt $OUT" >&2
  exit 0
fi
if [ -f "$OUT/.stamp" ]; then exit 0; fi
TMP="$(mktemp -d)"
cp -r "$REF" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$OUT" "$TMP/pkg"
python - "$OUT" <<'PY'
import sys; sys.path.insert(0, sys.argv[1])
from deltaserve import _kernels
assert _kernels.BACKEND == "native", _kernels.BACKEND
print("build_ref: reference deltaserve built, kernel backend =", _kernels.BACKEND)
PY
touch "$OUT/.stamp"
rm -rf "$TMP"
