#!/bin/bash
# Stage the UNMODIFIED reference package (/root/reference/pkg, pure Python +
# numpy) into oracle/_ref/ so bench.py's reference arm and cpu_baseline can
# time the reference itself on the GPU box, where /root/reference does not
# exist.  oracle/_ref/ is git-ignored (no reference source enters the repo
# history) but not gpurun-ignored, so it travels with the snapshot like the
# built .so.  The build runs from a copy under /tmp because /root/reference is
# read-only; --no-deps: numpy is already in the image.
set -euo pipefail
REF=${1:-/root/reference/pkg}
HERE="$(cd "$(dirname "$0")" && pwd)"
[ -f "$REF/pyproject.toml" ] || { echo "stage_ref: $REF not found (nothing staged)"; exit 0; }
TMP=$(mktemp -d /tmp/hlq_ref_build.XXXXXX)
cp -r "$REF" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import hlq
print("staged reference hlq", hlq.__version__, "from", hlq.__file__)
PY
