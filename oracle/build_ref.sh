#!/usr/bin/env bash
# Build the UNMODIFIED reference package `tensched` (pure Python + its one
# Cython kernel, pkg/src/tensched/_recurrent_cy.pyx) into oracle/_ref/.
#
# oracle/_ref/ is test infrastructure (the checker and the CPU baseline arm of
# bench.py) and is git-ignored; it travels to the GPU box with the snapshot.
# The reference mount is read-only, so the build happens in a scratch copy
# under /tmp (setup.py build_ext writes into the source tree).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF absent (GPU box) - using prebuilt $OUT" >&2
  exit 0
fi
SCRATCH="$(mktemp -d /tmp/tensched_ref.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$REF" "$SCRATCH/pkg"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$SCRATCH/site" "$SCRATCH/pkg" >/dev/null
rm -rf "$OUT"
mkdir -p "$OUT"
cp -r "$SCRATCH/site/tensched" "$OUT/tensched"
cp -r "$REF/assets" "$OUT/assets"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import tensched.backend as b
assert b.BACKEND == "cython", b.BACKEND
print("oracle/_ref: tensched built, backend =", b.BACKEND)
PY
