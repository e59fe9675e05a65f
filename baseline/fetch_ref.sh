#!/usr/bin/env bash
# Install the UNMODIFIED reference (cuclgen 0.1.0, pure Python + numpy) into
# baseline/_ref (git-ignored; gpurun ships it to the GPU box with the snapshot):
#   baseline/_ref/site   pip install --target of /root/reference/pkg (the package)
#   baseline/_ref/tests  the reference's own test helpers (pkg/tests/helpers.py is
#                        not part of the wheel; tests/test_reference_dropin.py uses it)
# Run in the build container (where /root/reference exists); idempotent.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_SRC:-/root/reference}"
DEST="$HERE/_ref"
if [ ! -d "$SRC/pkg" ]; then
    echo "fetch_ref: $SRC/pkg not found (the reference exists only in the build container)" >&2
    exit 1
fi
rm -rf "$DEST" /tmp/cuclgen_build
mkdir -p "$DEST"
# setuptools writes build/ and *.egg-info into the source tree: build from a copy
cp -r "$SRC/pkg" /tmp/cuclgen_build
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DEST/site" /tmp/cuclgen_build
cp -r "$SRC/pkg/tests" "$DEST/tests"
rm -rf /tmp/cuclgen_build
python - "$DEST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1] + "/site")
import cuclgen, cuclgen.oracle, cuclgen.runner
print("fetch_ref: cuclgen", getattr(cuclgen, "__version__", "?"), "installed at", cuclgen.__file__)
PY
