#!/usr/bin/env bash
# Build the UNMODIFIED reference (`/root/reference/pkg`, Python + its Cython core)
# into oracle/_ref/ -- test/bench infrastructure only (git-ignored, travels to the
# GPU box with the gpurun snapshot).  The reference build writes into its source
# tree, and /root/reference is read-only, so it is installed from a scratch copy.
# Nothing from the reference is ever copied into tracked files.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${LRAMM_REFERENCE:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; oracle/_ref left as is" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/lramm_ref_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP"
PYTHONPATH="$HERE/_ref" python -c "import lramm; print('reference lramm', lramm.__version__, 'backend', lramm.backend_name())"
