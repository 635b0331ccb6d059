#!/bin/bash
# Install the UNMODIFIED reference package (tomoblocks, pure Python: numpy +
# scipy) into oracle/_ref/ so the CPU baseline can time the reference's own
# harness (cli.py:339-371: build_reconstruction_pipeline + run_pipeline).
# TEST / MEASUREMENT INFRASTRUCTURE ONLY: nothing in the product imports it.
# The setuptools build writes into its source tree and /root/reference is
# read-only, so the install runs from a copy under /tmp.  oracle/_ref/ is
# git-ignored (never committed) but travels to the GPU box with gpurun.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=${1:-/root/reference/pkg}
if [ ! -d "$SRC/src/tomoblocks" ]; then
  echo "build_ref.sh: no reference sources at $SRC (the GPU box uses the prebuilt oracle/_ref)" >&2
  exit 0
fi
TMP=$(mktemp -d /tmp/tomoblocks-src.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP"
rm -rf "$TMP"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import tomoblocks, tomoblocks.pipeline, tomoblocks.cli  # noqa: F401
print("oracle/_ref: tomoblocks", getattr(tomoblocks, "__version__", "0.1.0"), "from", tomoblocks.__file__)
PY
