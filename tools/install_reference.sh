#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot).  Run in the build
# container, where /root/reference exists; the GPU box only uses the result.
#
#  * baseline/_ref/bttb       -- the reference package (pip --target install;
#                                the build needs a writable source tree, so it
#                                builds from a copy under /tmp)
#  * baseline/_ref/ref_tests  -- the reference's own test suite, run unchanged
#                                against the drop-in by tests/test_gpu_reference_suite.py
#                                (SURVEY.md section 8(b) "Conformance")
set -euo pipefail
here="$(cd "$(dirname "$0")/.." && pwd)"
src="${BTTB_REFERENCE:-/root/reference/pkg}"
if [ ! -d "$src/src/bttb" ]; then
  echo "reference sources not found at $src" >&2
  exit 1
fi
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
rm -rf "$here/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$here/baseline/_ref" "$tmp/pkg" > "$tmp/pip.log" 2>&1 || { cat "$tmp/pip.log"; exit 1; }
cp -r "$src/tests" "$here/baseline/_ref/ref_tests"
find "$here/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
echo "installed reference into $here/baseline/_ref"
