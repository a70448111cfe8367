#!/bin/bash
# Stage the REFERENCE into oracle/_ref/ (git-ignored; travels to the GPU box
# with the gpurun snapshot, like the built .so files).  Test/bench
# infrastructure only -- the product never imports anything under oracle/.
#
#   oracle/_ref/site/fmm2d   the reference package, installed from
#                            /root/reference/pkg by the offline pip recipe of
#                            the task (no index, no build isolation); bench.py
#                            --impl reference times its stock fmm_evaluate
#   oracle/_ref/tests        the reference's own unit tests (pkg/tests), run
#                            against the drop-in by tests/test_reference_suite.py
#                            with `fmm2d` aliased to paper_1205_4611_b200
#
# Sources are never copied into the repository history; rerun this script in
# the build container (where /root/reference exists) to refresh the stage.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=${REF:-/root/reference/pkg}
OUT="$HERE/_ref"
[ -d "$REF" ] || { echo "reference not present ($REF): keeping the existing stage"; exit 0; }
mkdir -p "$OUT"
TMP=$(mktemp -d)
cp -r "$REF" "$TMP/pkg"                       # the source tree is read-only: build from a copy
rm -rf "$OUT/site"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$OUT/site" "$TMP/pkg" \
  || { echo "pip install failed; staging the package sources instead"; mkdir -p "$OUT/site";
       cp -r "$TMP/pkg/src/fmm2d" "$OUT/site/"; }
rm -rf "$OUT/tests"
cp -r "$REF/tests" "$OUT/tests"
find "$OUT" -name __pycache__ -prune -exec rm -rf {} +
rm -rf "$TMP"
echo "staged: $(ls "$OUT/site") + $(ls "$OUT/tests" | wc -l) test files"
