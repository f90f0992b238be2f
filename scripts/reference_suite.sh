#!/bin/bash
# Run the REFERENCE's own pytest suite (/root/reference/pkg/tests, read-only,
# present only in the build container) against this package, through the
# `uotkit` shim in scripts/uotkit_shim (test-only; private helpers the tests
# import -- _smin_cols/_smin_rows/_h0/_neg_conj_neg_sum -- are restated there).
#
#   scripts/reference_suite.sh            # stage _reftests/ (git-ignored)
#   gpurun -- 'cd _reftests && PYTHONPATH=$GRAFT_REPO_ROOT/scripts/uotkit_shim:$GRAFT_REPO_ROOT:. \
#              python -m pytest tests -q -p no:cacheprovider -rf'
#
# The same suite on the reference itself (CPU, here) gives the baseline:
#   cd _reftests && PYTHONPATH=/root/reference/pkg/src python -m pytest tests -q
# Result (round 1): profiles/r1_reference_suite.txt.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf "$ROOT/_reftests"
mkdir -p "$ROOT/_reftests/tests"
cp /root/reference/pkg/tests/*.py "$ROOT/_reftests/tests/"
# the reference's own host-side certify helpers (out of the package's scope), for the shim
cp /root/reference/pkg/src/uotkit/certify.py "$ROOT/_reftests/_ref_certify.py"
echo "staged $(ls "$ROOT/_reftests/tests" | wc -l) reference test files in _reftests/tests"
