#!/bin/bash
# Bounds-checked build + the sanitizer cases (compute-sanitizer is closed on this pool); restores the
# product build afterwards.  Run on a GPU box: bash tools/bounds_check.sh
CIL_BUILD_DEFINES="-DCIL_BOUNDS_CHECK" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
python tools/sanitize_cases.py; rc=$?
python paper_2203_14742_b200/build.py --force > /dev/null
exit $rc
