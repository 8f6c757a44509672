#!/bin/bash
# Bounds-checked build + the sanitizer cases + the whole GPU test suite (compute-sanitizer is closed on
# this pool); restores the product build afterwards.  Run on a GPU box: bash tools/bounds_check.sh
CIL_BUILD_DEFINES="-DCIL_BOUNDS_CHECK" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
python tools/sanitize_cases.py; rc=$?
CIL_REPORT_BOUNDS=1 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | grep -E "bounds violations|passed|failed|error"; rc2=${PIPESTATUS[0]}
python paper_2203_14742_b200/build.py --force > /dev/null
[ $rc -ne 0 ] && exit $rc
exit $rc2
