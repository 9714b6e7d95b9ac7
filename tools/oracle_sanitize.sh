#!/bin/bash
# The oracle's pins under AddressSanitizer + UndefinedBehaviorSanitizer
# (SURVEY.md §5): builds oracle/liboracle_san.so (same sources, -fsanitize=
# address,undefined, UB aborts) and runs the CPU oracle tests against it.
#   bash tools/oracle_sanitize.sh [pytest args]
set -e
cd "$(dirname "$0")/.."
make -s -C oracle liboracle_san.so
ASAN_SO=$(gcc -print-file-name=libasan.so)
UBSAN_SO=$(gcc -print-file-name=libubsan.so)
export S3R_ORACLE_SO=oracle/liboracle_san.so
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
LD_PRELOAD="$ASAN_SO $UBSAN_SO" python -m pytest -q -p no:cacheprovider \
    tests/test_oracle_pins.py tests/test_oracle_backward.py tests/test_oracle_conventional.py \
    tests/test_oracle_jitter.py "$@"
