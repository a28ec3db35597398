#!/bin/bash
# Drop-in conformance: the reference's own test suite (pkg/tests, 175 tests)
# run against the B200 engine through the `splitplan` alias package
# (tests/golden/ref_shim).
#
#   bash tests/tools/ref_tests.sh stage     # here: copy the reference tests into
#                                           # tests/golden/_ref_tests (git-ignored;
#                                           # travels to the GPU box, never committed)
#   bash tests/tools/ref_tests.sh run [out] # on the GPU box: run them, log to out
set -u
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
DST=$ROOT/tests/golden/_ref_tests
case "${1:-run}" in
  stage)
    rm -rf "$DST" && mkdir -p "$DST"
    cp /root/reference/pkg/tests/*.py "$DST"/
    echo "staged $(ls "$DST"/test_*.py | wc -l) reference test modules into $DST"
    ;;
  run)
    out=$(realpath -m "${2:-$ROOT/gpurun_out/ref_tests.log}")
    mkdir -p "$(dirname "$out")"
    cd "$DST" && PYTHONPATH="$ROOT/tests/golden/ref_shim:$ROOT" \
      python -m pytest -q -p no:cacheprovider -c /dev/null --rootdir="$DST" --confcutdir="$DST" --continue-on-collection-errors . > "$out" 2>&1
    echo "rc=$?" >> "$out"
    tail -5 "$out"
    ;;
esac
