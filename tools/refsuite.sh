#!/usr/bin/env bash
# Run the reference's own test suites (pkg/tests, pkg/trainer/tests) against
# the B200 path via tools/refpatch.py.
#
#   tools/refsuite.sh stage   # HERE: install the reference into baseline/_ref
#                             # (git-ignored; travels with gpurun) + its tests
#   tools/refsuite.sh run     # GPU box: suites twice -- stock, then patched
#   tools/refsuite.sh clean   # HERE: drop the staged copy again (nothing of it stays)
#
# The staged tree is test infrastructure only: nothing in the product, tests/,
# smoke() or bench.py reads it.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF=/root/reference/pkg
STAGE="$ROOT/baseline/_ref"
OUT="$ROOT/gpurun_out/refsuite"

case "${1:-}" in
stage)
    tmp="$(mktemp -d)"
    cp -r "$REF" "$tmp/pkg"                  # the build writes egg-info next to the sources
    rm -rf "$STAGE"
    python -m pip install -q --no-index --no-build-isolation --no-deps --target "$STAGE" \
        "$tmp/pkg" "$tmp/pkg/trainer"
    mkdir -p "$STAGE/_tests"
    cp -r "$REF/tests" "$STAGE/_tests/pkg"
    cp -r "$REF/trainer/tests" "$STAGE/_tests/trainer"
    rm -rf "$tmp"
    ;;
run)
    mkdir -p "$OUT"
    cd "$STAGE/_tests"
    export PYTHONPATH="$STAGE:$ROOT"
    python -m pytest pkg trainer -q -p no:cacheprovider -rf > "$OUT/stock.txt" 2>&1 || true
    python -m pytest pkg trainer -q -p no:cacheprovider -rf -p tools.refpatch \
        > "$OUT/patched.txt" 2>&1 || true
    tail -n 12 "$OUT/stock.txt" "$OUT/patched.txt"
    ;;
clean)
    rm -rf "$STAGE"
    ;;
*)
    echo "usage: $0 stage|run|clean" >&2
    exit 2
    ;;
esac
