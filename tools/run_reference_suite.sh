#!/bin/sh
# Drop-in check: run the REFERENCE's own test-suite against this package.
# In the build container (where /root/reference exists):
#     sh tools/run_reference_suite.sh stage      # copies the reference's tests into build_exp/reftests (git-ignored, never committed)
#     gpurun -- 'sh tools/run_reference_suite.sh run'
# `import meshreg` resolves to tools/meshreg_shim, which aliases this package
# and its submodules under the reference's names.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
case "$1" in
  stage)
    mkdir -p "$ROOT/build_exp/reftests"
    cp /root/reference/pkg/tests/*.py "$ROOT/build_exp/reftests/"
    ;;
  run)
    mkdir -p "$ROOT/gpurun_out"
    cd "$ROOT/build_exp/reftests"
    PYTHONPATH="$ROOT/tools/meshreg_shim:$ROOT" python -m pytest . -q -p no:cacheprovider \
      --timeout 600 -rf --tb=line --durations=5 2>&1 | tail -40 > "$ROOT/gpurun_out/reference_suite.log" || true
    tail -15 "$ROOT/gpurun_out/reference_suite.log"
    ;;
  *) echo "usage: $0 stage|run"; exit 2;;
esac
