#!/usr/bin/env bash
# Run the reference's OWN test suite with rebk/rek/rabk/rk routed through
# librebk (tools/ref_shim_plugin.py).  Test infrastructure, not product.
#
# In this container (where /root/reference exists) it first stages the
# unmodified reference: the package is pip-installed into baseline/_ref (the
# install DESIGN.md §6 records) and its tests directory is placed beside it
# as baseline/_ref/kaczmarz_tests.  baseline/_ref is git-ignored (never
# committed) but travels to the GPU box with gpurun, where this script then
# runs the suite on the B200:
#
#   tools/run_reference_tests.sh stage            # here
#   gpurun -- tools/run_reference_tests.sh run    # on the box
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="$ROOT/baseline/_ref"

case "${1:-run}" in
stage)
    tmp="$(mktemp -d)"
    cp -r /root/reference/pkg "$tmp/pkg"
    python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
        --no-deps --target "$REF" --upgrade "$tmp/pkg" >/dev/null
    rm -rf "$REF/kaczmarz_tests"
    cp -r /root/reference/pkg/tests "$REF/kaczmarz_tests"
    rm -rf "$tmp"
    echo "staged kaczmarz into $REF (tests in $REF/kaczmarz_tests)"
    ;;
run)
    shift || true
    cd "$REF/kaczmarz_tests"
    PYTHONPATH="$REF:$ROOT" python -m pytest -q -p no:cacheprovider -p tools.ref_shim_plugin \
        --rootdir "$REF/kaczmarz_tests" -c /dev/null "$@" .
    ;;
*)
    echo "usage: $0 stage|run [pytest args]" >&2
    exit 2
    ;;
esac
