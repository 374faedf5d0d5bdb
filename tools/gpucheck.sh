#!/bin/bash
# Builds the library (and optional variants) and fails loudly, so a GPU call
# never runs a stale .so:  tools/gpucheck.sh [variant-name -DFLAG ...]
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2510_14392_b200/csrc 2>&1 | grep -iE "error" -A3 && exit 1
if [ $# -gt 0 ]; then tools/build_variant.sh "$@" > /dev/null; fi
echo build-ok
