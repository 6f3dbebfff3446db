#!/usr/bin/env bash
# Builds tests/cpp/_bin/dropin_test against the unmodified reference headers (+ Eigen shim),
# the drop-in header and libmomc_b200.so. Needs /root/reference; the binary travels to the
# GPU box (tests/cpp/_bin is git-ignored, not gpurun-ignored).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF_INC="${MOMC_REFERENCE_INCLUDE:-/root/reference/proj/include}"
[ -d "$REF_INC/momc" ] || { echo "reference headers not found; keeping prebuilt binary" >&2; exit 0; }
mkdir -p "$HERE/_bin"
g++ -std=gnu++20 -O2 -march=x86-64-v3 -mtune=generic -ffp-contract=off -pthread \
    -I"$ROOT/oracle/eigen_shim" -I"$REF_INC" -I"$ROOT/include" \
    -o "$HERE/_bin/dropin_test" "$HERE/dropin_test.cpp" \
    -L"$ROOT/paper_2604_26477_b200" -lmomc_b200 -Wl,-rpath,'$ORIGIN/../../../paper_2604_26477_b200'
echo "built $HERE/_bin/dropin_test"
