#!/usr/bin/env bash
# Builds the CPU checker from the UNMODIFIED reference headers (test infrastructure).
#   oracle/_ref/libmomc_ref.so  <- oracle/ref_capi.cpp + /root/reference/proj/include + oracle/eigen_shim
#   oracle/_ref/libmomc_oracle.so <- oracle/momc_oracle.c (the C restatement; no reference needed)
# The reference sources are compiled where they lie; nothing is copied into the repo.
# -ffp-contract=off pins the FP64 evaluation order (see oracle/eigen_shim/Eigen/Dense).
# -march=x86-64-v3 (not native): the .so travels to the GPU box whose host CPU may differ.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF_INC="${MOMC_REFERENCE_INCLUDE:-/root/reference/proj/include}"
OUT="$HERE/_ref"
mkdir -p "$OUT"
CXXFLAGS="-std=gnu++20 -O3 -march=x86-64-v3 -mtune=generic -ffp-contract=off -fPIC -pthread"

cc -std=c11 -O2 -march=x86-64-v3 -mtune=generic -ffp-contract=off -fPIC -pthread -shared \
   -o "$OUT/libmomc_oracle.so" "$HERE/momc_oracle.c" -lm

if [ -d "$REF_INC/momc" ]; then
  g++ $CXXFLAGS -shared -I"$HERE/eigen_shim" -I"$REF_INC" \
      -o "$OUT/libmomc_ref.so" "$HERE/ref_capi.cpp"
  echo "built $OUT/libmomc_ref.so"
else
  echo "reference headers not found at $REF_INC; keeping prebuilt $OUT/libmomc_ref.so (if any)" >&2
fi
echo "built $OUT/libmomc_oracle.so"
