#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the UNMODIFIED reference sources where they
# lie under /root/reference (never copied into this repo) together with the
# FFTW3 / Eigen stand-ins in oracle/shim and the extern "C" veneer
# oracle/ref_capi.cpp into oracle/_ref/libref_litho.so (git-ignored; travels to
# the GPU box with the snapshot). Release flags as the reference's own CMake
# default (-O2 here; no -ffast-math, no FMA contraction on x86-64 default).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${LITHO_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src/core" ]; then
  echo "build_ref: reference sources not found at $REF (skipped)" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
SRCS="geometry bvh boolean raster imaging ai contour segment mrc io"
JSON_INC="${LITHO_JSON_INC:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
CXXFLAGS="-O2 -std=c++20 -fPIC -fopenmp -I$HERE/shim -I$REF/src -I$REF/src/core -I$JSON_INC"
pids=()
for s in $SRCS; do
  g++ $CXXFLAGS -c "$REF/src/core/$s.cpp" -o "$OUT/obj/$s.o" & pids+=($!)
done
g++ $CXXFLAGS -c "$HERE/ref_capi.cpp" -o "$OUT/obj/ref_capi.o" & pids+=($!)
gcc -O2 -std=gnu11 -fPIC -fopenmp -c "$HERE/shim/fftw_shim.c" -o "$OUT/obj/fftw_shim.o" & pids+=($!)
gcc -O2 -std=gnu11 -fPIC -fopenmp -c "$HERE/fft64.c" -o "$OUT/obj/fft64.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
g++ -shared -fopenmp -o "$OUT/libref_litho.so" "$OUT"/obj/*.o
echo "build_ref: $OUT/libref_litho.so"
