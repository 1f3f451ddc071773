#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. The same UNMODIFIED reference sources as
# build_ref.sh, with their FFTW3 calls resolved by NVIDIA cuFFTW (the
# FFTW-compatible front end of cuFFT) instead of the CPU stand-in: the
# "reference + library GPU FFT" baseline SURVEY.md §8d asks for.  Output:
# oracle/_ref/libref_litho_cufftw.so (git-ignored; travels to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${LITHO_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
CUDA=/usr/local/cuda
if [ ! -d "$REF/src/core" ]; then
  echo "build_ref_cufftw: reference sources not found at $REF (skipped)" >&2
  exit 0
fi
mkdir -p "$OUT/obj_cufftw"
JSON_INC="${LITHO_JSON_INC:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
CXXFLAGS="-O2 -std=c++20 -fPIC -fopenmp -I$HERE/shim_cufftw -I$HERE/shim -I$CUDA/include -I$REF/src -I$REF/src/core -I$JSON_INC"
pids=()
for s in geometry bvh boolean raster imaging ai contour segment mrc io; do
  g++ $CXXFLAGS -c "$REF/src/core/$s.cpp" -o "$OUT/obj_cufftw/$s.o" & pids+=($!)
done
g++ $CXXFLAGS -c "$HERE/ref_capi.cpp" -o "$OUT/obj_cufftw/ref_capi.o" & pids+=($!)
gcc -O2 -fPIC -c "$HERE/shim_cufftw/threads_stub.c" -o "$OUT/obj_cufftw/threads_stub.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
g++ -shared -fopenmp -o "$OUT/libref_litho_cufftw.so" "$OUT"/obj_cufftw/*.o -L$CUDA/lib64 -lcufftw -lcufft \
  -Wl,-rpath,$CUDA/lib64
echo "build_ref_cufftw: $OUT/libref_litho_cufftw.so"
