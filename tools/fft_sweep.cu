// Exchange-layout sweep for the register FFT (fftr.cuh): for each plan length
// and shared-memory layout, run many row FFTs, check one row against an fp64
// DFT on the host, and time with CUDA events.  Run under ncu to read the
// shared-memory bank-conflict counters per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_15036_b200/csrc
#include <cmath>
#include <complex>
#include <cstdio>
#include <vector>

#include "fftr.cuh"

using namespace lg;

template <int LG, typename X>
__global__ void sweep_kernel(const cx<float>* __restrict__ in, cx<float>* __restrict__ out,
                             const cx<float>* __restrict__ tw, int rows, int reps) {
  constexpr int E = RPlan<(1 << LG)>::E, TPR = RPlan<(1 << LG)>::TPR, L = 1 << LG;
  extern __shared__ __align__(16) unsigned char raw[];
  const int groups = blockDim.x / TPR, gid = threadIdx.x / TPR, t = threadIdx.x % TPR;
  const int row = blockIdx.x * groups + gid;
  const int bytes = (X::template bytes<(1 << LG)>() + 15) / 16 * 16;
  cx<float>* sm = reinterpret_cast<cx<float>*>(raw + size_t(gid) * bytes);
  const GSync sync = make_gsync<(1 << LG)>(gid, groups);
  const int r = row < rows ? row : rows - 1;
  cx<float> v[E];
  for (int e = 0; e < E; ++e) v[e] = in[size_t(r) * L + t + e * TPR];
  for (int k = 0; k < reps; ++k) fftr<float, (1 << LG), -1, X>(v, sm, tw, t, sync);
  if (row < rows)
    for (int e = 0; e < E; ++e) out[size_t(row) * L + t + e * TPR] = v[e];
}

template <int LG, typename X>
void run(const char* name, int rows) {
  constexpr int L = 1 << LG, TPR = RPlan<(1 << LG)>::TPR;
  std::vector<cx<float>> h(size_t(rows) * L), o(size_t(rows) * L);
  for (size_t i = 0; i < h.size(); ++i) {
    h[i].x = float(std::sin(0.37 * double(i)) + 0.1 * double(i % 7));
    h[i].y = float(std::cos(0.11 * double(i)));
  }
  std::vector<cx<float>> tw(TwLen<(1 << LG)>::value + 1);
  fill_rtwiddles<(1 << LG)>([&](int idx, int rk, int NsR) {
    const double a = 2.0 * M_PI * double(rk) / double(NsR);
    tw[idx].x = float(std::cos(a));
    tw[idx].y = float(-std::sin(a));
  });
  cx<float>*din, *dout, *dtw;
  cudaMalloc(&din, h.size() * 8);
  cudaMalloc(&dout, h.size() * 8);
  cudaMalloc(&dtw, tw.size() * 8);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dtw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice);
  const int groups = TPR >= 256 ? 1 : 256 / TPR;
  const int bytes = (X::template bytes<(1 << LG)>() + 15) / 16 * 16;
  const size_t smem = size_t(groups) * bytes;
  cudaFuncSetAttribute(sweep_kernel<LG, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int grid = (rows + groups - 1) / groups;
  // correctness: 1 rep vs host DFT of row 0
  sweep_kernel<LG, X><<<grid, groups * TPR, smem>>>(din, dout, dtw, rows, 1);
  cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0, mag = 0;
  for (int k = 0; k < L; ++k) {
    std::complex<double> acc = 0;
    for (int x = 0; x < L; ++x)
      acc += std::complex<double>(h[x].x, h[x].y) * std::polar(1.0, -2.0 * M_PI * double(k) * x / L);
    err = std::max(err, std::abs(acc - std::complex<double>(o[k].x, o[k].y)));
    mag = std::max(mag, std::abs(acc));
  }
  const int reps = 20;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  sweep_kernel<LG, X><<<grid, groups * TPR, smem>>>(din, dout, dtw, rows, reps);
  cudaEventRecord(a);
  sweep_kernel<LG, X><<<grid, groups * TPR, smem>>>(din, dout, dtw, rows, reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 5.0 * L * LG * double(rows) * reps;
  std::printf("LG=%2d %-8s rel_err=%.2e  %.3f ms  %.1f TFLOP/s (5NlogN)  err=%s\n", LG, name, err / mag, ms,
              flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dtw);
}

template <int LG>
void all(int rows) {
  run<LG, Xch2<0>>("f2add4", rows);
  run<LG, Xch2<1>>("f2xor3", rows);
  run<LG, Xch2<2>>("f2xor4", rows);
  run<LG, Xch2<3>>("f2xor3b", rows);
  run<LG, XchS<0>>("saadd4", rows);
  run<LG, XchS<1>>("saxor3", rows);
  run<LG, XchS<2>>("saxor4", rows);
  run<LG, XchS<3>>("saxor3b", rows);
  run<LG, XchS<4>>("saadd5", rows);
}

int main() {
  all<9>(16384);
  all<10>(8192);
  all<11>(4096);
  all<12>(2048);
  return 0;
}
