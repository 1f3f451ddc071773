// Launch-overhead probe: what a kernel boundary costs inside a CUDA graph
// versus a grid-wide barrier inside one persistent kernel (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency_probe tools/latency_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_empty(float* p, int spin) {
  float x = threadIdx.x;
  for (int i = 0; i < spin; ++i) x = x * 0.999f + 1.f;
  if (x == -1.f) p[0] = x;
}

__global__ void k_pdl(float* p, int spin) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float x = threadIdx.x;
  for (int i = 0; i < spin; ++i) x = x * 0.999f + 1.f;
  if (x == -1.f) p[0] = x;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// hand-rolled sense-reversal grid barrier
__device__ __forceinline__ void gbar(unsigned* count, volatile unsigned* gen, unsigned nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblk - 1) {
      *count = 0;
      __threadfence();
      *gen = g + 1;
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_persist(float* p, int phases, int spin, unsigned* count, unsigned* gen) {
  float x = threadIdx.x;
  for (int ph = 0; ph < phases; ++ph) {
    for (int i = 0; i < spin; ++i) x = x * 0.999f + 1.f;
    gbar(count, gen, gridDim.x);
  }
  if (x == -1.f) p[0] = x;
}

__global__ void k_persist_cg(float* p, int phases, int spin) {
  cg::grid_group g = cg::this_grid();
  float x = threadIdx.x;
  for (int ph = 0; ph < phases; ++ph) {
    for (int i = 0; i < spin; ++i) x = x * 0.999f + 1.f;
    g.sync();
  }
  if (x == -1.f) p[0] = x;
}

int main() {
  float* p;
  unsigned *cnt, *gen;
  cudaMalloc(&p, 4);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int NK = 16, REPS = 50;
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int ctas : {148, 384, 768})
      for (int spin : {0, 2000}) {
        cudaGraph_t gr;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < REPS; ++r)
          for (int k = 0; k < NK; ++k) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctas);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = pdl;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (pdl)
              cudaLaunchKernelEx(&cfg, k_pdl, p, spin);
            else
              cudaLaunchKernelEx(&cfg, k_empty, p, spin);
          }
        cudaStreamEndCapture(s, &gr);
        cudaGraphExec_t ex;
        cudaGraphInstantiate(&ex, gr, 0);
        cudaGraphLaunch(ex, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("graph pdl=%d ctas=%d spin=%d: %.3f us per kernel\n", pdl, ctas, spin, ms * 1e3 / (NK * REPS));
        cudaGraphExecDestroy(ex);
        cudaGraphDestroy(gr);
      }
  for (int per : {1, 2})
    for (int spin : {0, 2000}) {
      const int blocks = nsm * per;
      const int phases = NK * REPS;
      k_persist<<<blocks, 256, 0, s>>>(p, 4, spin, cnt, gen);
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      k_persist<<<blocks, 256, 0, s>>>(p, phases, spin, cnt, gen);
      cudaEventRecord(e1, s);
      cudaStreamSynchronize(s);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("persistent (atomic barrier) blocks=%d spin=%d: %.3f us per phase\n", blocks, spin,
             ms * 1e3 / phases);
      void* args[] = {&p, (void*)&phases, &spin};
      cudaLaunchCooperativeKernel((void*)k_persist_cg, blocks, 256, args, 0, s);
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      cudaLaunchCooperativeKernel((void*)k_persist_cg, blocks, 256, args, 0, s);
      cudaEventRecord(e1, s);
      cudaStreamSynchronize(s);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("persistent (cg grid.sync) blocks=%d spin=%d: %.3f us per phase (%s)\n", blocks, spin,
             ms * 1e3 / phases, cudaGetErrorString(cudaGetLastError()));
    }
  // spin-only reference: one kernel, no barriers
  for (int spin : {2000}) {
    cudaEventRecord(e0, s);
    k_empty<<<nsm, 256, 0, s>>>(p, spin * NK * REPS);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("spin reference: %.3f us per phase-equivalent\n", ms * 1e3 / (NK * REPS));
  }
  return 0;
}
