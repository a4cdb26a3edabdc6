// Launch-gap probe: a chain of dependent small kernels (27 CTAs, ~N us of
// work each), plain vs with a memset between kernels vs PDL vs CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kwork(float* buf, int iters, int* ctr) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float a = buf[threadIdx.x + blockIdx.x * blockDim.x];
  for (int i = 0; i < iters; ++i) a = a * 0.999f + 0.001f;
  buf[threadIdx.x + blockIdx.x * blockDim.x] = a;
  if (threadIdx.x == 0) atomicAdd(ctr, 1);
}
int main() {
  float* buf; int* ctr; cudaMalloc(&buf, 1 << 20); cudaMalloc(&ctr, 64 * 4); cudaMemset(buf, 0, 1 << 20);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int N = 1000;
  for (int iters : {0, 1000, 4000}) {
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaGraph_t g = nullptr; cudaGraphExec_t ge = nullptr;
        auto body = [&](int m) {
          for (int i = 0; i < N; ++i) {
            if (m == 1) cudaMemsetAsync(ctr + (i & 7), 0, 4, s);
            cudaLaunchConfig_t cfg = {dim3(27), dim3(128), 0, s, nullptr, 0};
            cudaLaunchAttribute at[1];
            if (m == 2) { at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1; }
            cudaLaunchKernelEx(&cfg, kwork, buf, iters, ctr);
          }
        };
        if (mode == 3) { cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal); body(2); cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0); cudaGraphLaunch(ge, s); }
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        if (mode == 3) cudaGraphLaunch(ge, s); else body(mode);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        if (ge) { cudaGraphExecDestroy(ge); cudaGraphDestroy(g); }
      }
      const char* nm[] = {"plain", "memset+plain", "pdl", "graph(pdl)"};
      printf("iters %5d %-14s %8.2f us/kernel\n", iters, nm[mode], best * 1000 / N);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
