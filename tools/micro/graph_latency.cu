// Microbenchmark: per-kernel cost of a CUDA graph of k dependent kernels on
// B200 (empty kernels, 1 or 1250 CTAs, small or ~480-byte parameters).
#include <cstdio>
#include <cuda_runtime.h>
struct Big { char b[480]; };
__global__ void k_small(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p[0] == 12345) p[1] = 1; }
__global__ void k_big(const Big a, int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && a.b[7] == 3) p[1] = 1; }
__global__ void k_ticket(int* p, unsigned* t) {
  __shared__ int last;
  if (threadIdx.x == 0) { __threadfence(); last = atomicAdd(t, 1u) == gridDim.x - 1; }
  __syncthreads();
  if (last && threadIdx.x == 0) *t = 0;
}
int main() {
  int* p; unsigned* t; cudaMalloc(&p, 64); cudaMalloc(&t, 64); cudaMemset(p, 0, 64); cudaMemset(t, 0, 64);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  Big big{}; big.b[7] = 1;
  for (int variant = 0; variant < 5; ++variant) {
    const int K = 8;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < K; ++i) {
      if (variant == 0) k_small<<<1, 32, 0, s>>>(p);
      if (variant == 1) k_small<<<1250, 64, 0, s>>>(p);
      if (variant == 2) k_big<<<1250, 64, 0, s>>>(big, p);
      if (variant == 3) k_ticket<<<1250, 64, 0, s>>>(p, t);
      if (variant == 4) k_small<<<148, 512, 0, s>>>(p);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int R = 200;
    cudaEventRecord(a, s);
    for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("variant %d: %.2f us per kernel (graph of %d)\n", variant, 1000.0 * ms / R / K, K);
    // launch-by-launch
    cudaEventRecord(a, s);
    for (int r = 0; r < R; ++r)
      for (int i = 0; i < K; ++i) {
        if (variant == 0) k_small<<<1, 32, 0, s>>>(p);
        if (variant == 1) k_small<<<1250, 64, 0, s>>>(p);
        if (variant == 2) k_big<<<1250, 64, 0, s>>>(big, p);
        if (variant == 3) k_ticket<<<1250, 64, 0, s>>>(p, t);
        if (variant == 4) k_small<<<148, 512, 0, s>>>(p);
      }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("variant %d: %.2f us per kernel (stream launches)\n", variant, 1000.0 * ms / R / K);
  }
  return 0;
}
