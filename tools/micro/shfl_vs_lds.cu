// Microbenchmark: do warp shuffles compete with shared-memory loads for the
// same SM datapath?  A: LDS.128 stream, B: SHFL stream, C: both interleaved.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void kA(double* out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x & 1023;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double2 v = sm[(idx + u * 32 + it) & 1023];
      acc.x += v.x; acc.y += v.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

__global__ void kB(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = threadIdx.x + u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) a[u] += __shfl_xor_sync(0xffffffffu, a[u], (u + it) & 31);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void kC(double* out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  double a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = threadIdx.x + u;
  int idx = threadIdx.x & 1023;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double2 v = sm[(idx + u * 32 + it) & 1023];
      acc.x += v.x; acc.y += v.y;
      a[u] += __shfl_xor_sync(0xffffffffu, a[u], (u + it) & 31);
    }
  }
  double s = acc.x + acc.y;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int blocks = 148 * 2, threads = 256, iters = 2000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int k = 0; k < 3; ++k) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (k == 0) kA<<<blocks, threads>>>(out, iters);
      if (k == 1) kB<<<blocks, threads>>>(out, iters);
      if (k == 2) kC<<<blocks, threads>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double warp_instr = (double)blocks * threads / 32 * iters * 16;   // per stream
    const double cyc = ms * 1e-3 * 1.965e9 * 148;                          // SM-cycles
    printf("%s: %.3f ms, %.2f warp-instr per SM-cycle per stream\n",
           k == 0 ? "LDS.128" : (k == 1 ? "SHFL.64" : "both"), ms, warp_instr / cyc);
  }
  return 0;
}
