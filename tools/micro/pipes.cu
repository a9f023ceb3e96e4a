// Microbenchmarks behind the LINEAR_B pass design (round 2):
//  E1-E4  do FP64 (DFMA) and shared-memory loads (LDS.128) overlap on one SM at the
//         kernels' occupancy (8 warps/SM), in the same warp and in different warps?
//  E5     LDS.128 wavefront cost when lane pairs read the same 16 bytes (multicast)
//  E6     tile fill by cp.async.bulk (TMA bulk copy, UBLKCP) vs per-thread cp.async
//         (LDGSTS) while other warps stream LDS.128: who pays on the data pipe?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__

template <int NF, int NL, int MODE>   // MODE 0: every warp both; 1: even warps FP64, odd warps LDS
__global__ void __launch_bounds__(128, 2) k_mix(double* out, int iters) {
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, 1.0);
  __syncthreads();
  double a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = threadIdx.x + u;
  unsigned xacc = 0;
  const int idx = threadIdx.x & 31;
  const double m = 1.0000001, c = 1e-9;
  const bool doF = MODE == 0 || ((threadIdx.x >> 5) & 1) == 0;
  const bool doL = MODE == 0 || ((threadIdx.x >> 5) & 1) == 1;
  for (int it = 0; it < iters; ++it) {
    if (NF > 0 && doF) {
#pragma unroll
      for (int r = 0; r < NF / 16; ++r)
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = fma(a[u], m, c);
    }
    if (NL > 0 && doL) {
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const uint4 v = reinterpret_cast<const uint4*>(sm)[(idx + u * 32 + it * 32) & 2047];
        xacc ^= v.x ^ v.y ^ v.z ^ v.w;   // integer consumption: the FP64 pipe stays free
      }
    }
  }
  double s = (double)xacc;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// E5: SHARE = 1: every lane its own 16 B; 2: lanes (2i, 2i+1) the same 16 B; 3: lanes (l, l^16)
template <int SHARE>
__global__ void __launch_bounds__(128, 2) k_share(double* out, int iters) {
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, 1.0);
  __syncthreads();
  const int l = threadIdx.x & 31;
  const int idx = SHARE == 1 ? l : (SHARE == 2 ? (l >> 1) : (l & 15));
  unsigned xacc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint4 v = reinterpret_cast<const uint4*>(sm)[(idx + u * 32 + it * 32) & 2047];
      xacc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (double)xacc;
}

DEV uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
DEV void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n));
}
DEV void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(b)) : "memory");
}
DEV void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra DONE_%=;\n bra WAIT_%=;\n DONE_%=:\n}" ::"r"(saddr(b)), "r"(phase) : "memory");
}

// E6: warps 1..3 stream LDS.128 from region A; warp 0 fills region B (16 KB tiles from an
// L2-resident global buffer): FILL 0 none, 1 cp.async.bulk (one 512 B copy per lane per tile),
// 2 per-thread 16-byte cp.async.  Reports the time of a fixed LDS count and the fill count.
template <int FILL>
__global__ void __launch_bounds__(128, 2) k_fill(double* out, const double2* src, int iters, unsigned* tiles) {
  extern __shared__ __align__(128) double2 dyn[];
  double2* A = dyn;             // 2048 double2 = 32 KB
  double2* B = dyn + 2048;      // 2 x 1024 double2
  __shared__ uint64_t bar[2];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) A[i] = make_double2(i, 1.0);
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); stop = 0; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w == 0) {
    unsigned n = 0;
    if (FILL == 1) {
      uint32_t ph[2] = {0, 0};
      const double2* s = src + (size_t)(blockIdx.x & 63) * 1024;
      while (!stop) {
        const int b = n & 1;
        if (l == 0) mbar_expect(&bar[b], 16384);
        __syncwarp();
        bulk_g2s(B + b * 1024 + l * 32, s + l * 32, 512, &bar[b]);
        mbar_wait(&bar[b], ph[b]);
        ph[b] ^= 1;
        ++n;
      }
    } else if (FILL == 2) {
      const double2* s = src + (size_t)(blockIdx.x & 63) * 1024;
      while (!stop) {
        const int b = n & 1;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(B + b * 1024 + l + 32 * i)),
                       "l"(s + l + 32 * i) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        ++n;
      }
    }
    if (l == 0) atomicAdd(tiles, n);
    out[blockIdx.x * blockDim.x + threadIdx.x] = B[l].x;
  } else {
    unsigned xacc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint4 v = reinterpret_cast<const uint4*>(A)[(l + u * 32 + it * 32) & 2047];
        xacc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (double)xacc;
    __syncwarp();
    // the last LDS warp to finish stops the filler
    __shared__ int done;
    if (threadIdx.x == 32) done = 0;
    asm volatile("bar.sync 1, 96;");
    if (l == 0 && atomicAdd(&done, 1) == 2) stop = 1;
  }
}

template <class F> float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error: %s\n", cudaGetErrorString(e));
  return ms;
}

int main() {
  const int blocks = 148 * 2, threads = 128, iters = 4000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  int dev_clk = 0;
  cudaDeviceGetAttribute(&dev_clk, cudaDevAttrClockRate, 0);
  const double clk = dev_clk * 1e3;
  auto cyc = [&](float ms) { return ms * 1e-3 * clk; };   // cycles (per SM: all SMs run the same)
  const double warps_sm = 8;
  {
    // FP64 warp-instr = 0.5 SM-clk at 64 lanes/clk/SM; LDS.128 warp-instr = 4 SM-clk
    float f = timeit([&] { k_mix<128, 0, 0><<<blocks, threads>>>(out, iters); });
    float l = timeit([&] { k_mix<0, 16, 0><<<blocks, threads>>>(out, iters); });
    float m = timeit([&] { k_mix<128, 16, 0><<<blocks, threads>>>(out, iters); });
    float s = timeit([&] { k_mix<128, 16, 1><<<blocks, threads>>>(out, iters); });
    printf("E1 DFMA only      : %.3f ms  (%.3f SM-clk per warp DFMA)\n", f, cyc(f) / (warps_sm * iters * 128));
    printf("E2 LDS.128 only   : %.3f ms  (%.3f SM-clk per warp LDS.128)\n", l, cyc(l) / (warps_sm * iters * 16));
    printf("E3 both, same warp: %.3f ms  (sum %.3f, max %.3f)\n", m, f + l, f > l ? f : l);
    printf("E4 both, split warps (4 DFMA + 4 LDS warps, each stream half the work of E1/E2): %.3f ms (max of halves %.3f)\n",
           s, (f > l ? f : l) / 2);
    float m2 = timeit([&] { k_mix<64, 16, 0><<<blocks, threads>>>(out, iters); });
    float f2 = timeit([&] { k_mix<64, 0, 0><<<blocks, threads>>>(out, iters); });
    printf("E3b 64 DFMA + 16 LDS same warp: %.3f ms (DFMA alone %.3f, LDS alone %.3f)\n", m2, f2, l);
  }
  {
    float a = timeit([&] { k_share<1><<<blocks, threads>>>(out, iters); });
    float b = timeit([&] { k_share<2><<<blocks, threads>>>(out, iters); });
    float c = timeit([&] { k_share<3><<<blocks, threads>>>(out, iters); });
    printf("E5 LDS.128 distinct: %.3f SM-clk/instr; lanes (2i,2i+1) shared: %.3f; lanes (l,l^16) shared: %.3f\n",
           cyc(a) / (warps_sm * iters * 16), cyc(b) / (warps_sm * iters * 16), cyc(c) / (warps_sm * iters * 16));
  }
  {
    double2* src;
    cudaMalloc(&src, sizeof(double2) * 1024 * 64);
    cudaMemset(src, 0, sizeof(double2) * 1024 * 64);
    unsigned* tiles;
    cudaMalloc(&tiles, 4);
    const size_t smem = sizeof(double2) * 4096;
    cudaFuncSetAttribute(k_fill<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fill<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fill<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned n[3] = {0, 0, 0};
    float t[3];
    for (int k = 0; k < 3; ++k) {
      t[k] = timeit([&] {
        cudaMemset(tiles, 0, 4);
        if (k == 0) k_fill<0><<<blocks, threads, smem>>>(out, src, iters, tiles);
        if (k == 1) k_fill<1><<<blocks, threads, smem>>>(out, src, iters, tiles);
        if (k == 2) k_fill<2><<<blocks, threads, smem>>>(out, src, iters, tiles);
      });
      cudaMemcpy(&n[k], tiles, 4, cudaMemcpyDeviceToHost);
    }
    const double lds_wf = 6.0 * iters * 16 * 4;   // wavefronts per SM from the 6 LDS warps
    for (int k = 0; k < 3; ++k) {
      const double fill_wf = (double)n[k] / 148 * 128;   // 16 KB tile = 128 x 128 B per SM
      printf("E6 fill=%s: %.3f ms; LDS wavefronts/SM-clk %.3f; fill 128B-units/SM-clk %.3f (tiles %u)\n",
             k == 0 ? "none" : (k == 1 ? "bulk" : "cp.async16"), t[k], lds_wf / cyc(t[k]), fill_wf / cyc(t[k]), n[k]);
    }
  }
  return 0;
}
