// debug harness: T (unnormalised DST-I) of pairs with wdst::pair_dst<N>
#include "../../paper_2304_14074_b200/csrc/chp_wdst.cuh"
template <int N>
__global__ void kdst(const double* in, double* out, const double2* wtab, int npairs) {
  constexpr int L = wdst::Geo<N>::L;
  extern __shared__ __align__(16) double sm[];
  const int gpb = blockDim.x / L;
  double2* twt = reinterpret_cast<double2*>(sm + (size_t)gpb * 2 * N);
  wdst::load_twiddles<N>(twt, wtab + N);
  __syncthreads();
  const int g = threadIdx.x / L, l = threadIdx.x % L;
  const int p = blockIdx.x * gpb + g;
  const double* a = in + (size_t)p * 2 * N;
  const double* b = a + N;
  double* scr = sm + (size_t)g * 2 * N;
  const bool ok = p < npairs;
  auto ld = [&](int n, double& x, double& xm, double& y, double& ym) {
    x = (ok && n) ? a[n] : 0.0; xm = (ok && n) ? a[N - n] : 0.0;
    y = (ok && n) ? b[n] : 0.0; ym = (ok && n) ? b[N - n] : 0.0;
  };
  auto st = [&](int k, double a2, double a21, double b2, double b21) {
    if (!ok) return;
    out[(size_t)p * 2 * N + 2 * k] = a2; out[(size_t)p * 2 * N + 2 * k + 1] = a21;
    out[(size_t)p * 2 * N + N + 2 * k] = b2; out[(size_t)p * 2 * N + N + 2 * k + 1] = b21;
  };
  wdst::pair_dst<N>(ld, st, reinterpret_cast<double2*>(scr), twt, l, __ldg(&wtab[l]));
}
extern "C" int dbg_dst(int N, const double* in, double* out, const double2* wtab, int npairs) {
  const int threads = 256;
  if (N == 1024) {
    const int gpb = threads / 64;
    size_t sm = sizeof(double) * gpb * 2 * N + 16 * (N + 64);
    cudaFuncSetAttribute(kdst<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kdst<1024><<<(npairs + gpb - 1) / gpb, threads, sm>>>(in, out, wtab, npairs);
  } else if (N == 256) {
    const int gpb = threads / 16;
    size_t sm = sizeof(double) * gpb * 2 * N + 16 * (N + 64);
    cudaFuncSetAttribute(kdst<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kdst<256><<<(npairs + gpb - 1) / gpb, threads, sm>>>(in, out, wtab, npairs);
  }
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
