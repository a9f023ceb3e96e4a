// Parareal engine helpers shared by 1D and 2D (parareal.py:245-251, a20).
#include "chp_common.cuh"

namespace {

// max |a - b| over n fields (rows of m entries at pitch, m^(dim-1) rows).
__global__ void k_max_abs_diff(int rows, int m, int pitch, int n, const double* __restrict__ a,
                               long long as, const double* __restrict__ b, long long bs,
                               double* out) {
  double mx = 0.0;
  const long long per = (long long)rows * m;
  const long long total = per * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / per;
    const long long r = (t % per) / m;
    const long long j = t % m;
    const long long o = r * pitch + (pitch - m) + j;   // 2D rows lead with the pad
    const double d = fabs(a[f * as + o] - b[f * bs + o]);
    mx = (d > mx || d != d) ? d : mx;
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, mx);
}

}  // namespace

cudaError_t chp_launch_max_abs_diff(const chp_grid& g, int n_fields, const double* a,
                                    long long as, const double* b, long long bs, double* out,
                                    cudaStream_t st) {
  const int rows = g.dim == 1 ? 1 : g.m;
  const long long total = (long long)rows * g.m * n_fields;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_max_abs_diff<<<(int)blocks, 256, 0, st>>>(rows, g.m, g.pitch, n_fields, a, as, b, bs, out);
  return cudaGetLastError();
}
