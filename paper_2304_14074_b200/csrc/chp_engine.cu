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

// ---------------------------------------------------------------------------
// Field diagnostics (grid.py:147-181: l2_norm, energy, mass) on the device.
// One block per field, fixed-order reduction (per-thread strided sums, then a
// fixed shared-memory tree): bitwise reproducible.  Per field, out[4 f + q]:
//   q = 0: sum v^2                      (l2_norm = sqrt(h^d * .))
//   q = 1: sum (v^2 - 1)^2              (energy bulk, x 0.25)
//   q = 2: sum of squared differences   (np.diff with the Dirichlet zeros
//          prepended and appended along every axis, grid.py:168-175)
//   q = 3: sum v                        (mass = h^d * .)
// ---------------------------------------------------------------------------
namespace {

constexpr int kDiagThreads = 512;

__global__ void __launch_bounds__(kDiagThreads) k_field_stats(int dim, int m, int pitch,
                                                             const double* __restrict__ in,
                                                             long long stride, double* out) {
  __shared__ double red[4][kDiagThreads];
  const double* v = in + (long long)blockIdx.x * stride;
  const int off = dim == 2 ? pitch - m : 0;          // 2D rows lead with the pad column
  const long long total = dim == 2 ? (long long)m * m : m;
  double s2 = 0.0, sb = 0.0, sg = 0.0, s1 = 0.0;
  for (long long t = threadIdx.x; t < total; t += kDiagThreads) {
    const int i = dim == 2 ? (int)(t / m) : 0;
    const int j = dim == 2 ? (int)(t % m) : (int)t;
    const double x = v[(long long)i * pitch + off + j];
    const double q = x * x - 1.0;
    s2 += x * x;
    sb += q * q;
    s1 += x;
    // difference with the previous node along each axis (zero before the first),
    // plus the closing difference to the trailing zero at the last node
    const double xl = j > 0 ? v[(long long)i * pitch + off + j - 1] : 0.0;
    double g = (x - xl) * (x - xl);
    if (j == m - 1) g += x * x;
    if (dim == 2) {
      const double xu = i > 0 ? v[(long long)(i - 1) * pitch + off + j] : 0.0;
      g += (x - xu) * (x - xu);
      if (i == m - 1) g += x * x;
    }
    sg += g;
  }
  red[0][threadIdx.x] = s2;
  red[1][threadIdx.x] = sb;
  red[2][threadIdx.x] = sg;
  red[3][threadIdx.x] = s1;
  __syncthreads();
  for (int w = kDiagThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 4) out[4LL * blockIdx.x + threadIdx.x] = red[threadIdx.x][0];
}

}  // namespace

cudaError_t chp_launch_field_stats(const chp_grid& g, int n_fields, const double* in,
                                   long long stride, double* out, cudaStream_t st) {
  k_field_stats<<<n_fields, kDiagThreads, 0, st>>>(g.dim, g.m, g.pitch, in, stride, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FP64 peak probe (bench.py): 16 independent DFMA chains per thread, so the
// FP64 pipe, not the dependency latency, bounds it.  2 * 16 * iters flop per thread.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) k_dfma_probe(int iters, double* out) {
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = 1e-3 * (threadIdx.x + j);
  const double m = 0.9999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fma(a[j], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  if (s == 12345.678) out[0] = s;        // keeps the chains live; never true in practice
}
}  // namespace

cudaError_t chp_launch_dfma_probe(int blocks, int iters, double* out, cudaStream_t st) {
  k_dfma_probe<<<blocks, 256, 0, st>>>(iters, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Boundary hand-off of the sharded coarse chain (include/chp.h chp_hop).
// ---------------------------------------------------------------------------
namespace {

__global__ void k_hop_put(long long fs, int nic, const double* __restrict__ src, long long src_stride,
                          double* __restrict__ dst, long long dst_stride) {
  const long long total = fs * nic;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / fs, o = t % fs;
    dst[i * dst_stride + o] = src[i * src_stride + o];
  }
  __threadfence_system();
}

// one thread: the changed bytes, then the flag (release, system scope)
__global__ void k_hop_signal(int nic, const unsigned char* changed, long long changed_stride,
                             unsigned char* peer_changed, unsigned int* flag, unsigned int seq) {
  if (changed && peer_changed)
    for (int i = 0; i < nic; ++i) peer_changed[i] = changed[i * changed_stride] & 1;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
}

__global__ void k_hop_take(long long fs, int nic, const double* __restrict__ mail, long long mail_stride,
                           const unsigned char* mail_changed, double* __restrict__ U0,
                           long long ic_stride, unsigned char* changed, long long changed_stride) {
  const long long total = fs * nic;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / fs, o = t % fs;
    const unsigned char c = changed[i * changed_stride];
    if (c & 2) continue;                                   // frozen IC: keeps its boundary
    U0[i * ic_stride + o] = mail[i * mail_stride + o];
    if (o == 0) changed[i * changed_stride] = (unsigned char)((c & 2) | (mail_changed[i] & 1));
  }
}

}  // namespace

cudaError_t chp_launch_hop_put(long long fs, int nic, const double* src, long long src_stride,
                               const unsigned char* changed, long long changed_stride,
                               const chp_hop& hop, cudaStream_t st) {
  if (src) {
    long long blocks = (fs * nic + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_hop_put<<<(int)blocks, 256, 0, st>>>(fs, nic, src, src_stride, hop.peer_u, hop.peer_stride);
  }
  k_hop_signal<<<1, 1, 0, st>>>(nic, changed, changed_stride, hop.peer_changed, hop.peer_flag, hop.seq);
  return cudaGetLastError();
}

cudaError_t chp_launch_hop_take(long long fs, int nic, const double* mail, long long mail_stride,
                                const unsigned char* mail_changed, double* U0, long long ic_stride,
                                unsigned char* changed, long long changed_stride,
                                unsigned int* peer_ack, unsigned int seq, cudaStream_t st) {
  long long blocks = (fs * nic + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_hop_take<<<(int)blocks, 256, 0, st>>>(fs, nic, mail, mail_stride, mail_changed, U0, ic_stride,
                                         changed, changed_stride);
  if (peer_ack) k_hop_signal<<<1, 1, 0, st>>>(0, nullptr, 0, nullptr, peer_ack, seq);
  return cudaGetLastError();
}
