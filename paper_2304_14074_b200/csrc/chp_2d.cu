// 2D propagators (configs 3-5): batched DST-I spectral solves.
//
// Field layout: [m rows (x, i)][pitch = N = m+1 doubles (y, j)], N a power of
// two; column j = m is a zero pad.  All transforms are the unnormalised DST-I
// T (T^2 = (N/2) I) of chp_dst.cuh; the 2D orthonormal transform is
// S = (2/N) T_i T_j, so every normalisation folds into one scale per solve.
//
// LINEAR_B (schemes.py:249-267):  x = S D S rhs,  D = 1/(1 - 2dt lam + eps^2 dt lam^2),
// lam = lam_p + lam_q (grid.py:127-144, sin^2 form).  One step = two passes
// over HBM (32 B per grid-point-step):
//   row pass    (contiguous rows, tile of TR rows + 1 halo row each side):
//               P -> x = T_j P (physical), rhs = x + dt L(x^3 - 3x) (5-point,
//               CSR order of grid.py:110), Q = T_j rhs
//   column pass (tile of TC columns, all rows): P = T_i (D' .* (T_i Q))
// with D' = (2/N)^2 D.  J steps = J+1 row passes + J column passes.
#include <math.h>

#include <map>
#include <string>
#include <vector>

#include "chp_common.cuh"
#include "chp_dst.cuh"

using chpdst::Tables;

namespace {

constexpr int kMinN = 8;
constexpr int kMaxN = 1024;

template <int N> struct Cfg {
  static constexpr int T = (N >= 1024) ? 128 : (N >= 512 ? 64 : 32);  // threads / pair
  static constexpr int G = 4;                                          // pairs / block
  static constexpr int TR = 2 * G - 2;                                 // rows / row tile
  static constexpr int TC = 2 * G;                                     // cols / col tile
  static constexpr int THREADS = G * T;
  static constexpr size_t ROW_SMEM = sizeof(double) * ((size_t)(TR + 2) * N + (size_t)TR * N) +
                                     sizeof(double) * G * (T / 32);
  static constexpr size_t COL_SMEM = sizeof(double) * (size_t)TC * N + sizeof(double) * G * (T / 32);
};

enum RowMode { ROW_FIRST = 0, ROW_MID = 1, ROW_LAST = 2 };

struct RowArgs {
  const double* in;      // P (MID/LAST) or physical U (FIRST) base
  long long in_stride;
  double* out;           // Q (FIRST/MID) or physical result (LAST) base
  long long out_stride;
  const int* in_index;   // system -> field index for `in` (nullable)
  const int* out_index;  // system -> field index for `out` (nullable)
  int m;
  double dt, c1;
  int mode;
  chp_sys_info* info;    // indexed like `in_index`/`out_index` of the physical side
  const int* info_index;
};

// ---------------------------------------------------------------------------
// Row pass
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS)
k2d_row_pass(RowArgs a, Tables tb) {
  using C = Cfg<N>;
  extern __shared__ double sm[];
  double* X = sm;                                // (TR+2) rows, pairs of 2N
  double* R = sm + (size_t)(C::TR + 2) * N;      // TR rows
  double* ws = R + (size_t)C::TR * N;
  const int tid = threadIdx.x;
  const int g = tid / C::T, t = tid % C::T;
  const int s = blockIdx.y;
  const int m = a.m;
  const int i0 = blockIdx.x * C::TR;
  const long long fin = a.in_index ? a.in_index[s] : s;
  const long long fout = a.out_index ? a.out_index[s] : s;
  const double* in = a.in + fin * a.in_stride;
  double* out = a.out + fout * a.out_stride;

  // 1. load rows i0-1 .. i0+TR (zero outside), math index j+1
  for (int idx = tid; idx < (C::TR + 2) * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N;
    const int row = i0 - 1 + r;
    double v = 0.0;
    if (j > 0 && row >= 0 && row < m) v = in[(long long)row * N + (j - 1)];
    X[idx] = v;
  }
  __syncthreads();
  // 2. x = T_j P
  if (a.mode != ROW_FIRST) {
    chpdst::dst_pair<N, C::T>(X + (size_t)g * 2 * N, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
    __syncthreads();
    // non-finite check of the physical state (grid.py:84-85, every step)
    bool bad = false;
    for (int idx = tid; idx < C::TR * N; idx += C::THREADS) {
      const int r = idx / N, j = idx % N;
      if (i0 + r < m && j > 0) bad |= !isfinite(X[(size_t)(r + 1) * N + j]);
    }
    if (__syncthreads_or(bad) && tid == 0) {
      const long long fi = a.info_index ? a.info_index[s] : s;
      atomicCAS(&a.info[fi].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
    }
  }
  if (a.mode == ROW_LAST) {
    for (int idx = tid; idx < C::TR * N; idx += C::THREADS) {
      const int r = idx / N, j = idx % N;
      const int row = i0 + r;
      if (row < m) out[(long long)row * N + j] = (j < m) ? X[(size_t)(r + 1) * N + j + 1] : 0.0;
    }
    return;
  }
  // 3. R = inner rows of x;  X <- w = x^3 - 3x
  for (int idx = tid; idx < C::TR * N; idx += C::THREADS) R[idx] = X[idx + N];
  __syncthreads();
  for (int idx = tid; idx < (C::TR + 2) * N; idx += C::THREADS) {
    const double x = X[idx];
    X[idx] = fma(x, x * x, -3.0 * x);
  }
  __syncthreads();
  // 4. rhs = x + dt * L w  (CSR order: (i-1,j), (i,j-1), (i,j), (i,j+1), (i+1,j))
  const double c = a.c1, c4 = -4.0 * a.c1, dt = a.dt;
  for (int idx = tid; idx < C::TR * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N;
    double v = 0.0;
    if (j > 0) {
      const double* w0 = X + (size_t)(r + 1) * N;
      const double wl = w0[j - 1];                       // j-1 = 0 is the boundary (0)
      const double wr = (j + 1 < N) ? w0[j + 1] : 0.0;
      const double lw = (((X[(size_t)r * N + j] * c + wl * c) + w0[j] * c4) + wr * c) +
                        X[(size_t)(r + 2) * N + j] * c;
      v = R[idx] + dt * lw;
    }
    R[idx] = v;
  }
  __syncthreads();
  // 5. Q = T_j rhs
  if (g < C::G - 1)
    chpdst::dst_pair<N, C::T>(R + (size_t)g * 2 * N, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
  __syncthreads();
  for (int idx = tid; idx < C::TR * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N;
    const int row = i0 + r;
    if (row < m) out[(long long)row * N + j] = (j < m) ? R[(size_t)r * N + j + 1] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Column pass: P = T_i (D' .* T_i Q), in place.
// ---------------------------------------------------------------------------
struct ColArgs {
  double* buf;
  long long stride;
  int m;
  double a2dt, b, scale;   // den = (1 - a2dt*lam) + b*lam^2 ; scale = (2/N)^2
  const double* lam;       // lam[p], p = 1..m (index 0 unused)
};

template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS)
k2d_col_pass_b(ColArgs a, Tables tb) {
  using C = Cfg<N>;
  extern __shared__ double sm[];
  double* ws = sm + (size_t)C::TC * N;
  const int tid = threadIdx.x;
  const int g = tid / C::T, t = tid % C::T;
  const int s = blockIdx.y;
  const int m = a.m;
  const int j0 = blockIdx.x * C::TC;
  double* buf = a.buf + (long long)s * a.stride;
  // load: column c -> sm[c*N + i + 1]
  for (int idx = tid; idx < m * C::TC; idx += C::THREADS) {
    const int i = idx / C::TC, c = idx % C::TC;
    sm[(size_t)c * N + i + 1] = (j0 + c < m) ? buf[(long long)i * N + j0 + c] : 0.0;
  }
  if (tid < C::TC) sm[(size_t)tid * N] = 0.0;
  __syncthreads();
  double* pr = sm + (size_t)g * 2 * N;
  chpdst::dst_pair<N, C::T>(pr, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
  // scale by D' (each group scales its own pair)
  for (int idx = t; idx < 2 * N; idx += C::T) {
    const int c = 2 * g + idx / N, p = idx % N;
    const int q = j0 + c + 1;
    if (p > 0 && q <= m) {
      const double lam = a.lam[p] + a.lam[q];
      const double den = (1.0 - a.a2dt * lam) + a.b * (lam * lam);
      pr[idx] = pr[idx] * (a.scale / den);
    }
  }
  chpdst::group_sync(g + 1, C::T);
  chpdst::dst_pair<N, C::T>(pr, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
  __syncthreads();
  for (int idx = tid; idx < m * C::TC; idx += C::THREADS) {
    const int i = idx / C::TC, c = idx % C::TC;
    if (j0 + c < m) buf[(long long)i * N + j0 + c] = sm[(size_t)c * N + i + 1];
  }
}

// ---------------------------------------------------------------------------
// Variable-coefficient 2D solves (LINEAR_A, Newton Jacobian): matrix-free PCG
//
//   (I - a L diag(c) + b L^2) x = rhs,   L = -K (K SPD),  B = bK + a diag(c)
//   => (K^-1 + B) x = K^-1 rhs   (SPD)
// solved in the orthonormal DST basis (x^ = S x):
//   A^ x^ = d .* x^ + a S(c .* S x^),   d = 1/kappa + b kappa,  kappa = -(lam_p+lam_q)
//   b^ = (1/kappa) .* S rhs,   preconditioner M = d + a*mean(c)
// Each CG iteration is 3 transform passes (row T_j, column T_i*c*T_i, row T_j)
// plus two vector updates; every dot product is a fixed-order two-level
// reduction (block partials -> one warp per system), so results are bitwise
// reproducible run to run (determinism rule).
// ---------------------------------------------------------------------------

struct CgSys {
  double rho, rr0, rr, alpha, beta, acbar, pq, pad;
  int iters, done, active, fail;
};

constexpr int kPB = 64;   // partial-sum blocks per system for elementwise kernels

// generic row pass: out = T_j in (tile of 2G rows, no halo)
//   op 0: out = scale * T_j in
//   op 1 (CG q): out = d .* p + T_j in ; partial[s][tile] = sum p*q
struct RowDst {
  const double* in; double* out; long long stride;
  int m, op; double scale;
  const double* p; const double* lam; double b;
  double* partial; int nparts;
  const CgSys* cg; int skip_done;
};

template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS)
k2d_rowdst(RowDst a, Tables tb) {
  using C = Cfg<N>;
  constexpr int TRg = 2 * C::G;
  extern __shared__ double sm[];
  double* ws = sm + (size_t)TRg * N;
  const int tid = threadIdx.x, g = tid / C::T, t = tid % C::T;
  const int s = blockIdx.y, m = a.m;
  if (a.cg && (!a.cg[s].active || (a.skip_done && a.cg[s].done))) return;
  const int i0 = blockIdx.x * TRg;
  const double* in = a.in + (long long)s * a.stride;
  double* out = a.out + (long long)s * a.stride;
  for (int idx = tid; idx < TRg * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N, row = i0 + r;
    sm[idx] = (j > 0 && row < m) ? in[(long long)row * N + j - 1] : 0.0;
  }
  __syncthreads();
  chpdst::dst_pair<N, C::T>(sm + (size_t)g * 2 * N, tb, a.scale, ws + g * (C::T / 32), t, g + 1);
  __syncthreads();
  double part = 0.0;
  for (int idx = tid; idx < TRg * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N, row = i0 + r;
    if (row >= m) continue;
    double v = (j < m) ? sm[(size_t)r * N + j + 1] : 0.0;
    if (a.op == 1 && j < m) {
      const double kap = -(a.lam[row + 1] + a.lam[j + 1]);
      const double d = 1.0 / kap + a.b * kap;
      const double pv = a.p[(long long)s * a.stride + (long long)row * N + j];
      v = fma(d, pv, v);
      part = fma(pv, v, part);
    }
    out[(long long)row * N + j] = v;
  }
  if (a.op == 1) {
    // fixed-shape block reduction
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __syncthreads();
    if ((tid & 31) == 0) ws[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < C::THREADS / 32; ++w) tot += ws[w];
      a.partial[(long long)s * a.nparts + blockIdx.x] = tot;
    }
  }
}

// generic column pass (tile of TC columns, in -> out, in place allowed)
//   op 0: out = scale * T_i in
//   op 1: out = T_i ( (scale * c[i][j]) .* T_i in )        (CG operator)
//   op 2: out = T_i in .* (scale / kappa)                   (b^ = K^-1 rhs)
struct ColDst {
  const double* in; double* out; long long stride;
  int m, op; double scale;
  const double* c; const double* lam;
  const CgSys* cg; int skip_done;
};

template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS)
k2d_coldst(ColDst a, Tables tb) {
  using C = Cfg<N>;
  extern __shared__ double sm[];
  double* ws = sm + (size_t)C::TC * N;
  const int tid = threadIdx.x, g = tid / C::T, t = tid % C::T;
  const int s = blockIdx.y, m = a.m;
  if (a.cg && (!a.cg[s].active || (a.skip_done && a.cg[s].done))) return;
  const int j0 = blockIdx.x * C::TC;
  const double* in = a.in + (long long)s * a.stride;
  double* out = a.out + (long long)s * a.stride;
  for (int idx = tid; idx < m * C::TC; idx += C::THREADS) {
    const int i = idx / C::TC, c = idx % C::TC;
    sm[(size_t)c * N + i + 1] = (j0 + c < m) ? in[(long long)i * N + j0 + c] : 0.0;
  }
  if (tid < C::TC) sm[(size_t)tid * N] = 0.0;
  __syncthreads();
  double* pr = sm + (size_t)g * 2 * N;
  chpdst::dst_pair<N, C::T>(pr, tb, a.op == 0 ? a.scale : 1.0, ws + g * (C::T / 32), t, g + 1);
  if (a.op == 1) {
    const double* cs = a.c + (long long)s * a.stride;
    for (int idx = t; idx < 2 * N; idx += C::T) {
      const int c = 2 * g + idx / N, p = idx % N, q = j0 + c;
      if (p > 0 && q < m) pr[idx] *= a.scale * cs[(long long)(p - 1) * N + q];
    }
    chpdst::group_sync(g + 1, C::T);
    chpdst::dst_pair<N, C::T>(pr, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
  } else if (a.op == 2) {
    for (int idx = t; idx < 2 * N; idx += C::T) {
      const int c = 2 * g + idx / N, p = idx % N, q = j0 + c + 1;
      if (p > 0 && q <= m) pr[idx] *= a.scale / (-(a.lam[p] + a.lam[q]));
    }
  }
  __syncthreads();
  for (int idx = tid; idx < m * C::TC; idx += C::THREADS) {
    const int i = idx / C::TC, c = idx % C::TC;
    if (j0 + c < m) out[(long long)i * N + j0 + c] = sm[(size_t)c * N + i + 1];
  }
}

// ---- elementwise kernels over one field per system (grid: kPB x nsys) -----
template <class F>
CHP_DEV void for_points(int m, int N, F f) {
  const long long total = (long long)m * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / m), j = (int)(t % m);
    f(i, j, (long long)i * N + j);
  }
}

CHP_DEV double block_sum(double v, double* ws) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ws[w];
  return tot;
}

CHP_DEV double at(const double* f, int i, int j, int m, int N) {
  return (i >= 0 && i < m && j >= 0 && j < m) ? f[(long long)i * N + j] : 0.0;
}

// 5-point L in the CSR order of grid.py:110 (rows (i-1,j),(i,j-1),(i,j),(i,j+1),(i+1,j))
CHP_DEV double lap5(const double* f, int i, int j, int m, int N, double c) {
  return ((((at(f, i - 1, j, m, N) * c + at(f, i, j - 1, m, N) * c) +
            f[(long long)i * N + j] * (-4.0 * c)) + at(f, i, j + 1, m, N) * c) +
          at(f, i + 1, j, m, N) * c);
}

CHP_DEV double cube_at(const double* f, int i, int j, int m, int N) {
  const double v = at(f, i, j, m, N);
  return v * v * v;
}

CHP_DEV double lap5_cube(const double* f, int i, int j, int m, int N, double c) {
  return ((((cube_at(f, i - 1, j, m, N) * c + cube_at(f, i, j - 1, m, N) * c) +
            cube_at(f, i, j, m, N) * (-4.0 * c)) + cube_at(f, i, j + 1, m, N) * c) +
          cube_at(f, i + 1, j, m, N) * c);
}

struct Pt {
  int m, N; long long stride; double c1;
  const int* src_index; const int* dst_index;
};

// LINEAR_A prep: rhs = v - dt L v, c = v^2 (schemes.py:244-245); sum c -> partial
__global__ void k2d_prep_a(Pt pt, const double* src, long long src_stride, double* rhs,
                           double* cc, double dt, CgSys* cg, double* partial) {
  __shared__ double ws[32];
  const int s = blockIdx.y;
  if (!cg[s].active) return;
  const long long fi = pt.src_index ? pt.src_index[s] : s;
  const double* v = src + fi * src_stride;
  double* r = rhs + (long long)s * pt.stride;
  double* c = cc + (long long)s * pt.stride;
  double acc = 0.0;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    const double x = v[o];
    r[o] = x - dt * lap5(v, i, j, pt.m, pt.N, pt.c1);
    c[o] = x * x;
    acc += x * x;
  });
  const double tot = block_sum(acc, ws);
  if (threadIdx.x == 0) partial[(long long)s * kPB + blockIdx.x] = tot;
}

// Newton: yhat = u - d L u ; y = u
__global__ void k2d_newton_init(Pt pt, const double* src, long long src_stride, double* yhat,
                                double* y, long long y_stride, double d, const int* act,
                                int do_copy) {
  const int s = blockIdx.y;
  if (act && !act[s]) return;
  const long long fi = pt.src_index ? pt.src_index[s] : s;
  const long long fo = pt.dst_index ? pt.dst_index[s] : s;
  const double* u = src + fi * src_stride;
  double* yh = yhat + (long long)s * pt.stride;
  double* yy = y + fo * y_stride;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    yh[o] = u[o] - d * lap5(u, i, j, pt.m, pt.N, pt.c1);
  });
  if (do_copy)   // src != y (when they alias, y already holds u)
    for_points(pt.m, pt.N, [&](int i, int j, long long o) { yy[o] = u[o]; });
}

// Newton residual part 1: t1 = L y, t2 = L(y^3)
__global__ void k2d_newton_t(Pt pt, const double* y, long long y_stride, double* t1, double* t2,
                             const int* act) {
  const int s = blockIdx.y;
  if (act && !act[s]) return;
  const long long fo = pt.dst_index ? pt.dst_index[s] : s;
  const double* yy = y + fo * y_stride;
  double* a1 = t1 + (long long)s * pt.stride;
  double* a2 = t2 + (long long)s * pt.stride;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    a1[o] = lap5(yy, i, j, pt.m, pt.N, pt.c1);
    a2[o] = lap5_cube(yy, i, j, pt.m, pt.N, pt.c1);
  });
}

// Newton residual part 2: H = y + b L t1 - d t2 - yhat (schemes.py:288); partial sum H^2;
// also rhs = yhat - 2d t2, c = y^2 (schemes.py:303-304)
__global__ void k2d_newton_h(Pt pt, const double* y, long long y_stride, const double* t1,
                             const double* t2, const double* yhat, double* rhs, double* cc,
                             double b, double d, const int* act, double* partial,
                             double* partial_c) {
  __shared__ double ws[32];
  const int s = blockIdx.y;
  if (act && !act[s]) return;
  const long long fo = pt.dst_index ? pt.dst_index[s] : s;
  const double* yy = y + fo * y_stride;
  const double* a1 = t1 + (long long)s * pt.stride;
  const double* a2 = t2 + (long long)s * pt.stride;
  const double* yh = yhat + (long long)s * pt.stride;
  double* r = rhs + (long long)s * pt.stride;
  double* c = cc + (long long)s * pt.stride;
  double acc = 0.0, accc = 0.0;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    const double yv = yy[o];
    const double H = ((yv + b * lap5(a1, i, j, pt.m, pt.N, pt.c1)) - d * a2[o]) - yh[o];
    acc += H * H;
    r[o] = yh[o] - (2.0 * d) * a2[o];
    c[o] = yv * yv;
    accc += yv * yv;
  });
  const double tot = block_sum(acc, ws);
  if (threadIdx.x == 0) partial[(long long)s * kPB + blockIdx.x] = tot;
  const double totc = block_sum(accc, ws);
  if (threadIdx.x == 0) partial_c[(long long)s * kPB + blockIdx.x] = totc;
}

// fixed-order reduction of nparts partials per system (one warp per system)
CHP_DEV double warp_reduce_parts(const double* p, int n) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int k = lane; k < n; k += 32) v += p[k];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CG init: x = 0, r = b^ (in r already), p = r / M; partials rho, rr
__global__ void k2d_cg_init(Pt pt, double* x, double* r, double* p, const double* lam, double b,
                            CgSys* cg, double* partial) {
  __shared__ double ws[32];
  const int s = blockIdx.y;
  if (!cg[s].active) return;
  const double acb = cg[s].acbar;
  double* xs = x + (long long)s * pt.stride;
  double* rs = r + (long long)s * pt.stride;
  double* ps = p + (long long)s * pt.stride;
  double a1 = 0.0, a2 = 0.0;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    const double kap = -(lam[i + 1] + lam[j + 1]);
    const double M = (1.0 / kap + b * kap) + acb;
    const double rv = rs[o];
    xs[o] = 0.0;
    const double z = rv / M;
    ps[o] = z;
    a1 = fma(rv, z, a1);
    a2 = fma(rv, rv, a2);
  });
  const double t1 = block_sum(a1, ws);
  if (threadIdx.x == 0) partial[((long long)s * kPB + blockIdx.x) * 2] = t1;
  const double t2 = block_sum(a2, ws);
  if (threadIdx.x == 0) partial[((long long)s * kPB + blockIdx.x) * 2 + 1] = t2;
}

// reductions producing CG scalars; mode: 0 = after init, 1 = alpha, 2 = beta
__global__ void k2d_cg_reduce(int nsys, CgSys* cg, const double* partial, int nparts, int mode,
                              double tol2, int max_iter, double inv_count, double a_coef) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nsys) return;
  CgSys& q = cg[s];
  if (!q.active || (mode != 3 && q.done)) return;
  const int lane = threadIdx.x & 31;
  if (mode == 3) {         // mean(c) -> acbar
    const double tot = warp_reduce_parts(partial + (long long)s * nparts, nparts);
    if (lane == 0) { q.acbar = a_coef * (tot * inv_count); q.done = 0; q.iters = 0; q.fail = 0; }
    return;
  }
  if (mode == 1) {
    const double pq = warp_reduce_parts(partial + (long long)s * nparts, nparts);
    if (lane == 0) { q.pq = pq; q.alpha = q.rho / pq; }
    return;
  }
  // modes 0 and 2: interleaved (rho, rr) partials
  double v1 = 0.0, v2 = 0.0;
  const double* p = partial + (long long)s * nparts * 2;
  for (int k = lane; k < nparts; k += 32) { v1 += p[2 * k]; v2 += p[2 * k + 1]; }
  for (int o = 16; o > 0; o >>= 1) {
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  if (lane != 0) return;
  if (mode == 0) {
    q.rho = v1; q.rr0 = v2; q.rr = v2; q.iters = 0;
    q.done = (v2 == 0.0) ? 1 : 0;
  } else {
    q.beta = v1 / q.rho;
    q.rho = v1;
    q.rr = v2;
    q.iters += 1;
    if (!(v2 > tol2 * q.rr0)) q.done = 1;           // also stops on NaN
    else if (q.iters >= max_iter) { q.done = 1; q.fail = 1; }
    if (!isfinite(v2)) q.fail = 1;
  }
}

// x += alpha p ; r -= alpha q ; partials rho' = r.z, rr = r.r (z = r/M)
__global__ void k2d_cg_update1(Pt pt, double* x, double* r, const double* p, const double* qv,
                               const double* lam, double b, CgSys* cg, double* partial) {
  __shared__ double ws[32];
  const int s = blockIdx.y;
  if (!cg[s].active || cg[s].done) return;
  const double al = cg[s].alpha, acb = cg[s].acbar;
  double* xs = x + (long long)s * pt.stride;
  double* rs = r + (long long)s * pt.stride;
  const double* ps = p + (long long)s * pt.stride;
  const double* qs = qv + (long long)s * pt.stride;
  double a1 = 0.0, a2 = 0.0;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    xs[o] = fma(al, ps[o], xs[o]);
    const double rv = fma(-al, qs[o], rs[o]);
    rs[o] = rv;
    const double kap = -(lam[i + 1] + lam[j + 1]);
    const double M = (1.0 / kap + b * kap) + acb;
    a1 = fma(rv, rv / M, a1);
    a2 = fma(rv, rv, a2);
  });
  const double t1 = block_sum(a1, ws);
  if (threadIdx.x == 0) partial[((long long)s * kPB + blockIdx.x) * 2] = t1;
  const double t2 = block_sum(a2, ws);
  if (threadIdx.x == 0) partial[((long long)s * kPB + blockIdx.x) * 2 + 1] = t2;
}

// p = r/M + beta p
__global__ void k2d_cg_update2(Pt pt, const double* r, double* p, const double* lam, double b,
                               const CgSys* cg) {
  const int s = blockIdx.y;
  if (!cg[s].active || cg[s].done) return;
  const double be = cg[s].beta, acb = cg[s].acbar;
  const double* rs = r + (long long)s * pt.stride;
  double* ps = p + (long long)s * pt.stride;
  for_points(pt.m, pt.N, [&](int i, int j, long long o) {
    const double kap = -(lam[i + 1] + lam[j + 1]);
    const double M = (1.0 / kap + b * kap) + acb;
    ps[o] = fma(be, ps[o], rs[o] / M);
  });
}

// scatter the solution (written in a compact buffer) to the destination fields and check finiteness
__global__ void k2d_scatter(Pt pt, const double* x, double* dst, long long dst_stride,
                            const CgSys* cg, chp_sys_info* info, const int* info_index) {
  const int s = blockIdx.y;
  if (!cg[s].active) return;
  const long long fo = pt.dst_index ? pt.dst_index[s] : s;
  const double* xs = x + (long long)s * pt.stride;
  double* d = dst + fo * dst_stride;
  bool bad = false;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)pt.m * pt.N;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t % pt.N);
    const double v = (j < pt.m) ? xs[t] : 0.0;
    d[t] = v;
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    const long long fi = info_index ? info_index[s] : s;
    atomicCAS(&info[fi].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
  }
}

// coarse-sweep correction for slice n (2D): U[n+1] = (g + F[n]) - G[n]; G[n] = g
__global__ void k2d_correct(int m, int N, double* U, const double* F, double* G, const double* gb,
                            long long gb_stride, long long ic_stride, long long sl_stride, int n,
                            int nsl, unsigned char* changed, double* inc, int mode,
                            chp_sys_info* info) {
  __shared__ double ws[32];
  const int i = blockIdx.y;
  unsigned char* ch = changed ? changed + (long long)i * (nsl + 1) : nullptr;
  if (mode == 1 && (ch[0] & 2)) return;
  double* un1 = U + i * ic_stride + (long long)(n + 1) * sl_stride;
  double* gn = G + i * ic_stride + (long long)n * sl_stride;
  const double* g = gb + (long long)i * gb_stride;
  const double* fn = F ? F + i * ic_stride + (long long)n * sl_stride : nullptr;
  double dmax = 0.0;
  int any = 0;
  bool bad = false;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * N;
       t += (long long)gridDim.x * blockDim.x) {
    const double gv = g[t];
    if (mode == 0) {
      un1[t] = gv;
      gn[t] = gv;
      continue;
    }
    const double nv = (gv + fn[t]) - gn[t];
    const double ov = un1[t];
    any |= (__double_as_longlong(nv) != __double_as_longlong(ov));
    dmax = fmax(dmax, fabs(nv - ov));
    bad |= !isfinite(nv);
    un1[t] = nv;
    gn[t] = gv;
  }
  if (mode == 0) return;
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(inc + i, dmax);
  if (__syncthreads_or(any) && threadIdx.x == 0) ch[n + 1] = 1;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(&info[i].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
  (void)ws;
}

__global__ void k2d_set_active(CgSys* cg, int nsys, const int* act) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsys) { cg[s].active = act ? act[s] : 1; cg[s].done = 0; cg[s].fail = 0; cg[s].iters = 0; }
}

__global__ void k2d_cg_collect(int nsys, const CgSys* cg, chp_sys_info* info, const int* info_index) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys || !cg[s].active) return;
  const long long fi = info_index ? info_index[s] : s;
  info[fi].cg_total += cg[s].iters;
  info[fi].cg_max = max(info[fi].cg_max, cg[s].iters);
  if (cg[s].fail) atomicCAS(&info[fi].status, CHP_SYS_OK, CHP_SYS_CG);
}

__global__ void k2d_newton_norm(int nsys, const double* partial, double hd, double* res,
                                const int* act) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nsys || (act && !act[s])) return;
  const double tot = warp_reduce_parts(partial + (long long)s * kPB, kPB);
  if ((threadIdx.x & 31) == 0) res[s] = sqrt(hd * tot);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct NTables {
  double2* tw = nullptr;
  double* sj = nullptr;
  double* lam = nullptr;   // per-axis eigenvalues, index p = 1..m
};

struct Work2 {            // device workspace for one solve batch
  double *X, *Rv, *Pv, *Yv, *Cv, *RHS, *T1, *T2, *YH;
  double* partial;        // nsys * kPB * 2
  CgSys* cg;
  int* act;               // nsys
  double* res;            // nsys
  double* gbuf;           // coarse: nsys fields
};

template <int N>
void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k2d_row_pass<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<N>::ROW_SMEM);
  cudaFuncSetAttribute(k2d_col_pass_b<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<N>::COL_SMEM);
  cudaFuncSetAttribute(k2d_rowdst<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double) * (2 * Cfg<N>::G * N + Cfg<N>::G * (Cfg<N>::T / 32))));
  cudaFuncSetAttribute(k2d_coldst<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<N>::COL_SMEM);
  done = true;
}

template <int N>
cudaError_t run_linear_b(const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                         const double* in, long long in_stride, double* out, long long out_stride,
                         const int* sys_index, chp_sys_info* info, const NTables& nt,
                         double* scratch, cudaStream_t st) {
  using C = Cfg<N>;
  set_smem_attrs<N>();
  const Tables tb{nt.tw, nt.sj};
  const int m = g.m;
  const long long fs = (long long)m * N;
  double* buf[2] = {scratch, scratch + fs * nsys};
  const dim3 rgrid((m + C::TR - 1) / C::TR, nsys), cgrid((m + C::TC - 1) / C::TC, nsys);
  ColArgs ca{nullptr, fs, m, 2.0 * sp.dt, sp.b, (2.0 / N) * (2.0 / N), nt.lam};
  for (int s = 0; s < steps; ++s) {
    RowArgs ra{};
    ra.m = m; ra.dt = sp.dt; ra.c1 = g.c1; ra.info = info; ra.info_index = sys_index;
    if (s == 0) {
      ra.in = in; ra.in_stride = in_stride; ra.in_index = sys_index; ra.mode = ROW_FIRST;
    } else {
      ra.in = buf[(s - 1) & 1]; ra.in_stride = fs; ra.in_index = nullptr; ra.mode = ROW_MID;
    }
    ra.out = buf[s & 1]; ra.out_stride = fs; ra.out_index = nullptr;
    k2d_row_pass<N><<<rgrid, C::THREADS, C::ROW_SMEM, st>>>(ra, tb);
    ca.buf = buf[s & 1];
    k2d_col_pass_b<N><<<cgrid, C::THREADS, C::COL_SMEM, st>>>(ca, tb);
  }
  RowArgs ra{};
  ra.m = m; ra.dt = sp.dt; ra.c1 = g.c1; ra.info = info; ra.info_index = sys_index;
  ra.in = buf[(steps - 1) & 1]; ra.in_stride = fs; ra.in_index = nullptr; ra.mode = ROW_LAST;
  ra.out = out; ra.out_stride = out_stride; ra.out_index = sys_index;
  k2d_row_pass<N><<<rgrid, C::THREADS, C::ROW_SMEM, st>>>(ra, tb);
  return cudaGetLastError();
}

// PCG solve of (I - a L diag(c) + b L^2) x = RHS for every active system.
// Inputs in W.RHS, W.Cv (physical, compact per system) and W.cg[s].active;
// the solution is left in W.Yv (physical).  Host-synchronising every
// `chunk` iterations to test completion.
template <int N>
cudaError_t pcg_solve(const chp_grid& g, int nsys, double a, double b, double tol, int max_iter,
                      const NTables& nt, Work2& W, cudaStream_t st) {
  using C = Cfg<N>;
  set_smem_attrs<N>();
  const Tables tb{nt.tw, nt.sj};
  const int m = g.m;
  const long long fs = (long long)m * N;
  const int rtiles = (m + 2 * C::G - 1) / (2 * C::G);
  const dim3 rgrid(rtiles, nsys), cgrid((m + C::TC - 1) / C::TC, nsys), egrid(kPB, nsys);
  const size_t rsm = sizeof(double) * (2 * C::G * N + C::G * (C::T / 32));
  const Pt pt{m, N, fs, g.c1, nullptr, nullptr};
  const int red_blocks = (nsys + 7) / 8;
  const double s2 = (2.0 / N) * (2.0 / N);
  // mean(c): partials were produced by the prep kernel into W.partial (kPB per system)
  k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 3, 0, 0,
                                           1.0 / ((double)m * m), a);
  // b^ = (2/N)^2 / kappa .* T_i T_j rhs  -> Rv
  RowDst r0{W.RHS, W.Yv, fs, m, 0, 1.0, nullptr, nt.lam, b, nullptr, 0, W.cg, 0};
  k2d_rowdst<N><<<rgrid, C::THREADS, rsm, st>>>(r0, tb);
  ColDst c0{W.Yv, W.Rv, fs, m, 2, 2.0 / N, nullptr, nt.lam, W.cg, 0};   // S = (2/N) T_i T_j
  k2d_coldst<N><<<cgrid, C::THREADS, C::COL_SMEM, st>>>(c0, tb);
  k2d_cg_init<<<egrid, 256, 0, st>>>(pt, W.X, W.Rv, W.Pv, nt.lam, b, W.cg, W.partial);
  k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 0, 0, 0, 0, 0);
  const int chunk = 8;
  std::vector<CgSys> host(nsys);
  for (int it0 = 0; it0 < max_iter + chunk; it0 += chunk) {
    for (int it = 0; it < chunk; ++it) {
      RowDst r1{W.Pv, W.Yv, fs, m, 0, 1.0, nullptr, nt.lam, b, nullptr, 0, W.cg, 1};
      k2d_rowdst<N><<<rgrid, C::THREADS, rsm, st>>>(r1, tb);
      ColDst c1{W.Yv, W.Yv, fs, m, 1, a * s2, W.Cv, nt.lam, W.cg, 1};
      k2d_coldst<N><<<cgrid, C::THREADS, C::COL_SMEM, st>>>(c1, tb);
      RowDst r2{W.Yv, W.Yv, fs, m, 1, 1.0, W.Pv, nt.lam, b, W.partial, rtiles, W.cg, 1};
      k2d_rowdst<N><<<rgrid, C::THREADS, rsm, st>>>(r2, tb);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, rtiles, 1, 0, 0, 0, 0);
      k2d_cg_update1<<<egrid, 256, 0, st>>>(pt, W.X, W.Rv, W.Pv, W.Yv, nt.lam, b, W.cg,
                                            W.partial);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 2, tol * tol,
                                               max_iter, 0, 0);
      k2d_cg_update2<<<egrid, 256, 0, st>>>(pt, W.Rv, W.Pv, nt.lam, b, W.cg);
    }
    cudaError_t e = cudaMemcpyAsync(host.data(), W.cg, sizeof(CgSys) * nsys,
                                    cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    bool all = true;
    for (int s = 0; s < nsys; ++s) all = all && (!host[s].active || host[s].done);
    if (all) break;
  }
  // x = (2/N) T_i T_j x^  -> Yv.  ("done" systems must still be finalised)
  RowDst r3{W.X, W.Yv, fs, m, 0, 1.0, nullptr, nt.lam, b, nullptr, 0, W.cg, 0};
  k2d_rowdst<N><<<rgrid, C::THREADS, rsm, st>>>(r3, tb);
  ColDst c3{W.Yv, W.Yv, fs, m, 0, 2.0 / N, nullptr, nt.lam, W.cg, 0};
  k2d_coldst<N><<<cgrid, C::THREADS, C::COL_SMEM, st>>>(c3, tb);
  return cudaGetLastError();
}

__global__ void k2d_clear_flag(unsigned char* changed, int nic, int nsl, int slot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nic && !(changed[(long long)i * (nsl + 1)] & 2)) changed[(long long)i * (nsl + 1) + slot] = 0;
}

// add host-side Newton aggregates into the device sysinfo records
struct NewtonRec { long long steps, total; int maxit, status, fail_iter, pad; double maxres, fail_res; };
__global__ void k2d_newton_commit(int nsys, const NewtonRec* rec, chp_sys_info* info,
                                  const int* info_index) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  const long long fi = info_index ? info_index[s] : s;
  chp_sys_info& q = info[fi];
  q.newton_steps += rec[s].steps;
  q.newton_total += rec[s].total;
  q.newton_max = max(q.newton_max, rec[s].maxit);
  q.newton_maxres = fmax(q.newton_maxres, rec[s].maxres);
  if (rec[s].status != CHP_SYS_OK && q.status == CHP_SYS_OK) {
    q.status = rec[s].status;
    q.fail_iter = rec[s].fail_iter;
    q.fail_resid = rec[s].fail_res;
  }
}

}  // namespace

struct Chp2d {
  std::map<int, NTables> tables;
  double* scratch = nullptr;      // LINEAR_B ping-pong fields
  size_t scratch_bytes = 0;
  void* work = nullptr;           // PCG / Newton workspace
  size_t work_bytes = 0;
  int* host_act = nullptr;        // pinned
  double* host_res = nullptr;     // pinned
  NewtonRec* host_rec = nullptr;  // pinned
  int host_cap = 0;
};

Chp2d* chp2d_create() { return new Chp2d(); }

void chp2d_destroy(Chp2d* c) {
  if (!c) return;
  for (auto& kv : c->tables) {
    cudaFree(kv.second.tw);
    cudaFree(kv.second.sj);
    cudaFree(kv.second.lam);
  }
  if (c->scratch) cudaFree(c->scratch);
  if (c->work) cudaFree(c->work);
  if (c->host_act) cudaFreeHost(c->host_act);
  if (c->host_res) cudaFreeHost(c->host_res);
  if (c->host_rec) cudaFreeHost(c->host_rec);
  delete c;
}

namespace {

cudaError_t get_tables(Chp2d* c, int N, const NTables** out) {
  auto it = c->tables.find(N);
  if (it != c->tables.end()) { *out = &it->second; return cudaSuccess; }
  std::vector<double2> tw(N);
  std::vector<double> sj(N + 1), lam(N);
  const long double pi = 3.14159265358979323846264338327950288L;
  for (int k = 0; k < N; ++k) {
    const long double ang = -2.0L * pi * k / N;
    tw[k] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  for (int j = 0; j <= N; ++j) sj[j] = (double)sinl(pi * j / N);
  const long double h = 1.0L / N;
  lam[0] = 0.0;
  for (int p = 1; p < N; ++p) {
    const long double sp = sinl(pi * p / (2.0L * N));
    lam[p] = (double)(-4.0L / (h * h) * sp * sp);
  }
  NTables t;
  cudaError_t e;
  if ((e = cudaMalloc(&t.tw, sizeof(double2) * N)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.sj, sizeof(double) * (N + 1))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.lam, sizeof(double) * N)) != cudaSuccess) return e;
  cudaMemcpy(t.tw, tw.data(), sizeof(double2) * N, cudaMemcpyHostToDevice);
  cudaMemcpy(t.sj, sj.data(), sizeof(double) * (N + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(t.lam, lam.data(), sizeof(double) * N, cudaMemcpyHostToDevice);
  c->tables[N] = t;
  *out = &c->tables[N];
  return cudaSuccess;
}

cudaError_t grow(void** p, size_t* have, size_t bytes, cudaStream_t st) {
  if (bytes <= *have) return cudaSuccess;
  if (*p) {
    cudaStreamSynchronize(st);
    cudaFree(*p);
    *p = nullptr;
    *have = 0;
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) *have = bytes;
  return e;
}

cudaError_t host_bufs(Chp2d* c, int n) {
  if (n <= c->host_cap) return cudaSuccess;
  if (c->host_act) cudaFreeHost(c->host_act);
  if (c->host_res) cudaFreeHost(c->host_res);
  if (c->host_rec) cudaFreeHost(c->host_rec);
  cudaError_t e;
  if ((e = cudaMallocHost(&c->host_act, sizeof(int) * n)) != cudaSuccess) return e;
  if ((e = cudaMallocHost(&c->host_res, sizeof(double) * n)) != cudaSuccess) return e;
  if ((e = cudaMallocHost(&c->host_rec, sizeof(NewtonRec) * n)) != cudaSuccess) return e;
  c->host_cap = n;
  return cudaSuccess;
}

// Carve the PCG/Newton workspace for nsys systems (+ nic coarse buffers).
cudaError_t get_work(Chp2d* c, long long fs, int nsys, Work2* W, cudaStream_t st) {
  const size_t fields = 10;
  const size_t bytes = sizeof(double) * fs * nsys * fields + sizeof(double) * nsys * kPB * 4 +
                       sizeof(CgSys) * nsys + sizeof(int) * nsys + sizeof(double) * nsys + 1024;
  cudaError_t e = grow(&c->work, &c->work_bytes, bytes, st);
  if (e != cudaSuccess) return e;
  double* b = static_cast<double*>(c->work);
  const long long F = fs * nsys;
  W->X = b; W->Rv = b + F; W->Pv = b + 2 * F; W->Yv = b + 3 * F; W->Cv = b + 4 * F;
  W->RHS = b + 5 * F; W->T1 = b + 6 * F; W->T2 = b + 7 * F; W->YH = b + 8 * F;
  W->gbuf = b + 9 * F;
  W->partial = b + 10 * F;
  W->cg = reinterpret_cast<CgSys*>(W->partial + (long long)nsys * kPB * 4);
  W->act = reinterpret_cast<int*>(W->cg + nsys);
  W->res = reinterpret_cast<double*>(((uintptr_t)(W->act + nsys) + 15) & ~(uintptr_t)15);
  return host_bufs(c, nsys);
}

// J steps of LINEAR_A (PCG per step) or NONLINEAR_EYRE (Newton + PCG).
template <int N>
cudaError_t run_variable(Chp2d* cx, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                         const double* in, long long in_stride, double* out,
                         long long out_stride, const int* sys_index, chp_sys_info* info,
                         const NTables& nt, Work2& W, cudaStream_t st) {
  const int m = g.m;
  const long long fs = (long long)m * N;
  const dim3 egrid(kPB, nsys);
  const int sb = (nsys + 127) / 128;
  const double tol = sp.cg_tol;
  const int maxcg = sp.cg_max_iter;
  cudaError_t e;
  if (sp.scheme == CHP_LINEAR_A) {
    for (int s = 0; s < steps; ++s) {
      const double* src = (s == 0) ? in : out;
      const long long sst = (s == 0) ? in_stride : out_stride;
      Pt pt{m, N, fs, g.c1, sys_index, sys_index};
      k2d_set_active<<<sb, 128, 0, st>>>(W.cg, nsys, nullptr);
      k2d_prep_a<<<egrid, 256, 0, st>>>(pt, src, sst, W.RHS, W.Cv, sp.dt, W.cg, W.partial);
      if ((e = pcg_solve<N>(g, nsys, sp.dt, sp.b, tol, maxcg, nt, W, st)) != cudaSuccess) return e;
      k2d_scatter<<<egrid, 256, 0, st>>>(pt, W.Yv, out, out_stride, W.cg, info, sys_index);
      k2d_cg_collect<<<sb, 128, 0, st>>>(nsys, W.cg, info, sys_index);
    }
    return cudaGetLastError();
  }
  // ---- Newton (schemes.py:270-305) ----
  const double d = sp.dt, b = sp.b;
  NewtonRec* rec = cx->host_rec;
  int* hact = cx->host_act;
  double* hres = cx->host_res;
  for (int s = 0; s < nsys; ++s) rec[s] = NewtonRec{0, 0, 0, CHP_SYS_OK, 0, 0, 0.0, 0.0};
  std::vector<int> alive(nsys, 1);
  for (int step = 0; step < steps; ++step) {
    const double* src = (step == 0) ? in : out;
    const long long sst = (step == 0) ? in_stride : out_stride;
    Pt pt{m, N, fs, g.c1, sys_index, sys_index};
    for (int s = 0; s < nsys; ++s) hact[s] = alive[s];
    cudaMemcpyAsync(W.act, hact, sizeof(int) * nsys, cudaMemcpyHostToDevice, st);
    const int alias = (src == out && sst == out_stride) ? 1 : 0;
    k2d_newton_init<<<egrid, 256, 0, st>>>(pt, src, sst, W.YH, out, out_stride, d, W.act,
                                           1 - alias);
    std::vector<int> live = alive;
    for (int it = 0; it <= sp.newton_max_iter; ++it) {
      for (int s = 0; s < nsys; ++s) hact[s] = live[s];
      cudaMemcpyAsync(W.act, hact, sizeof(int) * nsys, cudaMemcpyHostToDevice, st);
      k2d_newton_t<<<egrid, 256, 0, st>>>(pt, out, out_stride, W.T1, W.T2, W.act);
      k2d_newton_h<<<egrid, 256, 0, st>>>(pt, out, out_stride, W.T1, W.T2, W.YH, W.RHS, W.Cv, b,
                                          d, W.act, W.partial + (long long)nsys * kPB * 2,
                                          W.partial);
      k2d_newton_norm<<<(nsys + 7) / 8, 256, 0, st>>>(nsys, W.partial + (long long)nsys * kPB * 2,
                                                      g.hd, W.res, W.act);
      cudaMemcpyAsync(hres, W.res, sizeof(double) * nsys, cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
      bool any = false;
      for (int s = 0; s < nsys; ++s) {
        if (!live[s]) continue;
        const double r = hres[s];
        if (r <= sp.newton_tol) {
          rec[s].steps += 1;
          rec[s].total += it;
          rec[s].maxit = rec[s].maxit > it ? rec[s].maxit : it;
          rec[s].maxres = rec[s].maxres > r ? rec[s].maxres : r;
          live[s] = 0;
        } else if (it == sp.newton_max_iter || !std::isfinite(r)) {
          rec[s].status = CHP_SYS_NEWTON;
          rec[s].fail_iter = it;
          rec[s].fail_res = r;
          live[s] = 0;
          alive[s] = 0;
        } else {
          any = true;
        }
      }
      if (!any) break;
      for (int s = 0; s < nsys; ++s) hact[s] = live[s];
      cudaMemcpyAsync(W.act, hact, sizeof(int) * nsys, cudaMemcpyHostToDevice, st);
      k2d_set_active<<<sb, 128, 0, st>>>(W.cg, nsys, W.act);
      if ((e = pcg_solve<N>(g, nsys, 3.0 * d, b, tol, maxcg, nt, W, st)) != cudaSuccess) return e;
      k2d_scatter<<<egrid, 256, 0, st>>>(pt, W.Yv, out, out_stride, W.cg, info, sys_index);
      k2d_cg_collect<<<sb, 128, 0, st>>>(nsys, W.cg, info, sys_index);
    }
  }
  NewtonRec* drec = reinterpret_cast<NewtonRec*>(W.partial);
  cudaMemcpyAsync(drec, rec, sizeof(NewtonRec) * nsys, cudaMemcpyHostToDevice, st);
  k2d_newton_commit<<<sb, 128, 0, st>>>(nsys, drec, info, sys_index);
  e = cudaStreamSynchronize(st);   // rec is reused by the next call
  return e != cudaSuccess ? e : cudaGetLastError();
}

bool pow2_ok(const chp_grid& g, std::string* err) {
  const int N = g.m + 1;
  if ((N & (N - 1)) != 0 || N < kMinN || N > kMaxN) {
    *err = "2D kernels need nodes_per_axis - 1 to be a power of two in [8, 1024]";
    return false;
  }
  if (g.pitch != N) {
    *err = "2D device fields must have pitch m + 1";
    return false;
  }
  return true;
}

template <int N>
cudaError_t propagate_n(Chp2d* c, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                        const double* in, long long in_stride, double* out, long long out_stride,
                        const int* idx, chp_sys_info* info, const NTables& nt, cudaStream_t st) {
  const long long fs = (long long)g.m * N;
  if (sp.scheme == CHP_LINEAR_B) {
    cudaError_t e = grow(reinterpret_cast<void**>(&c->scratch), &c->scratch_bytes,
                         2 * fs * nsys * sizeof(double), st);
    if (e != cudaSuccess) return e;
    return run_linear_b<N>(g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt,
                           c->scratch, st);
  }
  Work2 W;
  cudaError_t e = get_work(c, fs, nsys, &W, st);
  if (e != cudaSuccess) return e;
  set_smem_attrs<N>();
  return run_variable<N>(c, g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt, W,
                         st);
}

template <int N>
cudaError_t sweep_n(Chp2d* c, const chp_grid& g, const chp_spec& sp, int mode, int nic, int nsl,
                    int n0, int n1, double* U, const double* F, double* G, long long ics,
                    long long sls, unsigned char* changed, double* inc, chp_sys_info* info,
                    const NTables& nt, cudaStream_t st) {
  const long long fs = (long long)g.m * N;
  // g-buffer: nic compact fields (outside the propagate workspaces)
  double* gb = nullptr;
  cudaError_t e = cudaMallocAsync(&gb, sizeof(double) * fs * nic, st);
  if (e != cudaSuccess) return e;
  std::vector<unsigned char> first(nic, 1);
  if (mode == 1) {
    for (int i = 0; i < nic; ++i) {
      e = cudaMemcpyAsync(&first[i], changed + (long long)i * (nsl + 1) + n0, 1,
                          cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return e;
    }
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  }
  for (int n = n0; n < n1; ++n) {
    bool solve = true;
    if (mode == 1 && n == n0) {
      solve = false;
      for (int i = 0; i < nic; ++i) solve = solve || (first[i] & 1);
    }
    if (solve) {
      e = propagate_n<N>(c, g, sp, 1, nic, U + (long long)n * sls, ics, gb, fs, nullptr, info,
                         nt, st);
      if (e != cudaSuccess) break;
    }
    if (mode == 1 && n == n0) {
      // U_{n0} unchanged for ICs whose flag is 0: G(U_{n0}) is G[n0] bit for bit
      for (int i = 0; i < nic; ++i)
        if (!solve || !(first[i] & 1))
          cudaMemcpyAsync(gb + (long long)i * fs, G + (long long)i * ics + (long long)n * sls,
                          sizeof(double) * fs, cudaMemcpyDeviceToDevice, st);
    }
    if (mode == 1)
      k2d_clear_flag<<<(nic + 127) / 128, 128, 0, st>>>(changed, nic, nsl, n + 1);
    k2d_correct<<<dim3(kPB * 4, nic), 256, 0, st>>>(g.m, N, U, F, G, gb, fs, ics, sls, n, nsl,
                                                   changed, inc, mode, info);
  }
  cudaFreeAsync(gb, st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

#define CHP_N_SWITCH(N_, CALL)                 \
  switch (N_) {                                \
    case 8: { constexpr int NN = 8; CALL; }    \
    case 16: { constexpr int NN = 16; CALL; }  \
    case 32: { constexpr int NN = 32; CALL; }  \
    case 64: { constexpr int NN = 64; CALL; }  \
    case 128: { constexpr int NN = 128; CALL; } \
    case 256: { constexpr int NN = 256; CALL; } \
    case 512: { constexpr int NN = 512; CALL; } \
    case 1024: { constexpr int NN = 1024; CALL; } \
    default: break;                            \
  }

cudaError_t chp2d_propagate(Chp2d* c, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                            const double* in, long long in_stride, double* out,
                            long long out_stride, const int* sys_index, chp_sys_info* info,
                            cudaStream_t st, std::string* err) {
  if (!pow2_ok(g, err)) return cudaSuccess;
  const int N = g.m + 1;
  const NTables* nt = nullptr;
  cudaError_t e = get_tables(c, N, &nt);
  if (e != cudaSuccess) return e;
  CHP_N_SWITCH(N, return propagate_n<NN>(c, g, sp, steps, nsys, in, in_stride, out, out_stride,
                                         sys_index, info, *nt, st));
  *err = "unsupported N";
  return cudaSuccess;
}

cudaError_t chp2d_coarse_sweep(Chp2d* c, const chp_grid& g, const chp_spec& sp, int mode,
                               int nic, int nsl, int n0, int n1, double* U, const double* F,
                               double* G, long long ic_stride, long long sl_stride,
                               unsigned char* changed, double* inc, chp_sys_info* info,
                               cudaStream_t st, std::string* err) {
  if (!pow2_ok(g, err)) return cudaSuccess;
  const int N = g.m + 1;
  const NTables* nt = nullptr;
  cudaError_t e = get_tables(c, N, &nt);
  if (e != cudaSuccess) return e;
  CHP_N_SWITCH(N, return sweep_n<NN>(c, g, sp, mode, nic, nsl, n0, n1, U, F, G, ic_stride,
                                     sl_stride, changed, inc, info, *nt, st));
  *err = "unsupported N";
  return cudaSuccess;
}
