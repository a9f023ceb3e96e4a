// 2D propagators (configs 3-5): batched DST-I spectral solves.
//
// Field layout: [m rows (x, i)][pitch N = m+1 doubles (y, j)], N a power of
// two.  Storage column j holds math index j: column 0 is the zero Dirichlet
// pad, columns 1..m the interior -- so the pair (2k, 2k+1) of a row is one
// aligned double2.  Transforms are chp_fdst.cuh's pair DST-I (T' = 4T,
// T^2 = (N/2) I); every normalisation folds into one table per solve.
//
//   LINEAR_B (schemes.py:249-267)      chp_linb.cuh   row pass + column pass per step
//   LINEAR_A / Newton update solves    chp_pcg2.cuh   batched DST-preconditioned PCG
//   coarse sweep (LINEAR_A coarse)     chp_coarse2.cuh one cooperative persistent kernel
// This file: Newton residual kernels, the generic coarse correction, and the
// host side (tables, workspaces, dispatch by scheme and N).
#include <cooperative_groups.h>
#include <math.h>

#include <map>
#include <stdlib.h>
#include <string>
#include <vector>

#include "chp_common.cuh"
#include "chp_wdst.cuh"
#include "chp_linb.cuh"


namespace {

constexpr int kMinN = 8;
constexpr int kMaxN = 1024;
constexpr int kMaxDev = 64;
// short row-pass strips (phase-1 row pairs per block) for small batches
// (15 + 1 = 16 phase-0 pairs: whole chunks for G <= 16 lane groups per block)
template <int N> constexpr int kStripS = linb::RowG<N>::SP >= 32 ? 15 : linb::RowG<N>::SP;
// (single systems, e.g. the serial fine reference: 7 + 1 = 8 phase-0 pairs)
template <int N> constexpr int kStripT = linb::RowG<N>::SP >= 32 ? 7 : linb::RowG<N>::SP;

// per-device one-time launch setup (function attributes, occupancy) is indexed by
// the current device: the C ABI switches to the context's device on entry
int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}

// LINEAR_B divisors in the column pass's post-processing order (chp_linb.cuh):
// for column pair qp, lane l of L, r = 2j + h < 2C: (D''(p, 2qp), D''(p, 2qp+1)),
// p = 2(C l + j) + h, at double2 index qp N + r L + l; zero on the pad row/column.
__global__ void k2d_build_dtab3(int N, int L, const double* lam, double a2dt, double b,
                                double scale, double* d) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)N * N) return;
  const int C = N / (2 * L);
  const long long e = t / 2;                 // double2 index
  const int qp = (int)(e / N), w = (int)(e % N), r = w / L, l = w % L;
  const int p = 2 * (C * l + r / 2) + (r & 1);
  const int q = 2 * qp + (int)(t & 1);
  double v = 0.0;
  if (p > 0 && q > 0) {
    const double x = lam[p] + lam[q];
    v = scale / ((1.0 - a2dt * x) + b * (x * x));
  }
  d[t] = v;
}

// ---------------------------------------------------------------------------
// Variable-coefficient 2D solves (LINEAR_A, Newton Jacobian): matrix-free PCG
//
//   (I - a L diag(c) + b L^2) x = rhs,   L = -K (K SPD),  B = bK + a diag(c)
//   => (K^-1 + B) x = K^-1 rhs   (SPD)
// solved in the orthonormal DST basis (x^ = S x):
//   A^ x^ = d .* x^ + a S(c .* S x^),   d = 1/kappa + b kappa,  kappa = -(lam_p+lam_q)
//   b^ = (1/kappa) .* S rhs,   preconditioner M = d + a*mean(c)
// The batched solver is chp_pcg2.cuh, the cooperative coarse sweep
// chp_coarse2.cuh; below: per-system state and the elementwise kernels of the
// Newton residual (schemes.py:286-304).  Every dot product is a fixed-order
// two-level reduction, so results are bitwise reproducible run to run.
// ---------------------------------------------------------------------------

struct CgSys {
  double rho, rr0, rr, alpha, beta, acbar, pq, pad;
  int iters, done, active, fail;
};

constexpr int kPB = 64;   // partial-sum blocks per system for elementwise kernels

// ---- elementwise kernels over one field per system (grid: kPB x nsys) -----
template <class F>
CHP_DEV void for_points(int m, int N, F f) {
  const long long total = (long long)m * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / m), j = (int)(t % m);
    f(i, j, (long long)i * N + j + 1);
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
  return (i >= 0 && i < m && j >= 0 && j < m) ? f[(long long)i * N + j + 1] : 0.0;
}

// 5-point L in the CSR order of grid.py:110 (rows (i-1,j),(i,j-1),(i,j),(i,j+1),(i+1,j))
CHP_DEV double lap5(const double* f, int i, int j, int m, int N, double c) {
  return ((((at(f, i - 1, j, m, N) * c + at(f, i, j - 1, m, N) * c) +
            f[(long long)i * N + j + 1] * (-4.0 * c)) + at(f, i, j + 1, m, N) * c) +
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
  // modes 0, 2, 4, 5: interleaved (v1, v2) partials
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
  } else if (mode == 4) {            // warm start: |b^|^2 is the tolerance reference
    q.rr0 = v1;
  } else if (mode == 5) {            // warm start: initial residual of x^0
    q.rho = v1; q.rr = v2; q.iters = 0;
    q.done = !(v2 > tol2 * q.rr0) ? 1 : 0;
    if (!isfinite(v2)) { q.done = 1; q.fail = 1; }
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
    const double v = (j > 0) ? xs[t] : 0.0;
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

#include "chp_pcg2.cuh"

__global__ void k2d_newton_norm(int nsys, const double* partial, double hd, double* res,
                                const int* act) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nsys || (act && !act[s])) return;
  const double tot = warp_reduce_parts(partial + (long long)s * kPB, kPB);
  if ((threadIdx.x & 31) == 0) res[s] = sqrt(hd * tot);
}

// ---------------------------------------------------------------------------
// Device-resident coarse sweep (LINEAR_A coarse propagator, 2D): ONE
// cooperative persistent kernel runs the whole sequential recursion
//   for n in [n0, n1):  g = G(U_n) by DST-preconditioned CG;
//                       U_{n+1} = (g + F_n) - G_n;  G_n = g      (parareal.py:245-251)
// with grid-wide barriers between phases and no host round trip.  Every
// reduction is block partials -> a fixed-order sum that every block
// recomputes identically, so all blocks take the same branches and the
// result is bitwise reproducible.
// ---------------------------------------------------------------------------
// Grid-wide barrier for the co-resident (cooperative) launch: one relaxed
// spin per block and one fence on each side, instead of a fence per poll.
#ifndef CHP_C2_BAR
#define CHP_C2_BAR 1      // 1: red.release / ld.acquire; 0: fence + relaxed atomic + fence (0.820 vs 0.794 ms per slice)
#endif
struct GridBar {
  unsigned int* cnt;
  unsigned int gen;
  unsigned long long* trace;
  int cap;
};
CHP_DEV void gbar(GridBar& b) {
  __syncthreads();
  if (b.trace && blockIdx.x == 0 && threadIdx.x == 0 && (int)b.gen < b.cap) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    b.trace[b.gen] = t;
  }
  b.gen += 1;
  if (threadIdx.x == 0) {
    const unsigned int target = b.gen * gridDim.x;
    unsigned int v;
#if CHP_C2_BAR
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(b.cnt), "r"(1u) : "memory");
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b.cnt) : "memory");
    } while (v < target);
#else
    __threadfence();
    atomicAdd(b.cnt, 1u);
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b.cnt) : "memory");
    } while (v < target);
    __threadfence();
#endif
  }
  __syncthreads();
#ifdef CHP_C2_FT
  if (b.trace && blockIdx.x == 0 && threadIdx.x == 0 && (int)b.gen < b.cap)
    b.trace[4096 + 8 * b.gen] = (unsigned long long)clock64();
#endif
}

// fixed-order block reduction of (v0..v3) into part[blockIdx][0..3]
template <int K>
CHP_DEV void coop_block_partials(double (&v)[K], double* red, double* part) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) * K + k] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w * K + threadIdx.x];
    part[blockIdx.x * 8 + threadIdx.x] = t;
  }
  __syncthreads();
}

// every block: fixed-order sum over all blocks' partials -> out[0..K)
template <int K>
CHP_DEV void coop_total(const double* part, double* red, double (&out)[K]) {
  if (threadIdx.x < 32) {
    // same summation order as a per-k loop (b = lane, lane + 32, ...), with the loads
    // of eight blocks' K partials in flight together
    double x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = 0.0;
    for (int b0 = threadIdx.x; b0 < (int)gridDim.x; b0 += 32 * 8) {
      double v[8][K];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int b = b0 + 32 * e;
#pragma unroll
        for (int k = 0; k < K; ++k) v[e][k] = (b < (int)gridDim.x) ? part[b * 8 + k] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (b0 + 32 * e < (int)gridDim.x) {
#pragma unroll
          for (int k = 0; k < K; ++k) x[k] += v[e][k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double y = x[k];
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (threadIdx.x == 0) red[k] = y;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = red[k];
  __syncthreads();
}

#include "chp_coarse2.cuh"

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct NTables {
  double* lam = nullptr;   // per-axis eigenvalues, index p = 1..m
  double2* wtab = nullptr; // pair-DST lane tables: (cos, sin)(pi l/N), then W_N^{l k2} [k2][l]
};

struct Work2 {            // device workspace for one solve batch
  double *X, *Rv, *Pv, *Yv, *Cv, *RHS, *T1, *T2, *YH;
  double* partial;        // nsys * kPB * 2
  CgSys* cg;
  int* act;               // nsys
  double* res;            // nsys
  double* gbuf;           // coarse: nsys fields
  double* coop;           // cooperative coarse sweep: block partials (16 per block)
};

__global__ void k2d_clear_flag(unsigned char* changed, int nic, int nsl, int slot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nic && !(changed[(long long)i * (nsl + 1)] & 2)) changed[(long long)i * (nsl + 1) + slot] = 0;
}

// StepReport.residual_history (schemes.py:285-290): residual norm of Newton
// iteration `it` of every active system into hist[idx * hlen + it]
__global__ void k2d_newton_hist(int nsys, const double* res, const int* act, const int* sys_index,
                                double* hist, int hlen, int it) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys || !act[s] || it >= hlen) return;
  const int idx = sys_index ? sys_index[s] : s;
  hist[(long long)idx * hlen + it] = res[s];
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

// Newton control on the device (schemes.py:286-302), after the residual norms of
// iteration `it`: accept at r <= tol, NewtonDivergenceError at it == max_iter or a
// non-finite residual, otherwise stay active; the CG state follows `act`; *any is set
// while some system still needs a solve (the host polls it, no per-system decisions).
__global__ void k2d_newton_decide(int nsys, const double* res, int* act, int* alive, CgSys* cg,
                                  NewtonRec* rec, int it, int max_iter, double tol, int* any) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  int a = act[s];
  if (a) {
    const double r = res[s];
    NewtonRec& q = rec[s];
    if (r <= tol) {
      q.steps += 1;
      q.total += it;
      q.maxit = q.maxit > it ? q.maxit : it;
      q.maxres = fmax(q.maxres, r);
      a = 0;
    } else if (it == max_iter || !isfinite(r)) {
      if (q.status == CHP_SYS_OK) {
        q.status = CHP_SYS_NEWTON;
        q.fail_iter = it;
        q.fail_res = r;
      }
      a = 0;
      alive[s] = 0;
    } else {
      *any = 1;
    }
  }
  act[s] = a;
  cg[s].active = a; cg[s].done = 0; cg[s].fail = 0; cg[s].iters = 0;
}

// start of a step: every system that has not failed is active; first step: reset
__global__ void k2d_newton_begin(int nsys, int* alive, int* act, NewtonRec* rec, int reset) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  if (reset) {
    rec[s] = NewtonRec{0, 0, 0, CHP_SYS_OK, 0, 0, 0.0, 0.0};
    alive[s] = 1;
  }
  act[s] = alive[s];
}

}  // namespace

unsigned long long* g_coop_trace = nullptr;

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
  struct DTab { int N; double a2dt, b; double* d; };
  std::vector<DTab> dtabs;        // LINEAR_B spectral divisors, one per (N, dt, eps)
  void* coarse = nullptr;         // v2 coarse-sweep workspace
  double* hist = nullptr;         // Newton residual history of the current chp_propagate_hist
  int hlen = 0;                   // call (caller owned; null outside that call)
  size_t coarse_bytes = 0;
  void* pcg = nullptr;            // v2 batched PCG workspace
  size_t pcg_bytes = 0;
  double* pcg_tab = nullptr;      // Dk, SK (PI) for (pcg_tab_N, pcg_tab_b)
  int pcg_tab_N = 0;
  double pcg_tab_b = 0.0;
  void* newton = nullptr;         // device Newton control: rec[n], alive[n], any flag
  size_t newton_bytes = 0;
  int last_cg = 8;                // CG iterations of the last batched solve (first poll)
};

Chp2d* chp2d_create() { return new Chp2d(); }

void chp2d_destroy(Chp2d* c) {
  if (!c) return;
  for (auto& kv : c->tables) {
    cudaFree(kv.second.lam);
    cudaFree(kv.second.wtab);
  }
  if (c->scratch) cudaFree(c->scratch);
  for (auto& t : c->dtabs) cudaFree(t.d);
  if (c->work) cudaFree(c->work);
  if (c->coarse) cudaFree(c->coarse);
  if (c->pcg) cudaFree(c->pcg);
  if (c->pcg_tab) cudaFree(c->pcg_tab);
  if (c->newton) cudaFree(c->newton);
  if (c->host_act) cudaFreeHost(c->host_act);
  if (c->host_res) cudaFreeHost(c->host_res);
  if (c->host_rec) cudaFreeHost(c->host_rec);
  delete c;
}

namespace {

cudaError_t get_tables(Chp2d* c, int N, const NTables** out) {
  auto it = c->tables.find(N);
  if (it != c->tables.end()) { *out = &it->second; return cudaSuccess; }
  std::vector<double> lam(N);
  const long double pi = 3.14159265358979323846264338327950288L;
  const long double h = 1.0L / N;
  lam[0] = 0.0;
  for (int p = 1; p < N; ++p) {
    const long double sp = sinl(pi * p / (2.0L * N));
    lam[p] = (double)(-4.0L / (h * h) * sp * sp);
  }
  // pair-DST lane tables (chp_fdst.cuh) for wl = Geo<N>::L lanes per group:
  // [l] = (cos, sin)(pi l / N); [N + k2 wl + l] = W_N^{l k2}; [2N + k] = W_64^k
  const int wl = wdst::Geo<1024>::L == 32 && N == 1024 ? 32
               : (N == 8 ? 2 : N <= 32 ? 4 : N <= 128 ? 8 : N <= 512 ? 16 : wdst::Geo<1024>::L);
  std::vector<double2> wt(2 * N + 64);
  for (int k = 0; k < 64; ++k) {
    const long double ang = 2.0L * pi * k / 64;
    wt[2 * N + k] = make_double2((double)cosl(ang), (double)-sinl(ang));
  }
  for (int l = 0; l < N; ++l)
    wt[l] = make_double2((double)cosl(pi * l / N), (double)sinl(pi * l / N));
  for (int k2 = 0; k2 < N / wl; ++k2)
    for (int l = 0; l < wl; ++l) {
      const long double ang = 2.0L * pi * (long double)((l * k2) % N) / N;
      wt[N + k2 * wl + l] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
  NTables t;
  cudaError_t e;
  if ((e = cudaMalloc(&t.wtab, sizeof(double2) * (2 * N + 64))) != cudaSuccess) return e;
  cudaMemcpy(t.wtab, wt.data(), sizeof(double2) * (2 * N + 64), cudaMemcpyHostToDevice);
  if ((e = cudaMalloc(&t.lam, sizeof(double) * N)) != cudaSuccess) return e;
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
cudaError_t get_work(Chp2d* c, long long fs, int nsys, Work2* W, cudaStream_t st,
                     size_t coop_doubles = 0) {
  const size_t fields = 10;
  const size_t bytes = sizeof(double) * fs * nsys * fields + sizeof(double) * nsys * kPB * 4 +
                       sizeof(CgSys) * nsys + sizeof(int) * nsys + sizeof(double) * nsys + 1024 +
                       sizeof(double) * coop_doubles;
  cudaError_t e = grow(&c->work, &c->work_bytes, bytes, st);
  if (e != cudaSuccess) return e;
  static const bool poison = getenv("CHP_POISON") != nullptr;   // debug: NaN-fill workspaces
  if (poison) cudaMemsetAsync(c->work, 0xFF, c->work_bytes, st);
  double* b = static_cast<double*>(c->work);
  const long long F = fs * nsys;
  W->X = b; W->Rv = b + F; W->Pv = b + 2 * F; W->Yv = b + 3 * F; W->Cv = b + 4 * F;
  W->RHS = b + 5 * F; W->T1 = b + 6 * F; W->T2 = b + 7 * F; W->YH = b + 8 * F;
  W->gbuf = b + 9 * F;
  W->partial = b + 10 * F;
  W->cg = reinterpret_cast<CgSys*>(W->partial + (long long)nsys * kPB * 4);
  W->act = reinterpret_cast<int*>(W->cg + nsys);
  W->res = reinterpret_cast<double*>(((uintptr_t)(W->act + nsys) + 15) & ~(uintptr_t)15);
  W->coop = W->res + nsys + 2;             // cooperative sweep: barrier word + block partials
  return host_bufs(c, nsys);
}

// Batched PCG v2 (chp_pcg2.cuh): same contract as pcg_solve (inputs W.RHS,
// W.Cv, mean(c) partials in W.partial, W.cg[s].active; solution in W.Yv).
// warm != 0: start from the spectral solution X the previous solve left for the
// same system (Newton iterate / previous step), with the tolerance still
// relative to |b^| (the x0 = 0 criterion), which saves CG iterations.
template <int N>
cudaError_t pcg_solve2(Chp2d* cx, const chp_grid& g, int nsys, double a, double b, double tol,
                       int max_iter, const NTables& nt, Work2& W, cudaStream_t st, int warm) {
  using G2 = Pcg2G<N>;
  static bool attrs_dev[kMaxDev] = {};
  bool& attrs = attrs_dev[cur_dev()];
  if (!attrs) {
    const int sm = (int)G2::SMEM;
    cudaFuncSetAttribute(k_pcg2_rows<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pcg2_rows<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pcg2_rows<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pcg2_cols<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pcg2_cols<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pcg2_cols<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    attrs = true;
  }
  const long long NN = (long long)N * N;
  const double sigma = 1.0 / (8.0 * N);
  cudaError_t e;
  if (cx->pcg_tab_N != N || cx->pcg_tab_b != b) {
    if (cx->pcg_tab) { cudaStreamSynchronize(st); cudaFree(cx->pcg_tab); cx->pcg_tab = nullptr; }
    if ((e = cudaMalloc(&cx->pcg_tab, sizeof(double) * 2 * NN)) != cudaSuccess) return e;
    k_pcg2_tables<<<256, 256, 0, st>>>(N, nt.lam, b, sigma, cx->pcg_tab, cx->pcg_tab + NN);
    cx->pcg_tab_N = N;
    cx->pcg_tab_b = b;
  }
  const size_t per = 5 * (size_t)NN + 2;
  if (cx->pcg_bytes < sizeof(double) * per * nsys) warm = 0;   // workspace (re)allocated
  if ((e = grow(&cx->pcg, &cx->pcg_bytes, sizeof(double) * per * nsys, st)) != cudaSuccess) return e;
  double* w = static_cast<double*>(cx->pcg);
  Pcg2 p{};
  p.m = g.m; p.fs = (long long)g.m * N;
  p.rhs = W.RHS; p.cv = W.Cv; p.out = W.Yv;
  p.X = w; p.R = w + NN * nsys; p.P = w + 2 * NN * nsys; p.Y = w + 3 * NN * nsys;
  p.CT = w + 4 * NN * nsys;
  p.Dk = cx->pcg_tab; p.SK = cx->pcg_tab + NN;
  p.a = a; p.sigma = sigma; p.cg = W.cg; p.partial = W.partial; p.wtab = nt.wtab;
  const int red_blocks = (nsys + 7) / 8;
  const dim3 eg(kPB, nsys), rg(G2::RBLK, nsys), cgd(N / G2::TC, nsys);
  const size_t sm = G2::SMEM;
  const int m = g.m;
  k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 3, 0, 0,
                                           1.0 / ((double)m * m), a);
  k_pcg2_prep<N><<<eg, 256, 0, st>>>(p);
  k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 0);
  k_pcg2_cols<N, 0><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 0);
  if (warm) {
    k_pcg2_warm_a<N><<<eg, 256, 0, st>>>(p);
    k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 4, 0, 0, 0, 0);
    k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.P, p.Y, 0);
    k_pcg2_cols<N, 1><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 0);
    k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 0);
    k_pcg2_aptail<N><<<eg, 256, 0, st>>>(p, 0);
    k_pcg2_warm_b<N><<<eg, 256, 0, st>>>(p);
    k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 5, tol * tol, 0, 0, 0);
  } else {
    k_pcg2_init<N><<<eg, 256, 0, st>>>(p);
    k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 0, 0, 0, 0, 0);
  }
  // host poll of the CG states: first after as many iterations as the last solve took
  // (systems that finish early skip the remaining launches), then every 4
  std::vector<CgSys> host(nsys);
  int chunk = cx->last_cg < 4 ? 4 : (cx->last_cg > 32 ? 32 : cx->last_cg);
  for (int it0 = 0; it0 < max_iter + chunk; it0 += chunk, chunk = 4) {
    for (int it = 0; it < chunk; ++it) {
#if CHP_PCG2_FUSE
      k_pcg2_rows<N, 1><<<rg, G2::THREADS, sm, st>>>(p, p.P, p.Y, 1);
      k_pcg2_cols<N, 1><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k_pcg2_rows<N, 2><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, G2::RBLK, 1, 0, 0, 0, 0);
#else
      k_pcg2_pdir<N><<<eg, 256, 0, st>>>(p);
      k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.P, p.Y, 1);
      k_pcg2_cols<N, 1><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k_pcg2_aptail<N><<<eg, 256, 0, st>>>(p, 1);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 1, 0, 0, 0, 0);
#endif
      k_pcg2_update<N><<<eg, 256, 0, st>>>(p);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 2, tol * tol,
                                               max_iter, 0, 0);
    }
    if ((e = cudaMemcpyAsync(host.data(), W.cg, sizeof(CgSys) * nsys, cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    bool all = true;
    int mx = 0;
    for (int s = 0; s < nsys; ++s) {
      all = all && (!host[s].active || host[s].done);
      if (host[s].active && host[s].iters > mx) mx = host[s].iters;
    }
    if (all) {
      if (mx > 0) cx->last_cg = mx;
      break;
    }
  }
  // x = S x^ = sigma T'_i T'_j X -> W.Yv (external layout)
  k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.X, p.Y, 0);
  k_pcg2_cols<N, 2><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, W.Yv, 0);
  return cudaGetLastError();
}

template <int N>
cudaError_t pcg_dispatch(Chp2d* cx, const chp_grid& g, int nsys, double a, double b, double tol,
                         int max_iter, const NTables& nt, Work2& W, cudaStream_t st, int warm) {
  static const bool cold = getenv("CHP_PCG_COLD") != nullptr;   // A/B: no warm start
  return pcg_solve2<N>(cx, g, nsys, a, b, tol, max_iter, nt, W, st, cold ? 0 : warm);
}

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
      if ((e = pcg_dispatch<N>(cx, g, nsys, sp.dt, sp.b, tol, maxcg, nt, W, st, s > 0)) != cudaSuccess)
        return e;
      k2d_scatter<<<egrid, 256, 0, st>>>(pt, W.Yv, out, out_stride, W.cg, info, sys_index);
      k2d_cg_collect<<<sb, 128, 0, st>>>(nsys, W.cg, info, sys_index);
    }
    return cudaGetLastError();
  }
  // ---- Newton (schemes.py:270-305): decisions on the device, the host only polls
  // "any system still active" once per Newton solve from the second residual on ----
  const double d = sp.dt, b = sp.b;
  {
    const size_t need = sizeof(NewtonRec) * nsys + sizeof(int) * (nsys + 4);
    if ((e = grow(&cx->newton, &cx->newton_bytes, need, st)) != cudaSuccess) return e;
  }
  NewtonRec* drec = static_cast<NewtonRec*>(cx->newton);
  int* alive = reinterpret_cast<int*>(drec + nsys);
  int* any = alive + nsys;
  int* hany = cx->host_act;                 // pinned
  for (int step = 0; step < steps; ++step) {
    const double* src = (step == 0) ? in : out;
    const long long sst = (step == 0) ? in_stride : out_stride;
    Pt pt{m, N, fs, g.c1, sys_index, sys_index};
    k2d_newton_begin<<<sb, 128, 0, st>>>(nsys, alive, W.act, drec, step == 0);
    const int alias = (src == out && sst == out_stride) ? 1 : 0;
    k2d_newton_init<<<egrid, 256, 0, st>>>(pt, src, sst, W.YH, out, out_stride, d, W.act,
                                           1 - alias);
    for (int it = 0; it <= sp.newton_max_iter; ++it) {
      cudaMemsetAsync(any, 0, sizeof(int), st);
      k2d_newton_t<<<egrid, 256, 0, st>>>(pt, out, out_stride, W.T1, W.T2, W.act);
      k2d_newton_h<<<egrid, 256, 0, st>>>(pt, out, out_stride, W.T1, W.T2, W.YH, W.RHS, W.Cv, b,
                                          d, W.act, W.partial + (long long)nsys * kPB * 2,
                                          W.partial);
      k2d_newton_norm<<<(nsys + 7) / 8, 256, 0, st>>>(nsys, W.partial + (long long)nsys * kPB * 2,
                                                      g.hd, W.res, W.act);
      if (cx->hist != nullptr && it < cx->hlen)
        k2d_newton_hist<<<sb, 128, 0, st>>>(nsys, W.res, W.act, sys_index, cx->hist, cx->hlen,
                                            it);
      k2d_newton_decide<<<sb, 128, 0, st>>>(nsys, W.res, W.act, alive, W.cg, drec, it,
                                            sp.newton_max_iter, sp.newton_tol, any);
      if (it >= 1) {                        // the residual before the first solve is
        cudaMemcpyAsync(hany, any, sizeof(int), cudaMemcpyDeviceToHost, st);   // never polled
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        if (!*hany) break;
      }
      if ((e = pcg_dispatch<N>(cx, g, nsys, 3.0 * d, b, tol, maxcg, nt, W, st,
                               step > 0 || it > 0)) != cudaSuccess)
        return e;
      k2d_scatter<<<egrid, 256, 0, st>>>(pt, W.Yv, out, out_stride, W.cg, info, sys_index);
      k2d_cg_collect<<<sb, 128, 0, st>>>(nsys, W.cg, info, sys_index);
    }
  }
  k2d_newton_commit<<<sb, 128, 0, st>>>(nsys, drec, info, sys_index);
  return cudaGetLastError();
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

// LINEAR_B divisors D'' = (2/N)^2 D / 256 for one (N, dt, eps) (the _FACTOR_CACHE
// analogue, schemes.py:134-142), in the column-pair-major layout of chp_linb.cuh
cudaError_t get_dtab(Chp2d* c, int N, const chp_spec& sp, const NTables& nt, const double** out,
                     cudaStream_t st) {
  const double a2dt = 2.0 * sp.dt, b = sp.b;
  for (auto& t : c->dtabs)
    if (t.N == N && t.a2dt == a2dt && t.b == b) { *out = t.d; return cudaSuccess; }
  if (c->dtabs.size() >= 8) {              // bounded cache: drop the oldest table
    cudaStreamSynchronize(st);
    cudaFree(c->dtabs.front().d);
    c->dtabs.erase(c->dtabs.begin());
  }
  Chp2d::DTab t{N, a2dt, b, nullptr};
  cudaError_t e = cudaMalloc(&t.d, sizeof(double) * ((size_t)N * N + 2));
  if (e != cudaSuccess) return e;
  const long long n = (long long)N * N + 2;
  const double scale = (2.0 / N) * (2.0 / N) / 256.0;
  const int lanes = N == 8 ? 2 : N <= 32 ? 4 : N <= 128 ? 8 : N <= 512 ? 16 : 32;   // Geo<N>::L
  k2d_build_dtab3<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(N, lanes, nt.lam, a2dt, b, scale,
                                                              t.d);
  c->dtabs.push_back(t);
  *out = t.d;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaStreamSynchronize(st);        // usable from any stream afterwards
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (libchp links no libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// Tensor map of the Q scratch (nsys fields of N x N doubles, row-major) for the TMA column
// pass: a 2D tensor {N columns, N nsys rows}, boxes of {2 GROUPS columns, BR rows}
template <int N>
bool make_qmap(CUtensorMap* map, double* Qb, int nsys) {
  using CT = linb::ColT<N>;
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)N * (cuuint64_t)nsys};
  const cuuint64_t strides[1] = {(cuuint64_t)N * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)(CT::IB / 8), (cuuint32_t)CT::BR};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Qb, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             CT::IB == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                          : (CT::IB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B),
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor map of the P scratch for the column pass's TMA store (N = 1024): a row pair is 2N
// doubles; dimension order {columns, l, j} with row pair k = C l + j (chp_linb.cuh ColT)
template <int N>
bool make_pmap(CUtensorMap* map, double* P, int nsys) {
  using F = fdst::FG<N>;
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  const cuuint64_t rp = (cuuint64_t)2 * N * sizeof(double);   // bytes per row pair
  const cuuint64_t dims[3] = {(cuuint64_t)2 * N, (cuuint64_t)F::L * (cuuint64_t)nsys, (cuuint64_t)F::C};
  const cuuint64_t strides[2] = {rp * F::C, rp};
  const cuuint32_t box[3] = {(cuuint32_t)(linb::ColT<N>::PB / 8), (cuuint32_t)F::L, (cuuint32_t)F::C};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, P, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             linb::ColT<N>::PB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// LINEAR_B v2 (chp_linb.cuh): J steps = J+1 row passes + J column passes over
// pair-interleaved P / Q scratch fields (2 N^2 doubles per system).
template <int N>
cudaError_t run_linear_b2(const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                          const double* in, long long in_stride, double* out, long long out_stride,
                          const int* sys_index, chp_sys_info* info, const NTables& nt,
                          double* scratch, const double* dtab, cudaStream_t st) {
  using RG = linb::RowG<N>;
  using CG = linb::ColG<N>;
  static bool attrs_dev[kMaxDev] = {};
  bool& attrs = attrs_dev[cur_dev()];
  if (!attrs) {
    cudaFuncSetAttribute(linb::k2d_rowb<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    cudaFuncSetAttribute(linb::k2d_rowb<N, kStripS<N>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)RG::SMEM);
    cudaFuncSetAttribute(linb::k2d_rowb<N, kStripT<N>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)RG::SMEM);
    cudaFuncSetAttribute(linb::k2d_colb<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    if constexpr (N >= 64)
      cudaFuncSetAttribute(linb::k2d_colt<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)linb::ColT<N>::SMEM);
    if constexpr (N == 1024) {
      if constexpr (linb::ColT<N>::PB == 128)
        cudaFuncSetAttribute(linb::k2d_colt2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)linb::ColT2<N>::SMEM);
    }
    attrs = true;
  }
  const long long fs2 = (long long)N * N;
  double* P = scratch;
  double* Qb = scratch + fs2 * nsys;
  // strip length: the longest (fewest re-transformed halo pairs) that still gives
  // every SM several row-pass blocks; small batches (late Parareal iterations, config
  // 3, the serial fine reference) get short strips instead of idle SMs
  bool short_strips = false, tiny_strips = false;
  {
    static int sms_dev[kMaxDev] = {};
    int& sms = sms_dev[cur_dev()];
    if (sms == 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_dev());
    short_strips = (long long)((RG::NP + RG::SP - 1) / RG::SP) * nsys < (long long)sms * RG::MINB;
    tiny_strips = (long long)((RG::NP + kStripS<N> - 1) / kStripS<N>) * nsys < (long long)sms;
  }
  const int strip = tiny_strips ? kStripT<N> : short_strips ? kStripS<N> : RG::SP;
  const dim3 rgrid((RG::NP + strip - 1) / strip, nsys), cgrid(N / CG::TC, nsys);
  auto rowb = tiny_strips ? linb::k2d_rowb<N, kStripT<N>>
                          : short_strips ? linb::k2d_rowb<N, kStripS<N>> : linb::k2d_rowb<N>;
  linb::RowArgs ra{};
  ra.m = g.m; ra.cdt = sp.dt * g.c1; ra.info = info; ra.info_index = sys_index; ra.wtab = nt.wtab;
  linb::ColArgs ca{Qb, P, fs2, reinterpret_cast<const double2*>(dtab), nt.wtab};
  // column pass: TMA tile kernel for N >= 64 (CHP_COL_TMA=0 selects the cp.async kernel)
  CUtensorMap qmap, pmap;
  bool tma = false;
  if constexpr (N >= 64) {
    static const bool want = [] { const char* e = getenv("CHP_COL_TMA"); return !(e && e[0] == '0'); }();
    tma = want && make_qmap<N>(&qmap, Qb, nsys);
    if (tma && linb::ColT<N>::PSTORE) tma = make_pmap<N>(&pmap, P, nsys);
    else if (tma) pmap = qmap;
  }
  auto colpass = [&] {
    if constexpr (N >= 64) {
      if (tma) {
        if constexpr (N == 1024) {
          if constexpr (linb::ColT<N>::PB == 128) {
          // measured slower (kernel bench 17.08 vs 14.53 ms per 16 config-5-shaped steps): off by default
          static const bool teams = [] { const char* e = getenv("CHP_COL_TEAMS"); return e && e[0] == '1'; }();
          if (teams) {
            linb::k2d_colt2<N><<<dim3(cgrid.x / 2, cgrid.y), linb::ColT2<N>::THREADS, linb::ColT2<N>::SMEM, st>>>(
                qmap, pmap, ca);
            return;
          }
          }
        }
        linb::k2d_colt<N><<<cgrid, CG::THREADS, linb::ColT<N>::SMEM, st>>>(qmap, pmap, ca);
        return;
      }
    }
    linb::k2d_colb<N><<<cgrid, CG::THREADS, CG::SMEM, st>>>(ca);
  };
  for (int s = 0; s < steps; ++s) {
    if (s == 0) { ra.in = in; ra.in_stride = in_stride; ra.in_index = sys_index; ra.mode = linb::MODE_FIRST; }
    else { ra.in = P; ra.in_stride = fs2; ra.in_index = nullptr; ra.mode = linb::MODE_MID; }
    ra.out = Qb; ra.out_stride = fs2; ra.out_index = nullptr;
    rowb<<<rgrid, RG::THREADS, RG::SMEM, st>>>(ra);
    colpass();
  }
  ra.in = P; ra.in_stride = fs2; ra.in_index = nullptr; ra.mode = linb::MODE_LAST;
  ra.out = out; ra.out_stride = out_stride; ra.out_index = sys_index;
  rowb<<<rgrid, RG::THREADS, RG::SMEM, st>>>(ra);
  return cudaGetLastError();
}

template <int N>
cudaError_t propagate_n(Chp2d* c, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                        const double* in, long long in_stride, double* out, long long out_stride,
                        const int* idx, chp_sys_info* info, const NTables& nt, cudaStream_t st) {
  const long long fs = (long long)g.m * N;
  if (sp.scheme == CHP_LINEAR_B) {
    cudaError_t e = grow(reinterpret_cast<void**>(&c->scratch), &c->scratch_bytes,
                         2 * (long long)N * N * nsys * sizeof(double), st);
    if (e != cudaSuccess) return e;
    const double* dtab = nullptr;
    if ((e = get_dtab(c, N, sp, nt, &dtab, st)) != cudaSuccess) return e;
    return run_linear_b2<N>(g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt,
                            c->scratch, dtab, st);
  }
  Work2 W;
  cudaError_t e = get_work(c, fs, nsys, &W, st);
  if (e != cudaSuccess) return e;
  return run_variable<N>(c, g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt, W,
                         st);
}

template <int N>
cudaError_t sweep_n(Chp2d* c, const chp_grid& g, const chp_spec& sp, int mode, int nic, int nsl,
                    int n0, int n1, double* U, const double* F, double* G, long long ics,
                    long long sls, unsigned char* changed, double* inc, chp_sys_info* info,
                    const NTables& nt, cudaStream_t st, const chp_hop* hop, bool* fused) {
  const long long fs = (long long)g.m * N;
  // LINEAR_A coarse: the whole sweep in one cooperative persistent kernel
  // (chp_coarse2.cuh, no host round trips); other coarse schemes: one batched
  // propagate per slice + the correction kernel below
  if (sp.scheme == CHP_LINEAR_A) {
    using G2 = Coop2G<N>;
    static int blocks_dev[kMaxDev] = {};
    static bool res_ok_dev[kMaxDev] = {};
    int& blocks = blocks_dev[cur_dev()];
    bool& res_ok = res_ok_dev[cur_dev()];
    if (blocks == 0) {
      cudaFuncSetAttribute(k2d_coarse2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)G2::SMEM_RES);
      int dev = 0, sms = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2d_coarse2<N>, G2::THREADS,
                                                    G2::SMEM_RES);
      // One block per SM at most (half the grid-barrier arrivals of two), and for the smaller
      // grids only twice the blocks the transforms need (N / (2 GPB) row-pair groups, N / TC
      // column tiles): the others would only take part in the barriers and the elementwise
      // loops.  Config 3 (N = 256) to tolerance: 148 blocks 1.30 s, 64: 1.18 s, 32: 1.17 s,
      // 16: 1.22 s.  N = 1024 needs 128 and keeps every SM.  (The dot products' summation
      // order follows the block count, so results depend on it in the last bits.)
      const int need = (N / 2 + G2::GPB - 1) / G2::GPB;
      blocks = 2 * need < 8 ? 8 : 2 * need;
      if (blocks > sms) blocks = sms;
      res_ok = per >= 1;
      if (const char* e = getenv("CHP_C2_BLOCKS")) {      // A/B knob
        const int want = atoi(e);
        if (want > 0) blocks = want < need ? (need < sms ? need : sms) : (want < sms ? want : sms);
      }
    }
    const size_t NN = (size_t)N * N;
    const size_t doubles = 10 * NN + 2 + (size_t)fs + 16 * (size_t)blocks + 16;
    cudaError_t e = grow(&c->coarse, &c->coarse_bytes, sizeof(double) * doubles, st);
    if (e != cudaSuccess) return e;
    double* w = static_cast<double*>(c->coarse);
    Coop2Args ca{};
    ca.m = g.m; ca.nic = nic; ca.nsl = nsl; ca.n0 = n0; ca.n1 = n1; ca.mode = mode;
    ca.c1 = g.c1; ca.dt = sp.dt; ca.b = sp.b; ca.tol = sp.cg_tol; ca.max_iter = sp.cg_max_iter;
    ca.U = U; ca.F = F; ca.G = G; ca.ics = ics; ca.sls = sls;
    ca.changed = changed; ca.inc = inc; ca.info = info;
    ca.X = w; ca.R = w + NN; ca.P = w + 2 * NN; ca.Y = w + 3 * NN; ca.Mi = w + 4 * NN;
    ca.Dk = w + 5 * NN; ca.SK = w + 6 * NN; ca.CT = w + 7 * NN;       // CT: NN + 2 (slack)
    ca.S = w + 8 * NN + 2; ca.W = w + 9 * NN + 2;
    ca.gx = w + 10 * NN + 2;
    ca.part = ca.gx + fs;
    ca.bar = reinterpret_cast<unsigned int*>(ca.part + 16 * (size_t)blocks);
    {
      static unsigned long long* tr = nullptr;
      const char* env = getenv("CHP_COOP_TRACE");
      if (env && !tr) {
        cudaMalloc(&tr, sizeof(unsigned long long) * 4096 * 9);
        cudaMemset(tr, 0, sizeof(unsigned long long) * 4096 * 9);
      }
      ca.trace = env ? tr : nullptr;
      ca.trace_cap = 4096;
      if (env) g_coop_trace = tr;
    }
    // every lane group owns one row pair for the whole solve: r and w stay in shared memory
    static const bool no_res = getenv("CHP_C2_NORES") != nullptr;
    ca.res = (!no_res && res_ok && N / 2 <= blocks * G2::GPB) ? 1 : 0;
    cudaMemsetAsync(ca.bar, 0, sizeof(unsigned int), st);
    ca.lam = nt.lam; ca.wtab = nt.wtab;
    if (hop) {
      ca.hop_u = hop->peer_u; ca.hop_stride = hop->peer_stride; ca.hop_changed = hop->peer_changed;
      ca.hop_flag = hop->peer_flag; ca.hop_seq = hop->seq;
      *fused = true;
    }
    void* args[] = {&ca};
    return cudaLaunchCooperativeKernel((void*)k2d_coarse2<N>, dim3(blocks), dim3(G2::THREADS),
                                       args, ca.res ? G2::SMEM_RES : G2::SMEM, st);
  }
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
                            double* hist, int hlen, cudaStream_t st, std::string* err) {
  if (!pow2_ok(g, err)) return cudaSuccess;
  const int N = g.m + 1;
  const NTables* nt = nullptr;
  cudaError_t e = get_tables(c, N, &nt);
  if (e != cudaSuccess) return e;
  // the history buffer belongs to this call only (the caller holds the context lock)
  struct HistScope {
    Chp2d* c;
    ~HistScope() { c->hist = nullptr; c->hlen = 0; }
  } hs{c};
  c->hist = hist;
  c->hlen = hist ? hlen : 0;
  CHP_N_SWITCH(N, return propagate_n<NN>(c, g, sp, steps, nsys, in, in_stride, out, out_stride,
                                         sys_index, info, *nt, st));
  *err = "unsupported N";
  return cudaSuccess;
}

cudaError_t chp2d_coarse_sweep(Chp2d* c, const chp_grid& g, const chp_spec& sp, int mode,
                               int nic, int nsl, int n0, int n1, double* U, const double* F,
                               double* G, long long ic_stride, long long sl_stride,
                               unsigned char* changed, double* inc, chp_sys_info* info,
                               cudaStream_t st, std::string* err, const chp_hop* hop,
                               bool* fused) {
  *fused = false;
  if (!pow2_ok(g, err)) return cudaSuccess;
  const int N = g.m + 1;
  const NTables* nt = nullptr;
  cudaError_t e = get_tables(c, N, &nt);
  if (e != cudaSuccess) return e;
  c->hist = nullptr;            // coarse steps never record a residual history
  c->hlen = 0;
  CHP_N_SWITCH(N, return sweep_n<NN>(c, g, sp, mode, nic, nsl, n0, n1, U, F, G, ic_stride,
                                     sl_stride, changed, inc, info, *nt, st, hop, fused));
  *err = "unsupported N";
  return cudaSuccess;
}

// debug: copy the cooperative coarse kernel's barrier timestamps (ns) to the host
extern "C" int chp_debug_trace(unsigned long long* host, int n) {
  if (!g_coop_trace || !host || n <= 0) return 0;
  if (n > 4096 * 9) n = 4096 * 9;
  cudaMemcpy(host, g_coop_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  return n;
}
