// 1D propagators (configs 1 and 2): one CUDA thread per system.
//
// Compiled with --fmad=false: every multiply/add below rounds exactly as the
// reference's numpy / scipy sparsetools code does, and the only fused
// operations are the explicit fma() calls that mirror the FMA-contracted
// OpenBLAS kernels under LAPACK (verified bit-for-bit against scipy's
// dpbtrf/dpbtrs and dgbtf2/dgbtrs; see tests/test_oracle_golden.py and
// DESIGN.md section "1D arithmetic contract").
//
//   LINEAR_B  (schemes.py:249-267): rhs = v + dt*L(v^3 - 3v); banded Cholesky
//             factor cached per (m, dt, eps) (schemes.py:191-227), factored on
//             the device by k1d_pbtf2 (LAPACK dpbtf2 order), solved as dpbtrs.
//   LINEAR_A  (schemes.py:235-246): banded LU with partial pivoting, LAPACK
//             dgbtf2 + dgbtrs order, the L-solve fused into the factorisation
//             sweep (bit-identical: it touches the rhs in the same order).
//   EYRE      (schemes.py:270-305): undamped Newton, residual before each
//             solve, accept at <= tol, fail at max_iter or non-finite.
//
// Work arrays are interleaved [index][system] so that the per-thread
// sequential sweeps are coalesced across a warp.
#include <math.h>

#include "chp_common.cuh"

namespace {

struct G1 {
  int m;
  double c1, s_main, s_edge, s_off1, s_off2, hd;
};

CHP_DEV G1 make_g1(const chp_grid& g) {
  G1 r;
  r.m = g.m; r.c1 = g.c1; r.s_main = g.s_main; r.s_edge = g.s_edge;
  r.s_off1 = g.s_off1; r.s_off2 = g.s_off2; r.hd = g.hd;
  return r;
}

// (L v)_i, CSR row order (i-1, i, i+1) starting from 0 (grid.py:102-111);
// the zero Dirichlet pads add exact zeros.
CHP_DEV double lap3(double vm, double v0, double vp, double c1) {
  return (vm * c1 + v0 * (-2.0 * c1)) + vp * c1;
}

// (L@L y)_i in the CSR column order scipy's csr_matmat leaves in
// DiscreteOperator.squared (columns i+2, i+1, i, i-1, i-2).
CHP_DEV double bilap5(double ym2, double ym1, double y0, double yp1, double yp2,
                      double s0, const G1& g) {
  return (((yp2 * g.s_off2 + yp1 * g.s_off1) + y0 * s0) + ym1 * g.s_off1) + ym2 * g.s_off2;
}

CHP_DEV double ld(const double* v, int i, int m) { return (i >= 0 && i < m) ? v[i] : 0.0; }

// x / d correctly rounded, given r = RN(1/d): q0 = RN(x r), q = RN(q0 + (x - q0 d) r)
// (Markstein's theorem; exactly IEEE x/d, but three dependent FMA-class ops
// instead of the division subroutine on the sequential critical path).
CHP_DEV double div_rn(double x, double d, double r) {
  const double q0 = x * r;
  const double e = fma(-q0, d, x);
  return fma(e, r, q0);
}

// ---------------------------------------------------------------------------
// Banded (2,2) LU with partial pivoting, LAPACK dgbtf2 + dgbtrs(L part).
// gen(r, e[5], &rhs) produces row r of the ORIGINAL matrix, entries
// A[r][r-2..r+2], and rhs_r.  U rows and the forward-substituted rhs are
// written to ub (6 values per row, interleaved stride ks).
// Returns nonzero if a zero pivot was met (dgbtf2 INFO > 0).
// ---------------------------------------------------------------------------
// The raw inputs of the rows entering the elimination window (the iterate value
// y_{r+1} and a per-row auxiliary such as yhat_r) are loaded kPD rows ahead
// into a register queue; the row itself is formed only when it enters, so the
// global loads are in flight for kPD elimination steps instead of sitting on
// the sequential pivot/eliminate chain.  The arithmetic is unchanged (the row
// is formed from the same values with the same expressions: bit-identical).
//   load(r)                      -> double2 (y_{r+1} or 0, aux_r or 0)
//   make(r, ym, y0, yp, aux, e[5], rhs)  row r from y_{r-1}, y_r, y_{r+1}, aux_r
#ifndef CHP_1D_PD
#define CHP_1D_PD 8
#endif
constexpr int kPD = CHP_1D_PD;
#ifndef CHP_1D_SPECRCP
#define CHP_1D_SPECRCP 1
#endif
#ifndef CHP_1D_RQ
#define CHP_1D_RQ 16
#endif
constexpr int kRQ = CHP_1D_RQ > 0 ? CHP_1D_RQ : 1;   // residual loop: rows of y / yhat in flight

template <class Load, class Make>
CHP_DEV int band_lu_forward(int m, Load load, Make make, double* __restrict__ ub, long long ks) {
  double W[3][5];
  double bb[3];
  // rows 0..2 directly; y window for row 3 = (y_2, y_3)
  double yv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) yv[i] = (i < m) ? load(i - 1).x : 0.0;   // load(i-1).x = y_i
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 5; ++c) W[r][c] = 0.0;
    bb[r] = 0.0;
    if (r < m) {
      double e[5], rhs;
      make(r, r >= 1 ? yv[r - 1] : 0.0, yv[r], yv[r + 1], load(r).y, e, rhs);
#pragma unroll
      for (int d = -2; d <= 2; ++d) {
        const int col = r + d;
        if (col >= 0 && col < 5 && col < m) W[r][col] = e[d + 2];
      }
      bb[r] = rhs;
    }
  }
  double w0 = yv[2], w1 = yv[3];
  double2 Qy[kPD];
#pragma unroll
  for (int q = 0; q < kPD; ++q) Qy[q] = load(3 + q);
  int singular = 0;
  for (int j0 = 0; j0 < m; j0 += kPD) {
#pragma unroll
    for (int jj = 0; jj < kPD; ++jj) {
      const int j = j0 + jj;
      if (j >= m) break;
      const int km = min(2, m - 1 - j);
#if CHP_1D_SPECRCP
      // the reciprocals of the three pivot candidates start before the pivot is chosen: the
      // division is the longest link of the row-to-row dependence chain and the comparisons
      // and the row swap then run beside it instead of in front of it (same value: RN(1/pivot))
      const double rc0 = 1.0 / W[0][0], rc1 = 1.0 / W[1][0], rc2 = 1.0 / W[2][0];
#endif
      int jp = 0;
      double amax = fabs(W[0][0]);
      if (km >= 1 && fabs(W[1][0]) > amax) { jp = 1; amax = fabs(W[1][0]); }
      if (km >= 2 && fabs(W[2][0]) > amax) { jp = 2; }
      double piv = (jp == 0) ? W[0][0] : (jp == 1 ? W[1][0] : W[2][0]);
#if CHP_1D_SPECRCP
      const double rcpv = (jp == 0) ? rc0 : (jp == 1 ? rc1 : rc2);
#endif
      if (piv != 0.0) {
        if (jp != 0) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            const double t = W[0][c];
            W[0][c] = (jp == 1) ? W[1][c] : W[2][c];
            if (jp == 1) W[1][c] = t; else W[2][c] = t;
          }
          const double t = bb[0];
          bb[0] = (jp == 1) ? bb[1] : bb[2];
          if (jp == 1) bb[1] = t; else bb[2] = t;
        }
        if (km > 0) {
#if CHP_1D_SPECRCP
          const double rcp = rcpv;                    // DSCAL(km, ONE/AB(KV+1,J))
#else
          const double rcp = 1.0 / W[0][0];           // DSCAL(km, ONE/AB(KV+1,J))
#endif
          W[1][0] = W[1][0] * rcp;
          if (km >= 2) W[2][0] = W[2][0] * rcp;
#pragma unroll
          for (int c = 1; c < 5; ++c) {               // DGER(-1): fma(l_i, -u_jc, a)
            W[1][c] = fma(W[1][0], -W[0][c], W[1][c]);
            if (km >= 2) W[2][c] = fma(W[2][0], -W[0][c], W[2][c]);
          }
          bb[1] = fma(W[1][0], -bb[0], bb[1]);        // dgbtrs DGER on the rhs
          if (km >= 2) bb[2] = fma(W[2][0], -bb[0], bb[2]);
        }
      } else {
        singular = 1;
      }
      double* u = ub + (long long)j * 7 * ks;
#pragma unroll
      for (int c = 0; c < 5; ++c) u[c * ks] = W[0][c];
      u[5 * ks] = bb[0];
#if CHP_1D_SPECRCP
      u[6 * ks] = rcpv;                             // RN(1/U_jj) for the backward sweep
#else
      u[6 * ks] = 1.0 / W[0][0];                    // RN(1/U_jj) for the backward sweep
#endif
      // slide the window one row/column down; row r = j+3 enters from the queue
#pragma unroll
      for (int c = 0; c < 4; ++c) { W[0][c] = W[1][c + 1]; W[1][c] = W[2][c + 1]; }
      W[0][4] = 0.0;
      W[1][4] = 0.0;
      bb[0] = bb[1];
      bb[1] = bb[2];
      const int r = j + 3;
      const double2 q = Qy[jj];
#pragma unroll
      for (int c = 0; c < 5; ++c) W[2][c] = 0.0;
      bb[2] = 0.0;
      if (r < m) {
        double e[5], rhs;
        make(r, w0, w1, q.x, q.y, e, rhs);
#pragma unroll
        for (int c = 0; c < 5; ++c)  // window col c <-> matrix col j+1+c = r-2+c
          if (r - 2 + c < m) W[2][c] = e[c];
        bb[2] = rhs;
      }
      w0 = w1;
      w1 = q.x;
      Qy[jj] = load(r + kPD);        // refill: row r + kPD
    }
  }
  return singular;
}

// cp.async helpers and the per-lane shared ring of the backward sweep
#ifndef CHP_1D_RB
#define CHP_1D_RB 16
#endif
constexpr int kRB = CHP_1D_RB;
constexpr int kRingBytes = kRB * 7 * 32 * (int)sizeof(double);
static_assert(kRingBytes <= 48 * 1024, "default dynamic shared memory limit");

CHP_DEV void cp_async8(double* sdst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
CHP_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
CHP_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Upper-triangular band solve (dtbsv 'U','N', bandwidth KL+KU = 4).
// Returns whether every x_i is finite (checked on the values as they are
// produced: the Field validation of grid.py:84-85 without re-reading x).
CHP_DEV bool band_lu_backward(int m, const double* __restrict__ ub, long long ks,
                              double* __restrict__ x) {
  bool fin = true;
  // The 7 values of row i are staged kRB rows ahead into a per-lane shared
  // ring by cp.async: the prefetch depth costs no registers, so the chain of
  // dependent divides never waits on the L2 round trip of the ub rows that
  // the forward sweep has just written.  Launches are one warp per block.
  // The ring is dynamic shared memory (kRingBytes) so that LINEAR_B launches,
  // which never reach this sweep, keep the whole L1 carve-out.
  extern __shared__ double ring1d[];
  double(*ring)[7][32] = reinterpret_cast<double (*)[7][32]>(ring1d);
  const int lane = threadIdx.x & 31;
  auto issue = [&](int i) {
    if (i >= 0) {
      const double* u = ub + (long long)i * 7 * ks;
      double* s = &ring[i & (kRB - 1)][0][lane];
#pragma unroll
      for (int c = 0; c < 7; ++c) cp_async8(s + c * 32, u + c * ks);
    }
    cp_commit();
  };
#pragma unroll
  for (int p = 0; p < kRB; ++p) issue(m - 1 - p);
  double x1 = 0.0, x2 = 0.0, x3 = 0.0, x4 = 0.0;
#pragma unroll 4
  for (int i = m - 1; i >= 0; --i) {
    cp_wait<kRB - 1>();
    const double* q = &ring[i & (kRB - 1)][0][lane];
    double t = q[5 * 32];
    t = fma(-x4, q[4 * 32], t);
    t = fma(-x3, q[3 * 32], t);
    t = fma(-x2, q[2 * 32], t);
    t = fma(-x1, q[1 * 32], t);
    const double xi = div_rn(t, q[0], q[6 * 32]);
    x4 = x3; x3 = x2; x2 = x1; x1 = xi;
    x[i] = xi;
    fin = fin && isfinite(xi);
    issue(i - kRB);   // same slot: its values were consumed by the chain above
  }
  cp_wait<0>();
  return fin;
}

struct BandConst {   // scalars of I - a L diag(c) + b L^2 (schemes.py:149-153)
  double a_lmain;    // a * lap_main  = a * (-2 c1)
  double ma_loff;    // (-a) * lap_off = (-a) * c1
  double b_main, b_edge, b_off1, b_off2;
};

CHP_DEV BandConst band_const(double a, double b, const G1& g) {
  BandConst k;
  k.a_lmain = a * (-2.0 * g.c1);
  k.ma_loff = (-a) * g.c1;
  k.b_main = b * g.s_main;
  k.b_edge = b * g.s_edge;
  k.b_off1 = b * g.s_off1;
  k.b_off2 = b * g.s_off2;
  return k;
}

// Row r of I - a L diag(c) + b L^2 given c_{r-1}, c_r, c_{r+1}.
CHP_DEV void band_row(int r, int m, const BandConst& k, double cm, double c0, double cp,
                      double e[5]) {
  const double bm = (r == 0 || r == m - 1) ? k.b_edge : k.b_main;
  e[0] = (r >= 2) ? k.b_off2 : 0.0;
  e[1] = (r >= 1) ? k.ma_loff * cm + k.b_off1 : 0.0;
  e[2] = (1.0 - k.a_lmain * c0) + bm;
  e[3] = (r + 1 < m) ? k.ma_loff * cp + k.b_off1 : 0.0;
  e[4] = (r + 2 < m) ? k.b_off2 : 0.0;
}

// ---------------------------------------------------------------------------
// One step of each scheme for one system.  `src` may equal `dst`.
// ---------------------------------------------------------------------------

// LINEAR_A: (I - dt L diag(v^2) + b L^2) x = v - dt L v
CHP_DEV int step_linear_a(const G1& g, double dt, double b, const double* src, double* dst,
                          double* ub, long long ks) {
  const int m = g.m;
  const BandConst k = band_const(dt, b, g);
  auto load = [&](int r) { return make_double2(ld(src, r + 1, m), 0.0); };
  auto make = [&](int r, double vm, double v0, double vp, double, double e[5], double& rhs) {
    band_row(r, m, k, vm * vm, v0 * v0, vp * vp, e);
    rhs = v0 - dt * lap3(vm, v0, vp, g.c1);
  };
  const int sing = band_lu_forward(m, load, make, ub, ks);
  const bool fin = band_lu_backward(m, ub, ks, dst);
  return sing ? CHP_SYS_SINGULAR : (fin ? CHP_SYS_OK : CHP_SYS_NONFINITE);
}

// LINEAR_B with the cached Cholesky factor fac = [F0 | F1 | F2] (3*m):
// F2 = diagonal of U, F1[i] = U[i-1,i], F0[i] = U[i-2,i]  (LAPACK 'U' band).
CHP_DEV bool step_linear_b(const G1& g, double dt, const double* __restrict__ fac,
                           const double* src, double* dst, double* yb, long long ks) {
  const int m = g.m;
  const double* F0 = fac;
  const double* F1 = fac + m;
  const double* F2 = fac + 2 * m;
  const double* R2 = fac + 3 * m;               // RN(1 / F2[i])
  // forward: rhs_i on the fly, then U^T y = rhs (dtbsv 'U','T': dot then divide)
  double v0 = src[0];
  double w_m = 0.0;
  double w_0 = chp_cube_minus_3v(v0);
  double y1 = 0.0, y2 = 0.0;  // y_{i-1}, y_{i-2}
  #pragma unroll 8
  for (int i = 0; i < m; ++i) {
    const double vp = (i + 1 < m) ? src[i + 1] : 0.0;
    const double w_p = (i + 1 < m) ? chp_cube_minus_3v(vp) : 0.0;
    const double rhs = v0 + dt * lap3(w_m, w_0, w_p, g.c1);
    double dot = 0.0;
    if (i >= 2) dot = fma(y2, F0[i], dot);
    if (i >= 1) dot = fma(y1, F1[i], dot);
    const double yi = div_rn(rhs - dot, F2[i], R2[i]);
    yb[(long long)i * ks] = yi;
    y2 = y1; y1 = yi;
    w_m = w_0; w_0 = w_p; v0 = vp;
  }
  // backward: U x = y (dtbsv 'U','N': divide then axpy)
  double x1 = 0.0, x2 = 0.0;
  bool fin = true;
  #pragma unroll 8
  for (int i = m - 1; i >= 0; --i) {
    double t = yb[(long long)i * ks];
    if (i + 2 < m) t = fma(-x2, F0[i + 2], t);
    if (i + 1 < m) t = fma(-x1, F1[i + 1], t);
    const double xi = div_rn(t, F2[i], R2[i]);
    x2 = x1; x1 = xi;
    dst[i] = xi;
    fin = fin && isfinite(xi);
  }
  return fin;
}

// EYRE: Newton on H(Y) = Y + b L^2 Y - d L Y^3 - yhat, yhat = u - d L u.
// Returns the CHP_SYS_* status; on success *iters/*res hold the accepted
// iteration count and residual (StepReport fields, schemes.py:291-300).
CHP_DEV int step_eyre(const G1& g, double d, double b, double tol, int maxit,
                      const double* src, double* dst, double* yh, double* ub, long long ks,
                      int* iters, double* res, double* hist, int hlen) {
  const int m = g.m;
  #pragma unroll 8
  for (int i = 0; i < m; ++i) {
    const double u0 = src[i];
    yh[(long long)i * ks] = u0 - d * lap3(ld(src, i - 1, m), u0, ld(src, i + 1, m), g.c1);
  }
  if (dst != src)
    for (int i = 0; i < m; ++i) dst[i] = src[i];
  double* y = dst;
  const double d2 = 2.0 * d;
  const BandConst k = band_const(3.0 * d, b, g);
  for (int it = 0; it <= maxit; ++it) {
    // residual H and its cell-weighted L2 norm (schemes.py:287-289, grid.py:147-149)
    double ss = 0.0;
    {
      double ym2 = 0.0, ym1 = 0.0, y0 = y[0], yp1 = ld(y, 1, m);
      double cm = 0.0, c0 = chp_cube(y0);
#if CHP_1D_RQ > 0
      // y_{i+2} and yhat_i travel kRQ rows ahead of the (sequential) norm accumulation in a
      // register queue: the yhat rows are interleaved over the systems and always come from
      // L2, which an unrolled loop alone left exposed once per unrolled group of rows
      double yq[kRQ], hq[kRQ];
#pragma unroll
      for (int q = 0; q < kRQ; ++q) {
        yq[q] = ld(y, q + 2, m);
        hq[q] = (q < m) ? yh[(long long)q * ks] : 0.0;
      }
      auto row = [&](int i, double yp2, double yhi) {
        const double cp = (i + 1 < m) ? chp_cube(yp1) : 0.0;
        const double s0 = (i == 0 || i == m - 1) ? g.s_edge : g.s_main;
        const double H = ((y0 + b * bilap5(ym2, ym1, y0, yp1, yp2, s0, g)) -
                          d * lap3(cm, c0, cp, g.c1)) - yhi;
        ss = ss + H * H;
        ym2 = ym1; ym1 = y0; y0 = yp1; yp1 = yp2;
        cm = c0; c0 = cp;
      };
      int i0 = 0;
      for (; i0 + kRQ <= m; i0 += kRQ) {
        double yc[kRQ], hc[kRQ];
#pragma unroll
        for (int q = 0; q < kRQ; ++q) {
          yc[q] = yq[q];
          hc[q] = hq[q];
          yq[q] = ld(y, i0 + q + kRQ + 2, m);
          hq[q] = (i0 + q + kRQ < m) ? yh[(long long)(i0 + q + kRQ) * ks] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kRQ; ++q) row(i0 + q, yc[q], hc[q]);
      }
#pragma unroll
      for (int q = 0; q < kRQ; ++q)
        if (i0 + q < m) row(i0 + q, yq[q], hq[q]);
    }
#else
      #pragma unroll 8
      for (int i = 0; i < m; ++i) {
        const double yp2 = ld(y, i + 2, m);
        const double cp = (i + 1 < m) ? chp_cube(yp1) : 0.0;
        const double s0 = (i == 0 || i == m - 1) ? g.s_edge : g.s_main;
        const double H = ((y0 + b * bilap5(ym2, ym1, y0, yp1, yp2, s0, g)) -
                          d * lap3(cm, c0, cp, g.c1)) - yh[(long long)i * ks];
        ss = ss + H * H;
        ym2 = ym1; ym1 = y0; y0 = yp1; yp1 = yp2;
        cm = c0; c0 = cp;
      }
    }
#endif
    const double r = sqrt(g.hd * ss);
    if (hist != nullptr && it < hlen) hist[it] = r;   // StepReport.residual_history
    if (r <= tol) {
      *iters = it;
      *res = r;
      return CHP_SYS_OK;
    }
    if (it == maxit || !isfinite(r)) {
      *iters = it;
      *res = r;
      return CHP_SYS_NEWTON;
    }
    // (I + b L^2 - 3d L diag(y^2)) y_new = yhat - 2d L y^3   (schemes.py:303-304)
    auto load = [&](int rr) {
      return make_double2(ld(y, rr + 1, m),
                          (rr >= 0 && rr < m) ? yh[(long long)rr * ks] : 0.0);
    };
    auto make = [&](int rr, double ym, double y0, double yp, double yhr, double e[5],
                    double& rhs) {
      band_row(rr, m, k, ym * ym, y0 * y0, yp * yp, e);
      const double cm = (rr >= 1) ? chp_cube(ym) : 0.0;
      const double cp = (rr + 1 < m) ? chp_cube(yp) : 0.0;
      rhs = yhr - d2 * lap3(cm, chp_cube(y0), cp, g.c1);
    };
    if (band_lu_forward(m, load, make, ub, ks)) return CHP_SYS_SINGULAR;
    (void)band_lu_backward(m, ub, ks, y);   // a non-finite y makes the next residual non-finite
  }
  return CHP_SYS_NEWTON;  // unreachable
}

struct Scratch1 {   // per-launch interleaved scratch
  double* ub;       // [m][6][nthreads]
  double* yh;       // [m][nthreads]
  double* tmp;      // [m][nthreads] (coarse sweep: g)
  long long ks;     // nthreads
  double* hist;     // Newton residual history [nsys'][hlen] (chp_propagate_hist) or null
  int hlen;
};

// One step of `scheme` for thread t.  Returns CHP_SYS_* and updates info.
CHP_DEV int one_step(const G1& g, const chp_spec& sp, const double* fac, const double* src,
                     double* dst, const Scratch1& S, int t, SysInfo* info,
                     double* hist = nullptr) {
  int st = CHP_SYS_OK;
  double* ub = S.ub + t;
  double* yh = S.yh + t;
  if (sp.scheme == CHP_LINEAR_B) {
    if (!step_linear_b(g, sp.dt, fac, src, dst, yh, S.ks)) st = CHP_SYS_NONFINITE;
  } else if (sp.scheme == CHP_LINEAR_A) {
    st = step_linear_a(g, sp.dt, sp.b, src, dst, ub, S.ks);
  } else {
    // EYRE: an accepted step has a finite residual, hence a finite iterate
    // (schemes.py:287-302 raises before the Field check otherwise)
    int it = 0;
    double r = 0.0;
    st = step_eyre(g, sp.dt, sp.b, sp.newton_tol, sp.newton_max_iter, src, dst, yh, ub, S.ks,
                   &it, &r, hist, S.hlen);
    if (st == CHP_SYS_OK) {
      info->newton_steps += 1;
      info->newton_total += it;
      info->newton_max = max(info->newton_max, it);
      info->newton_maxres = fmax(info->newton_maxres, r);
    } else if (st == CHP_SYS_NEWTON) {
      sysinfo_fail(info, st, it, r);
      return st;
    }
  }
  if (st != CHP_SYS_OK) {
    sysinfo_fail(info, st, 0, 0.0);
    return st;
  }
  return CHP_SYS_OK;
}

}  // namespace

// dpbtf2 ('U', KD=2) of I - 2dt L + eps^2 dt L^2 (schemes.py:207-213), LAPACK
// order with the FMA-contracted OpenBLAS dsyr update.  One thread.
__global__ void k1d_pbtf2(chp_grid gg, double dt, double b, double* fac, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const G1 g = make_g1(gg);
  const int m = g.m;
  double* A0 = fac;
  double* A1 = fac + m;
  double* A2 = fac + 2 * m;
  const double a = 2.0 * dt;
  const double lap_main = -2.0 * g.c1, lap_off = g.c1;
  for (int j = 0; j < m; ++j) {
    const double sm = (j == 0 || j == m - 1) ? g.s_edge : g.s_main;
    A2[j] = (1.0 - a * lap_main) + b * sm;
    A1[j] = (j >= 1) ? (-a) * lap_off + b * g.s_off1 : 0.0;
    A0[j] = (j >= 2) ? b * g.s_off2 : 0.0;
  }
  int info = 0;
  for (int j = 0; j < m; ++j) {
    double ajj = A2[j];
    if (!(ajj > 0.0)) { info = j + 1; break; }
    ajj = sqrt(ajj);
    A2[j] = ajj;
    const int kn = min(2, m - 1 - j);
    if (kn > 0) {
      const double r = 1.0 / ajj;
      const double x0 = A1[j + 1] * r;
      A1[j + 1] = x0;
      double x1 = 0.0;
      if (kn > 1) { x1 = A0[j + 2] * r; A0[j + 2] = x1; }
      A2[j + 1] = fma(x0, -x0, A2[j + 1]);
      if (kn > 1) {
        A1[j + 2] = fma(x0, -x1, A1[j + 2]);
        A2[j + 2] = fma(x1, -x1, A2[j + 2]);
      }
    }
  }
  if (info == 0)
    for (int j = 0; j < m; ++j) fac[3 * m + j] = 1.0 / A2[j];   // RN(1/U_jj)
  *err = info;
}

// `steps` steps of one scheme on nsys systems (thread per system).
__global__ void k1d_propagate(chp_grid gg, chp_spec sp, int steps, int nsys,
                              const double* __restrict__ in, long long in_stride,
                              double* out, long long out_stride, const int* sys_index,
                              const double* fac, Scratch1 S, chp_sys_info* info_) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsys) return;
  const G1 g = make_g1(gg);
  const int sidx = sys_index ? sys_index[t] : t;
  const double* src = in + (long long)sidx * in_stride;
  double* dst = out + (long long)sidx * out_stride;
  SysInfo* info = reinterpret_cast<SysInfo*>(info_) + sidx;
  SysInfo loc = *info;
  if (loc.status == CHP_SYS_OK) {
    for (int s = 0; s < steps; ++s) {
      if (one_step(g, sp, fac, (s == 0) ? src : dst, dst, S, t, &loc,
                   S.hist ? S.hist + (long long)sidx * S.hlen : nullptr) != CHP_SYS_OK)
        break;
    }
  }
  *info = loc;
}

// Coarse init (mode 0) / coarse sweep + correction (mode 1), thread per IC.
__global__ void k1d_coarse_sweep(chp_grid gg, chp_spec sp, int mode, int nic, int nsl, int n0,
                                 int n1, double* U, const double* F, double* G,
                                 long long ic_stride, long long sl_stride, unsigned char* changed,
                                 double* inc, const double* fac, Scratch1 S,
                                 chp_sys_info* info_) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nic) return;
  const G1 g = make_g1(gg);
  const int m = g.m;
  SysInfo* info = reinterpret_cast<SysInfo*>(info_) + i;
  SysInfo loc = *info;
  double* Ui = U + (long long)i * ic_stride;
  const double* Fi = F ? F + (long long)i * ic_stride : nullptr;
  double* Gi = G + (long long)i * ic_stride;
  unsigned char* ch = changed ? changed + (long long)i * (nsl + 1) : nullptr;
  double* gt = S.tmp + i;
  double dmax = 0.0;
  if (mode == 1 && (ch[0] & 2)) return;  // IC frozen (converged in a batch run)
  for (int n = n0; n < n1 && loc.status == CHP_SYS_OK; ++n) {
    const double* un = Ui + (long long)n * sl_stride;
    double* un1 = Ui + (long long)(n + 1) * sl_stride;
    double* gn = Gi + (long long)n * sl_stride;
    if (mode == 0) {
      if (one_step(g, sp, fac, un, un1, S, i, &loc) != CHP_SYS_OK) break;
      for (int j = 0; j < m; ++j) gn[j] = un1[j];
      continue;
    }
    // U_n unchanged since G[n] was computed -> G(U_n) == G[n] bit for bit.
    const bool redo = ch[n] != 0;
    bool any = false;
    if (redo) {
      // stage the old U_{n+1} in the interleaved temp, compute g into the
      // U_{n+1} slot, then form the correction in place
      for (int j = 0; j < m; ++j) gt[(long long)j * S.ks] = un1[j];
      if (one_step(g, sp, fac, un, un1, S, i, &loc) != CHP_SYS_OK) break;
      const double* fn = Fi + (long long)n * sl_stride;
      for (int j = 0; j < m; ++j) {
        const double gj = un1[j];
        const double nv = (gj + fn[j]) - gn[j];
        const double ov = gt[(long long)j * S.ks];
        any = any || (__double_as_longlong(nv) != __double_as_longlong(ov));
        dmax = fmax(dmax, fabs(nv - ov));
        if (!isfinite(nv)) sysinfo_fail(&loc, CHP_SYS_NONFINITE, 0, 0.0);
        gn[j] = gj;
        un1[j] = nv;
      }
    } else {
      const double* fn = Fi + (long long)n * sl_stride;
      for (int j = 0; j < m; ++j) {
        const double gj = gn[j];
        const double nv = (gj + fn[j]) - gj;
        const double ov = un1[j];
        any = any || (__double_as_longlong(nv) != __double_as_longlong(ov));
        dmax = fmax(dmax, fabs(nv - ov));
        if (!isfinite(nv)) sysinfo_fail(&loc, CHP_SYS_NONFINITE, 0, 0.0);
        un1[j] = nv;
      }
    }
    ch[n + 1] = any ? 1 : 0;
  }
  if (mode == 1 && inc) atomic_max_nonneg(inc + i, dmax);
  *info = loc;
}

// ---------------------------------------------------------------------------
// host launchers (called from chp_api.cu)
// ---------------------------------------------------------------------------
cudaError_t chp1d_factor(const chp_grid& g, double dt, double b, double* fac, int* err,
                         cudaStream_t st) {
  k1d_pbtf2<<<1, 1, 0, st>>>(g, dt, b, fac, err);
  return cudaGetLastError();
}

cudaError_t chp1d_propagate(const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                            const double* in, long long in_stride, double* out,
                            long long out_stride, const int* sys_index, const double* fac,
                            double* ub, double* yh, double* tmp, chp_sys_info* info,
                            cudaStream_t st, double* hist, int hlen) {
  Scratch1 S{ub, yh, tmp, nsys, hist, hlen};
  const int bs = 32;
  const int smem = sp.scheme == CHP_LINEAR_B ? 0 : kRingBytes;
  k1d_propagate<<<(nsys + bs - 1) / bs, bs, smem, st>>>(g, sp, steps, nsys, in, in_stride, out,
                                                     out_stride, sys_index, fac, S, info);
  return cudaGetLastError();
}

cudaError_t chp1d_coarse_sweep(const chp_grid& g, const chp_spec& sp, int mode, int nic, int nsl,
                               int n0, int n1, double* U, const double* F, double* G,
                               long long ic_stride, long long sl_stride, unsigned char* changed,
                               double* inc, const double* fac, double* ub, double* yh,
                               double* tmp, chp_sys_info* info, cudaStream_t st) {
  Scratch1 S{ub, yh, tmp, nic};
  const int bs = 32;
  const int smem = sp.scheme == CHP_LINEAR_B ? 0 : kRingBytes;
  k1d_coarse_sweep<<<(nic + bs - 1) / bs, bs, smem, st>>>(g, sp, mode, nic, nsl, n0, n1, U, F, G,
                                                       ic_stride, sl_stride, changed, inc, fac,
                                                       S, info);
  return cudaGetLastError();
}
