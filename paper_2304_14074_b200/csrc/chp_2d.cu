// 2D propagators (configs 3-5): batched DST-I spectral solves.
//
// Field layout: [m rows (x, i)][pitch N = m+1 doubles (y, j)], N a power of
// two.  Storage column j holds math index j: column 0 is the zero Dirichlet
// pad, columns 1..m the interior -- so the pair (2k, 2k+1) of a row is one
// aligned double2.  All transforms are unnormalised DST-I (T^2 = (N/2) I,
// chp_wdst.cuh); the orthonormal 2D transform is S = (2/N) T_i T_j and every
// normalisation folds into one scale per solve.
//
// LINEAR_B (schemes.py:249-267):  x = S D S rhs,  D = 1/(1 - 2dt lam + eps^2 dt lam^2),
// lam = lam_p + lam_q (grid.py:127-144 eigenvalues in the sin^2 form).
// One step = two passes over HBM (32 B per grid-point-step):
//   row pass    (tile of TR rows + 1 halo row on each side; one lane group
//                per row pair):  x = T_j P (registers) -> w = x^3 - 3x (SMEM)
//                -> Q = (N/2) P + dt T_j(L w)      [T_j x = (N/2) P exactly]
//                (first step: Q = T_j(x + dt L w) from the physical input)
//   column pass (tile of TC columns, all rows, one lane group per column pair):
//                P = T_i (D' .* T_i Q),  D' = (2/N)^2 D
// J steps = J+1 row passes + J column passes, every slice of every IC in
// each launch.
#include <cooperative_groups.h>
#include <math.h>

#include <map>
#include <stdlib.h>
#include <string>
#include <vector>

#include "chp_common.cuh"
#include "chp_dst.cuh"
#include "chp_wdst.cuh"
#include "chp_linb.cuh"

using chpdst::Tables;

namespace {

constexpr int kMinN = 8;
constexpr int kMaxN = 1024;

// configuration of the smem (radix-4 Stockham) passes used by the PCG
template <int N> struct Cfg {
  static constexpr int T = (N >= 1024) ? 128 : (N >= 512 ? 64 : 32);  // threads / pair
  static constexpr int G = 4;                                          // pairs / block
  static constexpr int TC = 2 * G;                                     // cols / col tile
  static constexpr int THREADS = G * T;
  static constexpr size_t COL_SMEM = sizeof(double) * (size_t)TC * N + sizeof(double) * G * (T / 32);
};

// configuration of the register-resident (wdst) LINEAR_B passes
template <int N> struct WCfg {
  static constexpr int L = wdst::Geo<N>::L;
  static constexpr int WARPS = (N >= 1024) ? 8 * (L / 32) : ((N >= 64) ? 8 : 1);
  static constexpr int THREADS = WARPS * 32;
  static constexpr int GPB = THREADS / L;          // lane groups (pairs) per block
  static constexpr int ROWS = 2 * GPB;             // rows held per row tile (incl. halo)
  static constexpr int TR = ROWS - 2;              // inner rows per row tile
  static constexpr int TC = (2 * GPB < N) ? 2 * GPB : N;   // columns per column tile
  static constexpr int MINB = (N <= 256) ? 2 : 1;          // blocks/SM the registers allow
  static constexpr size_t ROW_SMEM = sizeof(double) * (size_t)ROWS * N + 16 * (size_t)(N + 64);
  static constexpr size_t COL_SMEM = sizeof(double) * (size_t)(2 * GPB) * N + 16 * (size_t)N;
};

// column pass: smaller blocks (no halo), so that two blocks overlap on an SM
template <int N> struct WCfgC {
  static constexpr int L = wdst::Geo<N>::L;
  static constexpr int WARPS = (N >= 1024) ? 4 * (L / 32) : ((N >= 64) ? 4 : 1);
  static constexpr int MINB = (N <= 256) ? 4 : 2;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int GPB = THREADS / L;
  static constexpr int TC = (2 * GPB < N) ? 2 * GPB : N;
  static constexpr size_t COL_SMEM = sizeof(double) * (size_t)(2 * GPB) * N + 16 * (size_t)(N + 64);
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
  chp_sys_info* info;    // per-system outcome, indexed through info_index
  const int* info_index;
  const double2* wtab;   // wdst lane tables for N
};

CHP_DEV double w_of(double x) { return fma(x, x * x, -3.0 * x); }   // x^3 - 3x

// ---------------------------------------------------------------------------
// LINEAR_B row pass
// ---------------------------------------------------------------------------
CHP_DEV void cp_async16(void* sdst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
CHP_DEV void cp_async8(void* sdst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
CHP_DEV void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <int N>
__global__ void __launch_bounds__(WCfg<N>::THREADS, WCfg<N>::MINB)
k2d_row_pass(RowArgs a) {
  using C = WCfg<N>;
  constexpr int L = C::L;
  extern __shared__ __align__(16) double sm[];   // ROWS rows of N (swizzled rsw) + twiddles
  double2* twt = reinterpret_cast<double2*>(sm + (size_t)C::ROWS * N);
  const int tid = threadIdx.x;
  const int g = tid / L, l = tid % L;
  const int s = blockIdx.y;
  const int m = a.m;
  const int i0 = blockIdx.x * C::TR;              // first inner row of the tile
  const long long fin = a.in_index ? a.in_index[s] : s;
  const long long fout = a.out_index ? a.out_index[s] : s;
  const double* __restrict__ in = a.in + fin * a.in_stride;
  double* __restrict__ out = a.out + fout * a.out_stride;
  // all ROWS input rows (P, or U for the first step) in flight at once
  for (int idx = tid; idx < C::ROWS * (N / 2); idx += C::THREADS) {
    const int r = idx / (N / 2), jj = 2 * (idx % (N / 2));
    const int row = i0 - 1 + r;
    double* d = sm + (size_t)r * N + wdst::rsw(jj);
    if (row >= 0 && row < m) cp_async16(d, in + (long long)row * N + jj);
    else *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);
  }
  wdst::load_twiddles<N>(twt, a.wtab + N);
  const double2 ac = __ldg(&a.wtab[l]);
  cp_async_wait_all();
  __syncthreads();
  double* wr0 = sm + (size_t)(2 * g) * N;         // this group's two tile rows
  double* wr1 = wr0 + N;
  double2* scr = reinterpret_cast<double2*>(wr0);
  const bool last = a.mode == ROW_LAST;
  const double c = a.c1, c4 = -4.0 * a.c1, dt = a.dt;
  constexpr int PL = N / L;                       // values per lane per row
  // phase 0: x = T_j P of tile rows (2g, 2g+1)      (skipped for the first step)
  // phase 1: Q = T_j(x + dt L(x^3 - 3x)) of inner tile rows (1+2g, 2+2g)
  // One pair_dst call site for both phases keeps the kernel's code small.
#pragma unroll 1
  for (int ph = (a.mode == ROW_FIRST) ? 1 : 0; ph < 2; ++ph) {
    const int ra = (ph == 0) ? i0 - 1 + 2 * g : i0 + 2 * g;     // global rows of the pair
    const int rb = ra + 1;
    const bool active = (ph == 0) || (g < C::GPB - 1);
    bool oa, ob;                                                // rows this group outputs
    if (ph == 0) {
      oa = ra >= i0 && ra < i0 + C::TR && ra < m;
      ob = rb >= i0 && rb < i0 + C::TR && rb < m;
    } else {
      oa = active && ra < m;
      ob = active && rb < m;
      // rhs = x + dt L w, w = x^3 - 3x, for the lane's contiguous chunk of
      // PL points of rows r0 and r0+1: pairs (n, n+1) read as double2 from the
      // tile (conflict free under rsw), w computed once per value read, the
      // horizontal neighbours carried in registers.  Stencil order as the
      // reference's CSR matvec: (i-1,j), (i,j-1), (i,j), (i,j+1), (i+1,j).
      double la[PL], lb[PL];
      const int r0 = 1 + 2 * g;
      const int nb = l * PL;
      auto ld2 = [&](int r, int n) -> double2 {
        return *reinterpret_cast<const double2*>(sm + (size_t)r * N + wdst::rsw(n));
      };
      auto w2 = [](double2 v) { return make_double2(w_of(v.x), w_of(v.y)); };
      if (active) {
        double wam = 0.0, wbm = 0.0;                 // w at n - 1
        if (nb > 0) {
          wam = w_of(sm[(size_t)r0 * N + wdst::rsw(nb - 1)]);
          wbm = w_of(sm[(size_t)(r0 + 1) * N + wdst::rsw(nb - 1)]);
        }
        double2 xa = ld2(r0, nb), xb = ld2(r0 + 1, nb);
        double2 wa = w2(xa), wb = w2(xb);
#pragma unroll
        for (int j = 0; j < PL / 2; ++j) {
          const int n = nb + 2 * j;
          const bool more = n + 2 < N;
          const double2 xan = more ? ld2(r0, n + 2) : make_double2(0.0, 0.0);
          const double2 xbn = more ? ld2(r0 + 1, n + 2) : make_double2(0.0, 0.0);
          const double2 wup = w2(ld2(r0 - 1, n)), wdn = w2(ld2(r0 + 2, n));
          const double2 wan = w2(xan), wbn = w2(xbn);
          const double la0 = (((wup.x * c + wam * c) + wa.x * c4) + wa.y * c) + wb.x * c;
          const double la1 = (((wup.y * c + wa.x * c) + wa.y * c4) + wan.x * c) + wb.y * c;
          const double lb0 = (((wa.x * c + wbm * c) + wb.x * c4) + wb.y * c) + wdn.x * c;
          const double lb1 = (((wa.y * c + wb.x * c) + wb.y * c4) + wbn.x * c) + wdn.y * c;
          la[2 * j] = (n > 0) ? xa.x + dt * la0 : 0.0;
          lb[2 * j] = (n > 0) ? xb.x + dt * lb0 : 0.0;
          la[2 * j + 1] = xa.y + dt * la1;
          lb[2 * j + 1] = xb.y + dt * lb1;
          wam = wa.y; wbm = wb.y;
          xa = xan; xb = xbn; wa = wan; wb = wbn;
        }
      } else {
#pragma unroll
        for (int i = 0; i < PL; ++i) { la[i] = 0.0; lb[i] = 0.0; }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < PL / 2; ++j) {
        *reinterpret_cast<double2*>(wr0 + wdst::rsw(nb + 2 * j)) = make_double2(la[2 * j], la[2 * j + 1]);
        *reinterpret_cast<double2*>(wr1 + wdst::rsw(nb + 2 * j)) = make_double2(lb[2 * j], lb[2 * j + 1]);
      }
      wdst::group_sync<N>();
    }
    double fin = 0.0;
    auto ld = [&](int n, double& x, double& xm, double& y, double& ym) {
      const bool z0 = (n == 0);
      x = z0 ? 0.0 : wr0[wdst::rsw(n)];
      xm = z0 ? 0.0 : wr0[wdst::rsw(N - n)];
      y = z0 ? 0.0 : wr1[wdst::rsw(n)];
      ym = z0 ? 0.0 : wr1[wdst::rsw(N - n)];
    };
    auto st = [&](int k, double a2, double a21, double b2, double b21) {
      if (last) {                      // x * 0 is 0 unless x is NaN/Inf
        if (oa) fin = fma(a2, 0.0, fma(a21, 0.0, fin));
        if (ob) fin = fma(b2, 0.0, fma(b21, 0.0, fin));
      }
      if (ph == 1 || last) {
        if (oa) *reinterpret_cast<double2*>(out + (long long)ra * N + 2 * k) = make_double2(a2, a21);
        if (ob) *reinterpret_cast<double2*>(out + (long long)rb * N + 2 * k) = make_double2(b2, b21);
      } else {
        *reinterpret_cast<double2*>(wr0 + wdst::rsw(2 * k)) = make_double2(a2, a21);
        *reinterpret_cast<double2*>(wr1 + wdst::rsw(2 * k)) = make_double2(b2, b21);
      }
    };
    wdst::pair_dst<N>(ld, st, scr, twt, l, ac);
    if (last) {
      if (__syncthreads_or(fin != 0.0) && tid == 0) {
        const long long fi = a.info_index ? a.info_index[s] : s;
        atomicCAS(&a.info[fi].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
      }
      if (last) return;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// LINEAR_B column pass: P = T_i (D' .* T_i Q), in place
// ---------------------------------------------------------------------------
struct ColArgs {
  double* buf;
  long long stride;
  int m;
  const double* dtab;      // D'[q][p] = (2/N)^2 / ((1 - 2dt lam) + b lam^2), lam = lam_p + lam_q
  const double2* wtab;
};

// D' table for one (N, dt, eps): [q][p], zero on the pad row / column.  Exact
// division (the column pass only multiplies).
__global__ void k2d_build_dtab(int N, const double* lam, double a2dt, double b, double scale,
                               double* d) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)N * N) return;
  const int q = (int)(t / N), p = (int)(t % N);
  double v = 0.0;
  if (p > 0 && q > 0) {
    const double l = lam[p] + lam[q];
    v = scale / ((1.0 - a2dt * l) + b * (l * l));
  }
  d[t] = v;
}

// v2 layout (chp_linb.cuh): [q/2][n] double2 (D(n, q), D(n, q+1)), + 1 slack double2
__global__ void k2d_build_dtab2(int N, const double* lam, double a2dt, double b, double scale,
                                double* d) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)N * N + 2) return;
  double v = 0.0;
  if (t < (long long)N * N) {
    const int qp = (int)(t / (2 * N)), n = (int)((t / 2) % N), q = 2 * qp + (int)(t & 1);
    if (n > 0 && q > 0) {
      const double l = lam[n] + lam[q];
      v = scale / ((1.0 - a2dt * l) + b * (l * l));
    }
  }
  d[t] = v;
}

template <int N>
CHP_DEV int csw(int c, int n) { return c * N + (n ^ c ^ (((n >> 5) & 15) << 1)); }

template <int N>
__global__ void __launch_bounds__(WCfgC<N>::THREADS, WCfgC<N>::MINB)
k2d_col_pass_b(ColArgs a) {
  using C = WCfgC<N>;
  constexpr int L = C::L, TC = C::TC;
  extern __shared__ __align__(16) double sm[];    // 2*GPB columns of N (swizzled) + twiddles
  double2* twt = reinterpret_cast<double2*>(sm + (size_t)(2 * C::GPB) * N);
  const int tid = threadIdx.x;
  const int g = tid / L, l = tid % L;
  const int s = blockIdx.y;
  const int m = a.m;
  const int j0 = blockIdx.x * TC;                 // storage column of tile column 0
  double* buf = a.buf + (long long)s * a.stride;
  wdst::load_twiddles<N>(twt, a.wtab + N);
  const double2 ac = __ldg(&a.wtab[l]);
  // logical (column c, math row n) at csw(c, n)
  for (int idx = tid; idx < N * TC; idx += C::THREADS) {
    const int n = idx / TC, cc = idx % TC;
    if (n > 0) cp_async8(&sm[csw<N>(cc, n)], buf + (long long)(n - 1) * N + j0 + cc);
    else sm[csw<N>(cc, n)] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  // groups beyond the tile (small N) run on zeros so every lane of the warp
  // takes part in pair_dst's shuffles / __syncwarp
  const int ca = 2 * g, cb = ca + 1;
  const bool grp = ca < TC;
  double2* scr = reinterpret_cast<double2*>(sm + (size_t)ca * N);
  const int qa = j0 + ca, qb = j0 + cb;           // math column indices
  bool scale_pass = true;
  auto ld = [&](int n, double& x, double& xm, double& y, double& ym) {
    const bool z = !grp || n == 0;
    x = z ? 0.0 : sm[csw<N>(ca, n)];
    xm = z ? 0.0 : sm[csw<N>(ca, N - n)];
    y = z ? 0.0 : sm[csw<N>(cb, n)];
    ym = z ? 0.0 : sm[csw<N>(cb, N - n)];
  };
  const double* __restrict__ da = a.dtab + (long long)(grp ? qa : 0) * N;
  const double* __restrict__ db = a.dtab + (long long)(grp ? qb : 0) * N;
  auto st = [&](int k, double a2, double a21, double b2, double b21) {
    if (!grp) return;
    if (scale_pass) {
      const double2 sa = __ldg(reinterpret_cast<const double2*>(da + 2 * k));
      const double2 sb = __ldg(reinterpret_cast<const double2*>(db + 2 * k));
      a2 *= sa.x;
      a21 *= sa.y;
      b2 *= sb.x;
      b21 *= sb.y;
    }
    sm[csw<N>(ca, 2 * k)] = a2;
    sm[csw<N>(ca, 2 * k + 1)] = a21;
    sm[csw<N>(cb, 2 * k)] = b2;
    sm[csw<N>(cb, 2 * k + 1)] = b21;
  };
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    scale_pass = (pass == 0);
    wdst::pair_dst<N>(ld, st, scr, twt, l, ac);
    wdst::group_sync<N>();
  }
  __syncthreads();
#pragma unroll 8
  for (int idx = tid; idx < m * TC; idx += C::THREADS) {
    const int i = idx / TC, cc = idx % TC;
    const int j = j0 + cc;
    buf[(long long)i * N + j] = (j > 0) ? sm[csw<N>(cc, i + 1)] : 0.0;
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
    sm[idx] = (j > 0 && row < m) ? in[(long long)row * N + j] : 0.0;
  }
  __syncthreads();
  chpdst::dst_pair<N, C::T>(sm + (size_t)g * 2 * N, tb, a.scale, ws + g * (C::T / 32), t, g + 1);
  __syncthreads();
  double part = 0.0;
  for (int idx = tid; idx < TRg * N; idx += C::THREADS) {
    const int r = idx / N, j = idx % N, row = i0 + r;
    if (row >= m) continue;
    double v = (j > 0) ? sm[(size_t)r * N + j] : 0.0;
    if (a.op == 1 && j > 0) {
      const double kap = -(a.lam[row + 1] + a.lam[j]);
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
    sm[(size_t)c * N + i + 1] = (j0 + c > 0) ? in[(long long)i * N + j0 + c] : 0.0;
  }
  if (tid < C::TC) sm[(size_t)tid * N] = 0.0;
  __syncthreads();
  double* pr = sm + (size_t)g * 2 * N;
  chpdst::dst_pair<N, C::T>(pr, tb, a.op == 0 ? a.scale : 1.0, ws + g * (C::T / 32), t, g + 1);
  if (a.op == 1) {
    const double* cs = a.c + (long long)s * a.stride;
    for (int idx = t; idx < 2 * N; idx += C::T) {
      const int c = 2 * g + idx / N, p = idx % N, q = j0 + c;
      if (p > 0 && q > 0) pr[idx] *= a.scale * cs[(long long)(p - 1) * N + q];
    }
    chpdst::group_sync(g + 1, C::T);
    chpdst::dst_pair<N, C::T>(pr, tb, 1.0, ws + g * (C::T / 32), t, g + 1);
  } else if (a.op == 2) {
    for (int idx = t; idx < 2 * N; idx += C::T) {
      const int c = 2 * g + idx / N, p = idx % N, q = j0 + c;
      if (p > 0 && q > 0) pr[idx] *= a.scale / (-(a.lam[p] + a.lam[q]));
    }
  }
  __syncthreads();
  for (int idx = tid; idx < m * C::TC; idx += C::THREADS) {
    const int i = idx / C::TC, c = idx % C::TC;
    out[(long long)i * N + j0 + c] = (j0 + c > 0) ? sm[(size_t)c * N + i + 1] : 0.0;
  }
}

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
struct CoopArgs {
  int m, nic, nsl, n0, n1, mode;
  double c1, dt, b, tol;
  int max_iter, pad_;
  double* U; const double* F; double* G; long long ics, sls;
  unsigned char* changed; double* inc; chp_sys_info* info;
  double *X, *Rv, *Pv, *Yv, *Cv, *CT;   // per-IC work fields (stride fs), nic-major
  double* Mi;                            // 1 / preconditioner (per IC, stride fs)
  double* Dk;                            // 1/kappa + b kappa ([m][N], shared by all ICs)
  double* part;                          // [2][gridDim][8] block partials
  unsigned int* bar;                     // grid barrier counter (zeroed by the host)
  const double* lam; const double2* wtab;
  unsigned long long* trace;             // optional: globaltimer after each barrier
  int trace_cap, pad2_;
};

// Grid-wide barrier for the co-resident (cooperative) launch: one relaxed
// spin per block and one fence on each side, instead of a fence per poll.
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
    __threadfence();
    atomicAdd(b.cnt, 1u);
    const unsigned int target = b.gen * gridDim.x;
    unsigned int v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b.cnt) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// lanes per pair in the cooperative coarse kernel: one pair per two warps at
// N = 1024 (a single field leaves most of the GPU idle with one warp per pair)
template <int N> struct CoopGeo {
  static constexpr int L = (N == 1024) ? 64 : wdst::Geo<N>::L;
  static constexpr int GPB = 256 / L;
  // op-1 operands (p rows, d rows) staged in shared memory when they fit
  static constexpr bool STAGE_P = (size_t)GPB * 6 * N * 8 + 16 * (size_t)(N + 64) <= 200 * 1024;
  static constexpr size_t SMEM =
      sizeof(double) * (size_t)GPB * (STAGE_P ? 6 : 2) * N + 16 * (size_t)(N + 64);
};

template <int N>
struct CoopCtx {
  const CoopArgs& a;
  double* sm;          // dynamic smem: GPB groups x 2N doubles (row pairs / column tile),
  double* sm2;         // [STAGE_P] GPB groups x 4N doubles (op-1 operands), then twiddles
  double2* twt;
  double* red;         // 32 doubles of static smem for block reductions
  int tid, g, l, gpb, ngroups, gg;
  double2 ac;
  CHP_DEV long long fs() const { return (long long)a.m * N; }
};

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
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = 0.0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) x += part[b * 8 + k];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (threadIdx.x == 0) red[k] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = red[k];
  __syncthreads();
}

// row-pair DST over the field: dst rows = T_j src rows (+ optional CG op)
//   op 0: dst = T_j src
//   op 1: dst = d .* p + T_j src ; returns thread partial of p.q
// With upd != nullptr the group first applies the CG direction update to its
// two rows in place, src = upd: P = R / M + beta P (no separate grid phase).
template <int N>
__device__ __noinline__ double coop_rows(CoopCtx<N>& x, const double* src, double* dst, int op,
                                         const double* p, double* upd = nullptr,
                                         const double* Rv = nullptr, double beta = 0.0,
                                         const double* Mi = nullptr) {
  constexpr int L = CoopGeo<N>::L;
  const auto& a = x.a;
  const int m = a.m;
  double part = 0.0;
  // the group's two source rows are staged in its scratch (cp.async, all in
  // flight at once) and consumed by in() before the FFT reuses the space
  double* rows = x.sm + (size_t)x.g * 2 * N;
  double2* scr = reinterpret_cast<double2*>(rows);
  // op 1: p rows and d rows (1/kappa + b kappa) staged in the second region
  double* prow = CoopGeo<N>::STAGE_P ? x.sm2 + (size_t)x.g * 4 * N : nullptr;
  // whole warps iterate together (pair_dst needs every lane of the warp);
  // groups without a pair run on zeros and store nothing
  for (int it = 0;; ++it) {
    const int pr = x.gg + it * x.ngroups;
    const bool have = pr < (m + 1) / 2;
    if (!__any_sync(0xffffffffu, have)) break;
    const int ra = have ? 2 * pr : 0, rb = ra + 1;
    const bool vb = have && rb < m;
    if (have) {
      const int nr = vb ? 2 : 1;
      if (upd) {
        // CG direction update of the two rows: P = R / M + beta P
        for (int h = 0; h < nr; ++h) {
          const long long o = (long long)(ra + h) * N;
          for (int n = x.l; n < N; n += L) {
            double v = 0.0;
            if (n > 0) {
              v = fma(beta, upd[o + n], Rv[o + n] * Mi[o + n]);
              upd[o + n] = v;
            }
            rows[h * N + n] = v;
          }
        }
      } else {
        for (int idx = x.l; idx < nr * (N / 2); idx += L) {
          const int h = idx / (N / 2), jj = 2 * (idx % (N / 2));
          cp_async16(rows + h * N + jj, src + (long long)(ra + h) * N + jj);
        }
      }
      if (op == 1 && prow) {
        for (int idx = x.l; idx < nr * (N / 2); idx += L) {
          const int h = idx / (N / 2), jj = 2 * (idx % (N / 2));
          cp_async16(prow + h * N + jj, p + (long long)(ra + h) * N + jj);
          cp_async16(prow + 2 * N + h * N + jj, a.Dk + (long long)(ra + h) * N + jj);
        }
      }
      cp_async_wait_all();
    }
    wdst::group_sync<N, L>();
    auto ld = [&](int n, double& u, double& um, double& v, double& vm) {
      const bool z = n == 0 || !have;
      u = z ? 0.0 : rows[n];
      um = z ? 0.0 : rows[N - n];
      v = (z || !vb) ? 0.0 : rows[N + n];
      vm = (z || !vb) ? 0.0 : rows[2 * N - n];
    };
    auto st = [&](int k, double a2, double a21, double b2, double b21) {
      if (!have) return;
      if (op == 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = ra + h;
          if (r >= m) break;
          double y0 = h ? b2 : a2, y1 = h ? b21 : a21;
          double2 pv, dv;
          if (prow) {
            pv = *reinterpret_cast<const double2*>(prow + h * N + 2 * k);
            dv = *reinterpret_cast<const double2*>(prow + 2 * N + h * N + 2 * k);
          } else {
            pv = *reinterpret_cast<const double2*>(p + (long long)r * N + 2 * k);
            dv = *reinterpret_cast<const double2*>(a.Dk + (long long)r * N + 2 * k);
          }
          if (k > 0) { y0 = fma(dv.x, pv.x, y0); part = fma(pv.x, y0, part); }
          else y0 = 0.0;
          y1 = fma(dv.y, pv.y, y1);
          part = fma(pv.y, y1, part);
          *reinterpret_cast<double2*>(dst + (long long)r * N + 2 * k) = make_double2(y0, y1);
        }
      } else {
        *reinterpret_cast<double2*>(dst + (long long)ra * N + 2 * k) = make_double2(a2, a21);
        if (vb) *reinterpret_cast<double2*>(dst + (long long)rb * N + 2 * k) = make_double2(b2, b21);
      }
    };
    wdst::pair_dst<N, L>(ld, st, scr, x.twt, x.l, x.ac);
    wdst::group_sync<N, L>();
  }
  return part;
}

// column-pair DST over the field (in place allowed):
//   op 0: dst = scale * T_i src
//   op 1: dst = T_i ((scale * c) .* T_i src)
//   op 2: dst = T_i src .* (scale / kappa)
template <int N>
__device__ __noinline__ void coop_cols(CoopCtx<N>& x, const double* src, double* dst, int op, double scale,
                       const double* cT) {
  // Block-tiled column pass: TC = 2*gpb columns per tile, coalesced tile
  // load/store through shared memory (swizzle csw), one lane group per pair.
  //   op 0: dst = scale * T_i src
  //   op 1: dst = T_i ((scale * c) .* T_i src)   (cT: c transposed, [q-1][n])
  //   op 2: dst = T_i src .* (scale / kappa)
  const auto& a = x.a;
  const int m = a.m;
  const int TC = (8 < N) ? 8 : N;            // small tiles: spread over all SMs
  const int ca = 2 * x.g, cb = ca + 1;
  double2* scr = reinterpret_cast<double2*>(x.sm + (size_t)ca * N);
  for (int tile = blockIdx.x; tile < N / TC; tile += gridDim.x) {
    const int j0 = tile * TC;
    for (int idx = threadIdx.x; idx < N * TC; idx += blockDim.x) {
      const int n = idx / TC, cc = idx % TC;
      if (n > 0 && j0 + cc > 0) cp_async8(&x.sm[csw<N>(cc, n)], src + (long long)(n - 1) * N + j0 + cc);
      else x.sm[csw<N>(cc, n)] = 0.0;
    }
    const int qa = j0 + ca, qb = j0 + cb;
    const bool act = ca < TC;
    // op 1: this group's two rows of c^T staged next to the tile
    double* crow = (CoopGeo<N>::STAGE_P && op == 1) ? x.sm2 + (size_t)x.g * 4 * N : nullptr;
    if (crow && act) {
      const double* ga = cT + (long long)(qa > 0 ? qa - 1 : 0) * N;
      const double* gb = cT + (long long)(qb - 1) * N;
      for (int jj = 2 * x.l; jj < N; jj += 2 * CoopGeo<N>::L) {
        cp_async16(crow + jj, ga + jj);
        cp_async16(crow + N + jj, gb + jj);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    auto ld = [&](int n, double& u, double& um, double& v, double& vm) {
      const bool z = n == 0 || !act;
      u = z ? 0.0 : x.sm[csw<N>(ca, n)];
      um = z ? 0.0 : x.sm[csw<N>(ca, N - n)];
      v = z ? 0.0 : x.sm[csw<N>(cb, n)];
      vm = z ? 0.0 : x.sm[csw<N>(cb, N - n)];
    };
    int pass = 0;
    auto st = [&](int k, double a2, double a21, double b2, double b21) {
      if (!act) return;
      const int p0 = 2 * k, p1 = p0 + 1;
      if (op == 1 && pass == 0) {
        // column qa = 0 is the pad (its outputs are zeroed below)
        const double2 c_a = crow ? *reinterpret_cast<const double2*>(crow + p0)
                                 : *reinterpret_cast<const double2*>(cT + (long long)(qa > 0 ? qa - 1 : 0) * N + p0);
        const double2 c_b = crow ? *reinterpret_cast<const double2*>(crow + N + p0)
                                 : *reinterpret_cast<const double2*>(cT + (long long)(qb - 1) * N + p0);
        a2 *= scale * c_a.x; a21 *= scale * c_a.y;
        b2 *= scale * c_b.x; b21 *= scale * c_b.y;
      } else if (op == 0) {
        a2 *= scale; a21 *= scale; b2 *= scale; b21 *= scale;
      } else if (op == 2) {
        a2 = (p0 > 0 && qa > 0) ? a2 * (scale / (-(a.lam[p0] + a.lam[qa]))) : 0.0;
        b2 = (p0 > 0) ? b2 * (scale / (-(a.lam[p0] + a.lam[qb]))) : 0.0;
        a21 = (qa > 0) ? a21 * (scale / (-(a.lam[p1] + a.lam[qa]))) : 0.0;
        b21 = b21 * (scale / (-(a.lam[p1] + a.lam[qb])));
      }
      x.sm[csw<N>(ca, p0)] = (qa > 0 && p0 > 0) ? a2 : 0.0;
      x.sm[csw<N>(ca, p1)] = (qa > 0) ? a21 : 0.0;
      x.sm[csw<N>(cb, p0)] = (p0 > 0) ? b2 : 0.0;
      x.sm[csw<N>(cb, p1)] = b21;
    };
    // every group runs (small N: several groups share a warp); groups beyond
    // the tile read zeros and store nothing
    wdst::pair_dst<N, CoopGeo<N>::L>(ld, st, scr, x.twt, x.l, x.ac);
    wdst::group_sync<N, CoopGeo<N>::L>();
    if (op == 1) {
      pass = 1;
      wdst::pair_dst<N, CoopGeo<N>::L>(ld, st, scr, x.twt, x.l, x.ac);
      wdst::group_sync<N, CoopGeo<N>::L>();
    }
    __syncthreads();
#pragma unroll 8
    for (int idx = threadIdx.x; idx < m * TC; idx += blockDim.x) {
      const int i = idx / TC, cc = idx % TC;
      const int j = j0 + cc;
      dst[(long long)i * N + j] = (j > 0) ? x.sm[csw<N>(cc, i + 1)] : 0.0;
    }
    __syncthreads();
  }
}

template <int N>
__global__ void __launch_bounds__(256, 1) k2d_coarse_coop(CoopArgs a) {
  GridBar grid{a.bar, 0u, a.trace, a.trace_cap};
  extern __shared__ __align__(16) double smc[];
  __shared__ double red[64];
  constexpr int L = CoopGeo<N>::L;
  CoopCtx<N> x{a};
  x.sm = smc;
  x.gpb = blockDim.x / L;
  x.sm2 = smc + (size_t)x.gpb * 2 * N;
  x.twt = reinterpret_cast<double2*>(smc + (size_t)x.gpb * (CoopGeo<N>::STAGE_P ? 6 : 2) * N);
  x.red = red;
  x.tid = threadIdx.x;
  x.g = x.tid / L;
  x.l = x.tid % L;
  x.ngroups = gridDim.x * x.gpb;
  x.gg = x.g * gridDim.x + blockIdx.x;       // spread pairs over all SMs first
  x.ac = __ldg(&a.wtab[x.l]);
  wdst::load_twiddles<N>(x.twt, a.wtab + N);
  __syncthreads();
  const int m = a.m;
  const long long fs = (long long)m * N;
  const long long tot = fs;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const double s2 = (2.0 / N) * (2.0 / N);
  const double tol2 = a.tol * a.tol;
  // d = 1/kappa + b kappa (the constant part of the operator and of M); visible
  // to all blocks after the first slice barrier
  for (long long t = gtid; t < tot; t += gstride) {
    const int i = (int)(t / N), j = (int)(t % N);
    double d = 0.0;
    if (j > 0) {
      const double kap = -(a.lam[i + 1] + a.lam[j]);
      d = 1.0 / kap + a.b * kap;
    }
    a.Dk[t] = d;
  }
  int pb = 0;                                      // alternating partial buffer

  for (int ic = 0; ic < a.nic; ++ic) {
    double* X = a.X + ic * fs;
    double* Rv = a.Rv + ic * fs;
    double* Pv = a.Pv + ic * fs;
    double* Yv = a.Yv + ic * fs;
    double* Cv = a.Cv + ic * fs;
    double* Mi = a.Mi + ic * fs;
    double* CT = a.CT + ic * fs;
    unsigned char* ch = a.changed ? a.changed + (long long)ic * (a.nsl + 1) : nullptr;
    double* Ui = a.U + ic * a.ics;
    double* Gi = a.G + ic * a.ics;
    const double* Fi = a.F ? a.F + ic * a.ics : nullptr;
    if (a.mode == 1 && (ch[0] & 2)) continue;    // IC frozen
    double dmax = 0.0;
    for (int n = a.n0; n < a.n1; ++n) {
      const double* un = Ui + (long long)n * a.sls;
      double* un1 = Ui + (long long)(n + 1) * a.sls;
      double* gn = Gi + (long long)n * a.sls;
      if (a.mode == 1 && blockIdx.x == 0 && threadIdx.x == 0) ch[n + 1] = 0;
      gbar(grid);                                   // ch[n] / U_n written by the previous slice
      const bool solve = (a.mode == 0) || (*(volatile unsigned char*)&ch[n] & 1);
      if (solve) {
        // ---- prep: rhs = v - dt L v (into Yv), c = v^2, sum c ------------------
        double sc[1] = {0.0};
        for (long long t = gtid; t < tot; t += gstride) {
          const int i = (int)(t / N), j = (int)(t % N);
          double r = 0.0, cv = 0.0;
          if (j > 0) {
            const double v = un[t];
            const double vu = i > 0 ? un[t - N] : 0.0, vd = i + 1 < m ? un[t + N] : 0.0;
            const double vl = j > 1 ? un[t - 1] : 0.0, vr = j < m ? un[t + 1] : 0.0;
            const double lv = ((((vu * a.c1 + vl * a.c1) + v * (-4.0 * a.c1)) + vr * a.c1) + vd * a.c1);
            r = v - a.dt * lv;
            cv = v * v;
          }
          Yv[t] = r;
          Cv[t] = cv;
          sc[0] += cv;
        }
        double* pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
        coop_block_partials<1>(sc, red, pbuf);
        gbar(grid);
        double tc[1];
        coop_total<1>(pbuf, red, tc);
        const double acbar = a.dt * (tc[0] / ((double)m * m));
        // c transposed for the column phases: CT[q-1][n] = c[n-1][q], q, n = 1..m;
        // the inverse preconditioner 1 / M, M = 1/kappa + b kappa + dt mean(c)
        for (long long t = gtid; t < tot; t += gstride) {
          const int q1 = (int)(t / N), nn = (int)(t % N);
          CT[t] = (nn > 0) ? Cv[(long long)(nn - 1) * N + q1 + 1] : 0.0;
          Mi[t] = (nn > 0) ? 1.0 / (a.Dk[t] + acbar) : 0.0;
        }
        // ---- b^ = (2/N)/kappa .* T_i T_j rhs -> Rv -----------------------------
        coop_rows<N>(x, Yv, Yv, 0, nullptr);
        gbar(grid);
        coop_cols<N>(x, Yv, Rv, 2, 2.0 / N, nullptr);
        gbar(grid);
        // ---- x = 0, p = r / M, rho = r.z, rr0 = r.r ---------------------------
        double pr[2] = {0.0, 0.0};
        for (long long t = gtid; t < tot; t += gstride) {
          const int i = (int)(t / N), j = (int)(t % N);
          X[t] = 0.0;
          double z = 0.0;
          if (j > 0) {
            const double rv = Rv[t];
            z = rv * Mi[t];
            pr[0] = fma(rv, z, pr[0]);
            pr[1] = fma(rv, rv, pr[1]);
          }
          Pv[t] = z;
        }
        pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
        coop_block_partials<2>(pr, red, pbuf);
        gbar(grid);
        double t0[2];
        coop_total<2>(pbuf, red, t0);
        double rho = t0[0];
        const double rr0 = t0[1];
        int it = 0;
        bool fail = false;
        bool done = !(rr0 > 0.0);
        double beta = 0.0;
        while (!done) {
          if (it == 0) coop_rows<N>(x, Pv, Yv, 0, nullptr);
          else coop_rows<N>(x, Pv, Yv, 0, nullptr, Pv, Rv, beta, Mi);
          gbar(grid);
          coop_cols<N>(x, Yv, Yv, 1, a.dt * s2, CT);
          gbar(grid);
          double pq[1];
          pq[0] = coop_rows<N>(x, Yv, Yv, 1, Pv);
          pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
          coop_block_partials<1>(pq, red, pbuf);
          gbar(grid);
          double tq[1];
          coop_total<1>(pbuf, red, tq);
          const double alpha = rho / tq[0];
          // X += alpha P, R -= alpha Q; (r.z, r.r).  Pad entries are zero in
          // every field (and Mi), so the loop runs over whole rows as double2.
          double rz[2] = {0.0, 0.0};
          {
            double2* X2 = reinterpret_cast<double2*>(X);
            double2* R2 = reinterpret_cast<double2*>(Rv);
            const double2* P2 = reinterpret_cast<const double2*>(Pv);
            const double2* Y2 = reinterpret_cast<const double2*>(Yv);
            const double2* M2 = reinterpret_cast<const double2*>(Mi);
#pragma unroll 4
            for (long long t = gtid; t < tot / 2; t += gstride) {
              double2 xv = X2[t], rv = R2[t];
              const double2 pv = P2[t], yv = Y2[t], mi = M2[t];
              xv.x = fma(alpha, pv.x, xv.x);
              xv.y = fma(alpha, pv.y, xv.y);
              rv.x = fma(-alpha, yv.x, rv.x);
              rv.y = fma(-alpha, yv.y, rv.y);
              X2[t] = xv;
              R2[t] = rv;
              rz[0] = fma(rv.x, rv.x * mi.x, rz[0]);
              rz[0] = fma(rv.y, rv.y * mi.y, rz[0]);
              rz[1] = fma(rv.x, rv.x, rz[1]);
              rz[1] = fma(rv.y, rv.y, rz[1]);
            }
          }
          pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
          coop_block_partials<2>(rz, red, pbuf);
          gbar(grid);
          double t1[2];
          coop_total<2>(pbuf, red, t1);
          beta = t1[0] / rho;
          rho = t1[0];
          ++it;
          if (!(t1[1] > tol2 * rr0)) done = true;
          else if (it >= a.max_iter) { done = true; fail = true; }
          if (!isfinite(t1[1])) { done = true; fail = true; }
        }
        if (gtid == 0) {
          a.info[ic].cg_total += it;
          a.info[ic].cg_max = max(a.info[ic].cg_max, it);
          if (fail) atomicCAS(&a.info[ic].status, CHP_SYS_OK, CHP_SYS_CG);
        }
        // ---- g = (2/N) T_i T_j x -> Yv ---------------------------------------
        coop_rows<N>(x, X, Yv, 0, nullptr);
        gbar(grid);
        coop_cols<N>(x, Yv, Yv, 0, 2.0 / N, nullptr);
        gbar(grid);
      }
      // ---- correction / init ---------------------------------------------------
      const double* gsrc = solve ? Yv : gn;
      bool any = false, bad = false;
      for (long long t = gtid; t < tot; t += gstride) {
        const int j = (int)(t % N);
        const double gv = (j > 0) ? gsrc[t] : 0.0;
        if (a.mode == 0) {
          un1[t] = gv;
          gn[t] = gv;
          bad |= !isfinite(gv);
          continue;
        }
        const double nv = (gv + Fi[(long long)n * a.sls + t]) - gn[t];
        const double ov = un1[t];
        any |= (__double_as_longlong(nv) != __double_as_longlong(ov));
        dmax = fmax(dmax, fabs(nv - ov));
        bad |= !isfinite(nv) || !isfinite(gv);
        un1[t] = nv;
        gn[t] = gv;
      }
      if (a.mode == 1) {
        // changed[n+1]: any block saw a differing bit (zeroed by the host first)
        if (__syncthreads_or(any) && threadIdx.x == 0) ch[n + 1] = 1;
      }
      if (__syncthreads_or(bad) && threadIdx.x == 0)
        atomicCAS(&a.info[ic].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
    }
    if (a.mode == 1) {
      for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      if ((threadIdx.x & 31) == 0) atomic_max_nonneg(a.inc + ic, dmax);
    }
    gbar(grid);
  }
}

#include "chp_coarse2.cuh"

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct NTables {
  double2* tw = nullptr;
  double* sj = nullptr;
  double* lam = nullptr;   // per-axis eigenvalues, index p = 1..m
  double2* wtab = nullptr; // wdst lane tables: (cos, sin)(pi l/N), then W_N^l
  double2* wtab_coop = nullptr;  // the same for the coarse kernel's 64-lane geometry (N = 1024)
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

template <int N>
void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k2d_row_pass<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)WCfg<N>::ROW_SMEM);
  cudaFuncSetAttribute(k2d_col_pass_b<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)WCfgC<N>::COL_SMEM);
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
                         double* scratch, const double* dtab, cudaStream_t st) {
  using C = WCfg<N>;
  set_smem_attrs<N>();
  const int m = g.m;
  const long long fs = (long long)m * N;
  double* buf[2] = {scratch, scratch + fs * nsys};
  using CC = WCfgC<N>;
  const dim3 rgrid((m + C::TR - 1) / C::TR, nsys), cgrid(N / CC::TC, nsys);
  ColArgs ca{nullptr, fs, m, dtab, nt.wtab};
  for (int s = 0; s < steps; ++s) {
    RowArgs ra{};
    ra.m = m; ra.dt = sp.dt; ra.c1 = g.c1; ra.info = info; ra.info_index = sys_index;
    ra.wtab = nt.wtab;
    if (s == 0) {
      ra.in = in; ra.in_stride = in_stride; ra.in_index = sys_index; ra.mode = ROW_FIRST;
    } else {
      ra.in = buf[(s - 1) & 1]; ra.in_stride = fs; ra.in_index = nullptr; ra.mode = ROW_MID;
    }
    ra.out = buf[s & 1]; ra.out_stride = fs; ra.out_index = nullptr;
    k2d_row_pass<N><<<rgrid, C::THREADS, C::ROW_SMEM, st>>>(ra);
    ca.buf = buf[s & 1];
    k2d_col_pass_b<N><<<cgrid, CC::THREADS, CC::COL_SMEM, st>>>(ca);
  }
  RowArgs ra{};
  ra.m = m; ra.dt = sp.dt; ra.c1 = g.c1; ra.info = info; ra.info_index = sys_index;
  ra.wtab = nt.wtab;
  ra.in = buf[(steps - 1) & 1]; ra.in_stride = fs; ra.in_index = nullptr; ra.mode = ROW_LAST;
  ra.out = out; ra.out_stride = out_stride; ra.out_index = sys_index;
  k2d_row_pass<N><<<rgrid, C::THREADS, C::ROW_SMEM, st>>>(ra);
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
  const dim3 rgrid(rtiles, nsys), cgrid(N / C::TC, nsys), egrid(kPB, nsys);
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
  struct DTab { int N; double a2dt, b, scale; int layout; double* d; };
  std::vector<DTab> dtabs;        // LINEAR_B spectral divisors, one per (N, dt, eps)
  void* coarse = nullptr;         // v2 coarse-sweep workspace
  size_t coarse_bytes = 0;
  void* pcg = nullptr;            // v2 batched PCG workspace
  size_t pcg_bytes = 0;
  double* pcg_tab = nullptr;      // Dk, SK (PI) for (pcg_tab_N, pcg_tab_b)
  int pcg_tab_N = 0;
  double pcg_tab_b = 0.0;
};

Chp2d* chp2d_create() { return new Chp2d(); }

void chp2d_destroy(Chp2d* c) {
  if (!c) return;
  for (auto& kv : c->tables) {
    cudaFree(kv.second.tw);
    cudaFree(kv.second.sj);
    cudaFree(kv.second.lam);
    cudaFree(kv.second.wtab);
    if (kv.second.wtab_coop) cudaFree(kv.second.wtab_coop);
  }
  if (c->scratch) cudaFree(c->scratch);
  for (auto& t : c->dtabs) cudaFree(t.d);
  if (c->work) cudaFree(c->work);
  if (c->coarse) cudaFree(c->coarse);
  if (c->pcg) cudaFree(c->pcg);
  if (c->pcg_tab) cudaFree(c->pcg_tab);
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
  // lane tables of a wdst geometry with wl lanes per group
  auto lane_tables = [&](int wl) {
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
    return wt;
  };
  const int wl = N == 8 ? 2 : N <= 32 ? 4 : N <= 128 ? 8 : N <= 512 ? 16 : wdst::Geo<1024>::L;
  const std::vector<double2> wt = lane_tables(wl);
  NTables t;
  cudaError_t e;
  if ((e = cudaMalloc(&t.wtab, sizeof(double2) * (2 * N + 64))) != cudaSuccess) return e;
  cudaMemcpy(t.wtab, wt.data(), sizeof(double2) * (2 * N + 64), cudaMemcpyHostToDevice);
  if (N == 1024 && wl != 64) {
    const std::vector<double2> wc = lane_tables(64);
    if ((e = cudaMalloc(&t.wtab_coop, sizeof(double2) * (2 * N + 64))) != cudaSuccess) return e;
    cudaMemcpy(t.wtab_coop, wc.data(), sizeof(double2) * (2 * N + 64), cudaMemcpyHostToDevice);
  }
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
  static bool attrs = false;
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
    k_pcg2_rows<N, 2><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 0);
    k_pcg2_warm_b<N><<<eg, 256, 0, st>>>(p);
    k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 5, tol * tol, 0, 0, 0);
  } else {
    k_pcg2_init<N><<<eg, 256, 0, st>>>(p);
    k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 0, 0, 0, 0, 0);
  }
  const int chunk = 8;
  std::vector<CgSys> host(nsys);
  for (int it0 = 0; it0 < max_iter + chunk; it0 += chunk) {
    for (int it = 0; it < chunk; ++it) {
      k_pcg2_rows<N, 1><<<rg, G2::THREADS, sm, st>>>(p, nullptr, p.Y, 1);
      k_pcg2_cols<N, 1><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k_pcg2_rows<N, 2><<<rg, G2::THREADS, sm, st>>>(p, p.Y, p.Y, 1);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, G2::RBLK, 1, 0, 0, 0, 0);
      k_pcg2_update<N><<<eg, 256, 0, st>>>(p);
      k2d_cg_reduce<<<red_blocks, 256, 0, st>>>(nsys, W.cg, W.partial, kPB, 2, tol * tol,
                                               max_iter, 0, 0);
    }
    if ((e = cudaMemcpyAsync(host.data(), W.cg, sizeof(CgSys) * nsys, cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    bool all = true;
    for (int s = 0; s < nsys; ++s) all = all && (!host[s].active || host[s].done);
    if (all) break;
  }
  // x = S x^ = sigma T'_i T'_j X -> W.Yv (external layout)
  k_pcg2_rows<N, 0><<<rg, G2::THREADS, sm, st>>>(p, p.X, p.Y, 0);
  k_pcg2_cols<N, 2><<<cgd, G2::THREADS, sm, st>>>(p, p.Y, W.Yv, 0);
  return cudaGetLastError();
}

template <int N>
cudaError_t pcg_dispatch(Chp2d* cx, const chp_grid& g, int nsys, double a, double b, double tol,
                         int max_iter, const NTables& nt, Work2& W, cudaStream_t st, int warm) {
  static const bool v1 = getenv("CHP_PCG_V1") != nullptr;   // A/B: previous passes
  static const bool cold = getenv("CHP_PCG_COLD") != nullptr;
  if (v1) return pcg_solve<N>(g, nsys, a, b, tol, max_iter, nt, W, st);
  return pcg_solve2<N>(cx, g, nsys, a, b, tol, max_iter, nt, W, st, cold ? 0 : warm);
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
      if ((e = pcg_dispatch<N>(cx, g, nsys, sp.dt, sp.b, tol, maxcg, nt, W, st, s > 0)) != cudaSuccess)
        return e;
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
      if ((e = pcg_dispatch<N>(cx, g, nsys, 3.0 * d, b, tol, maxcg, nt, W, st,
                               step > 0 || it > 0)) != cudaSuccess)
        return e;
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

cudaError_t get_dtab(Chp2d* c, int N, const chp_spec& sp, const NTables& nt, double scale,
                     int layout, const double** out, cudaStream_t st) {
  const double a2dt = 2.0 * sp.dt, b = sp.b;
  for (auto& t : c->dtabs)
    if (t.N == N && t.a2dt == a2dt && t.b == b && t.scale == scale && t.layout == layout) {
      *out = t.d;
      return cudaSuccess;
    }
  if (c->dtabs.size() >= 8) {              // bounded cache: drop the oldest table
    cudaStreamSynchronize(st);
    cudaFree(c->dtabs.front().d);
    c->dtabs.erase(c->dtabs.begin());
  }
  Chp2d::DTab t{N, a2dt, b, scale, layout, nullptr};
  cudaError_t e = cudaMalloc(&t.d, sizeof(double) * ((size_t)N * N + 2));
  if (e != cudaSuccess) return e;
  const long long n = (long long)N * N + 2;
  if (layout == 0)
    k2d_build_dtab<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(N, nt.lam, a2dt, b, scale, t.d);
  else
    k2d_build_dtab2<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(N, nt.lam, a2dt, b, scale, t.d);
  c->dtabs.push_back(t);
  *out = t.d;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaStreamSynchronize(st);        // usable from any stream afterwards
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
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(linb::k2d_rowb<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    cudaFuncSetAttribute(linb::k2d_colb<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    attrs = true;
  }
  const long long fs2 = (long long)N * N;
  double* P = scratch;
  double* Qb = scratch + fs2 * nsys;
  const dim3 rgrid((RG::NP + RG::SP - 1) / RG::SP, nsys), cgrid(N / CG::TC, nsys);
  linb::RowArgs ra{};
  ra.m = g.m; ra.cdt = sp.dt * g.c1; ra.info = info; ra.info_index = sys_index; ra.wtab = nt.wtab;
  linb::ColArgs ca{Qb, P, fs2, reinterpret_cast<const double2*>(dtab), nt.wtab};
  for (int s = 0; s < steps; ++s) {
    if (s == 0) { ra.in = in; ra.in_stride = in_stride; ra.in_index = sys_index; ra.mode = linb::MODE_FIRST; }
    else { ra.in = P; ra.in_stride = fs2; ra.in_index = nullptr; ra.mode = linb::MODE_MID; }
    ra.out = Qb; ra.out_stride = fs2; ra.out_index = nullptr;
    linb::k2d_rowb<N><<<rgrid, RG::THREADS, RG::SMEM, st>>>(ra);
    linb::k2d_colb<N><<<cgrid, CG::THREADS, CG::SMEM, st>>>(ca);
  }
  ra.in = P; ra.in_stride = fs2; ra.in_index = nullptr; ra.mode = linb::MODE_LAST;
  ra.out = out; ra.out_stride = out_stride; ra.out_index = sys_index;
  linb::k2d_rowb<N><<<rgrid, RG::THREADS, RG::SMEM, st>>>(ra);
  return cudaGetLastError();
}

template <int N>
cudaError_t propagate_n(Chp2d* c, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                        const double* in, long long in_stride, double* out, long long out_stride,
                        const int* idx, chp_sys_info* info, const NTables& nt, cudaStream_t st) {
  const long long fs = (long long)g.m * N;
  if (sp.scheme == CHP_LINEAR_B) {
    static const bool v1 = getenv("CHP_LINB_V1") != nullptr;   // A/B: previous passes
    cudaError_t e = grow(reinterpret_cast<void**>(&c->scratch), &c->scratch_bytes,
                         2 * (v1 ? fs : (long long)N * N) * nsys * sizeof(double), st);
    if (e != cudaSuccess) return e;
    const double* dtab = nullptr;
    const double s2 = (2.0 / N) * (2.0 / N);
    if ((e = get_dtab(c, N, sp, nt, v1 ? s2 : s2 / 256.0, v1 ? 0 : 1, &dtab, st)) != cudaSuccess)
      return e;
    if (!v1)
      return run_linear_b2<N>(g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt,
                              c->scratch, dtab, st);
    return run_linear_b<N>(g, sp, steps, nsys, in, in_stride, out, out_stride, idx, info, nt,
                           c->scratch, dtab, st);
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
  // default: the pair-DST cooperative kernel (chp_coarse2.cuh), 1.5 ms per config-5
  // slice over a 512-slice sweep; CHP_COARSE_V1 selects the previous kernel (A/B)
  static const bool coarse_v1 = getenv("CHP_COARSE_V1") != nullptr;
  if (sp.scheme == CHP_LINEAR_A && !coarse_v1) {
    using G2 = Coop2G<N>;
    static int blocks = 0;
    if (blocks == 0) {
      cudaFuncSetAttribute(k2d_coarse2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)G2::SMEM);
      int dev = 0, sms = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2d_coarse2<N>, G2::THREADS, G2::SMEM);
      // one block per SM: enough lane groups for every row pair, and half the
      // grid-barrier arrivals of two
      blocks = sms * (per > 0 ? 1 : 1);
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
      if (env && !tr) cudaMalloc(&tr, sizeof(unsigned long long) * 4096);
      ca.trace = env ? tr : nullptr;
      ca.trace_cap = 4096;
      if (env) g_coop_trace = tr;
    }
    cudaMemsetAsync(ca.bar, 0, sizeof(unsigned int), st);
    ca.lam = nt.lam; ca.wtab = nt.wtab;
    void* args[] = {&ca};
    return cudaLaunchCooperativeKernel((void*)k2d_coarse2<N>, dim3(blocks), dim3(G2::THREADS),
                                       args, G2::SMEM, st);
  }
  if (sp.scheme == CHP_LINEAR_A) {
    // whole sweep in one cooperative persistent kernel (no host round trips)
    static int grid_blocks = 0;
    const size_t smem = CoopGeo<N>::SMEM;
    if (grid_blocks == 0) {
      cudaFuncSetAttribute(k2d_coarse_coop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      int dev = 0, sms = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2d_coarse_coop<N>, 256, smem);
      grid_blocks = sms * (per > 0 ? per : 1);
      if (grid_blocks > 4 * sms) grid_blocks = 4 * sms;
    }
    Work2 W;
    cudaError_t e = get_work(c, fs, nic, &W, st, 16 * (size_t)grid_blocks + 8);
    if (e != cudaSuccess) return e;
    CoopArgs ca{};
    ca.m = g.m; ca.nic = nic; ca.nsl = nsl; ca.n0 = n0; ca.n1 = n1; ca.mode = mode;
    ca.c1 = g.c1; ca.dt = sp.dt; ca.b = sp.b; ca.tol = sp.cg_tol; ca.max_iter = sp.cg_max_iter;
    ca.U = U; ca.F = F; ca.G = G; ca.ics = ics; ca.sls = sls;
    ca.changed = changed; ca.inc = inc; ca.info = info;
    ca.X = W.X; ca.Rv = W.Rv; ca.Pv = W.Pv; ca.Yv = W.Yv; ca.Cv = W.Cv; ca.CT = W.T2; ca.Mi = W.T1; ca.Dk = W.YH;
    ca.part = W.coop;                    // 2 x 8 doubles per block (alternating)
    ca.bar = reinterpret_cast<unsigned int*>(W.res);
    {
      static unsigned long long* tr = nullptr;
      const char* env = getenv("CHP_COOP_TRACE");
      if (env && !tr) cudaMalloc(&tr, sizeof(unsigned long long) * 4096);
      ca.trace = env ? tr : nullptr;
      ca.trace_cap = 4096;
      if (env) g_coop_trace = tr;
    }
    cudaMemsetAsync(ca.bar, 0, sizeof(unsigned int), st);
    ca.lam = nt.lam; ca.wtab = (CoopGeo<N>::L == wdst::Geo<N>::L) ? nt.wtab : nt.wtab_coop;
    void* args[] = {&ca};
    return cudaLaunchCooperativeKernel((void*)k2d_coarse_coop<N>, dim3(grid_blocks), dim3(256),
                                       args, smem, st);
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

// debug: copy the cooperative coarse kernel's barrier timestamps (ns) to the host
extern "C" int chp_debug_trace(unsigned long long* host, int n) {
  if (!g_coop_trace || !host || n <= 0) return 0;
  if (n > 4096) n = 4096;
  cudaMemcpy(host, g_coop_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  return n;
}
