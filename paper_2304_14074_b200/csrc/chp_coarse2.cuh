// Device-resident 2D coarse sweep, v2 (included inside chp_2d.cu's anonymous
// namespace, after GridBar / coop_block_partials / coop_total).
//
// One cooperative persistent kernel runs the whole sequential recursion of
// parareal.py:245-251 (mode 1) or coarse_init (parareal.py:167-185, mode 0):
//   for n in [n0, n1):  g = G(U_n)   (LINEAR_A, schemes.py:235-246)
//                       U_{n+1} = (g + F_n) - G_n ;  G_n = g
// G solves (I - a L diag(c) + b L^2) x = rhs, c = v^2, a = dt, b = eps^2 dt,
// as the SPD system (K^-1 + bK + a diag(c)) x = K^-1 rhs in the orthonormal DST
// basis (x^ = S x, S = (2/N) T_i T_j) by PCG with the diagonal preconditioner
// M = d + a mean(c), d = 1/kappa + b kappa:
//   A x^ = d .* x^ + a S (c .* S x^),   b^ = S rhs / kappa.
// Transforms are chp_fdst.cuh's T' = 4T, so S = sigma T'_i T'_j, sigma = 1/(8N).
// CG vectors (X, R, P, Y) live in the pair-interleaved layout of chp_linb.cuh
// (row pairs (2s, 2s+1), N x N doubles, zero pads); c is stored column-pair
// major ([q/2][n] double2, pre-scaled by a sigma^2) so the column phase applies
// it coalesced in the inverse transform's pre-processing.
// CG in the Chronopoulos-Gear form (one reduction per iteration, mathematically
// the same iterates as standard PCG): with u = M^-1 r, w = A u,
//   gamma = (r, u), delta = (w, u), beta = gamma / gamma_old,
//   alpha = gamma / (delta - beta gamma / alpha_old),
//   p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s.
// Phases per iteration (grid barrier after each):
//   R1  rows: p, s, x, r updates fused; u = M^-1 r; Y = T'_j u
//   C   cols: Y = T'_i (c'' .* T'_i Y)
//   R3  rows: w = d .* u + T'_j Y; partials gamma, delta, (r, r)
// Every dot product is a fixed-order two-level reduction: bitwise reproducible.

#ifndef CHP_C2_UNROLL
#define CHP_C2_UNROLL 8
#endif
constexpr int kC2U = CHP_C2_UNROLL;
#ifndef CHP_C2_FB
#define CHP_C2_FB 8          // column tile fill / store: items per batch of loads (0: one by one)
#endif
#ifndef CHP_C2_CTS
#define CHP_C2_CTS 0         // 1: c'' vector staged in shared memory by cp.async (measured: no gain)
#endif

// CHP_C2_FT (debug builds only): clock64 stamps of block 0 / thread 0 inside the phases,
// slot [4096 + 8 gen + code] of the trace buffer (gen = barriers passed so far)
#ifdef CHP_C2_FT
#define C2_FT(a, gen, code)                                                           \
  do {                                                                                \
    if ((a).trace && blockIdx.x == 0 && threadIdx.x == 0 && (int)(gen) < (a).trace_cap) \
      (a).trace[4096 + 8 * (gen) + (code)] = (unsigned long long)clock64();           \
  } while (0)
#else
#define C2_FT(a, gen, code) do {} while (0)
#endif   // loads in flight per lane in the elementwise phase parts

struct Coop2Args {
  int m, nic, nsl, n0, n1, mode;
  double c1, dt, b, tol;
  int max_iter, pad_;
  double* U; const double* F; double* G; long long ics, sls;
  unsigned char* changed; double* inc; chp_sys_info* info;
  double *X, *R, *P, *Y, *Mi;   // PI layout, N*N each
  double *S, *W;                // Chronopoulos-Gear: s = A p, w = A u
  double* Dk;                   // PI: d = 1/kappa + b kappa (constant)
  double* SK;                   // PI: sigma / kappa (constant)
  double* CT;                   // [q/2][n] double2: a sigma^2 c(n, q), + slack
  double* gx;                   // g in the external layout (m x N)
  double* part;                 // [2][gridDim][8]
  unsigned int* bar;
  const double* lam; const double2* wtab;
  unsigned long long* trace;
  int trace_cap, res;             // res: r and w resident in shared memory (one row pair per group)
  // fused boundary hand-off (include/chp.h chp_hop): U[n1] of every IC is also stored to
  // the next rank's mailbox by the last slice's correction, then the flag is released
  double* hop_u; long long hop_stride;
  unsigned char* hop_changed; unsigned int* hop_flag; unsigned int hop_seq, pad3_;
};

template <int N> struct Coop2G {
  using F = fdst::FG<N>;
  static constexpr int L = F::L;
  static constexpr int THREADS = 128;
  static constexpr int GPB = THREADS / L;                        // lane groups per block
  static constexpr int GROUPS = (GPB < N / 2) ? GPB : N / 2;     // column pairs per column tile
  static constexpr int TC = 2 * GROUPS;
  static constexpr int RBASE(int c) { return c * F::RS + 2 * (c >> 1); }
  // after the transform regions: one staged c'' column-pair vector (n = 0..N) per group
  static constexpr int CBASE = RBASE(GPB - 1) + F::RS;
  static constexpr int CS = N + 2;
  static constexpr int XBASE = CBASE + (CHP_C2_CTS ? GPB * CS : 0);
  static constexpr size_t SMEM = sizeof(double2) * (size_t)XBASE;
  // resident CG vectors (Coop2Args::res): the residual r and w = A u of the row pair a lane
  // group owns for the whole solve stay in shared memory (N double2 each)
  static constexpr size_t SMEM_RES = SMEM + sizeof(double2) * (size_t)(GPB * 2 * N);
};

// One out-of-line copy of each transform variant for the whole kernel: the
// phases are latency bound, so a small instruction footprint (every phase
// runs the same code) and a per-call register budget matter more than inlining.
template <int N, int DS>
__device__ __noinline__ void c2_dst(double2* reg, const double2* __restrict__ twl, int l,
                                    double sa2, double ca2, const double2* __restrict__ dsc,
                                    const double2* __restrict__ dsm) {
  double2* ob = fdst::out_base<N>(reg, l);
  fdst::pair_dst<N, DS>(reg, reg, twl, l, sa2, ca2,
                        [&](int j, double a0, double a1, double b0, double b1) {
                          ob[2 * j] = make_double2(a0, b0);
                          ob[2 * j + 1] = make_double2(a1, b1);
                        }, dsc, dsm);
}

// ---- row phase: for every row pair s (grid-strided over lane groups) -------
//   op 0: out = T' in
//   op 3: CG-CG update (p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s,
//         u = Mi .* r), out = T' u           (first: p = u, s = w)
//   op 4: W = Dk .* u + T' in (u = Mi .* R); partials (r.u, w.u, r.r) into part[0..2]
//   op 5: R = SK .* in, X = 0, u = Mi .* R, out = T' u  (CG start, x0 = 0)
template <int N>
CHP_DEV void c2_rows(const Coop2Args& a, double2* sm, int op, const double* in, double* out,
                     bool first, double alpha, double beta, double2 ac, double (&part)[3],
                     unsigned int gen = 0) {
  using F = fdst::FG<N>;
  using G2 = Coop2G<N>;
  constexpr int L = F::L, R = F::R, Q = F::Q;
  const int g = threadIdx.x / L, l = threadIdx.x % L;
  const int gg = g * gridDim.x + blockIdx.x, ngr = gridDim.x * G2::GPB;
  double2* reg = sm + G2::RBASE(g);
  double2* resR = sm + G2::XBASE + g * 2 * N;   // a.res: the group's r and w rows
  double2* resW = resR + N;
  const double2* twl = a.wtab + N + l;
  for (int s0 = 0; s0 < N / 2; s0 += ngr) {
    const int s = s0 + gg;
    const bool have = s < N / 2;              // whole warps iterate together
    const long long base = (long long)(have ? s : 0) * N;   // double2 index of the pair row
    if (op == 3 || op == 5) {
      double2* Rr = a.res ? resR : reinterpret_cast<double2*>(a.R) + base;
      double2* Xr = reinterpret_cast<double2*>(a.X) + base;
      const double2* Mr = reinterpret_cast<const double2*>(a.Mi) + base;
      double2* Pr = reinterpret_cast<double2*>(a.P) + base;
      double2* Sr = reinterpret_cast<double2*>(a.S) + base;
      const double2* Wr = a.res ? resW : reinterpret_cast<const double2*>(a.W) + base;
      const double2* Ir = reinterpret_cast<const double2*>(in) + base;
      const double2* Kr = reinterpret_cast<const double2*>(a.SK) + base;
      // the loads of UN elements are issued together, ahead of the stores (which the
      // compiler must otherwise keep in order with the next element's loads: the vectors
      // may alias for all it knows, and every element then costs one L2 round trip)
      constexpr int UN = kC2U < R ? kC2U : R;
#pragma unroll 1
      for (int i0 = 0; i0 < R; i0 += UN) {
        double2 mi[UN], rv[UN], xv[UN], wv[UN], pv[UN], sv[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int n = l + L * (i0 + u);
          mi[u] = Mr[n];
          if (op == 5) {
            rv[u] = Ir[n];           // y
            xv[u] = Kr[n];           // sk
          } else {
            rv[u] = Rr[n];
            xv[u] = Xr[n];
            wv[u] = Wr[n];
            if (!first) { pv[u] = Pr[n]; sv[u] = Sr[n]; }
          }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int i = i0 + u, n = l + L * i;
          double2 r, x;
          if (op == 5) {
            r = make_double2(rv[u].x * xv[u].x, rv[u].y * xv[u].y);
            x = make_double2(0.0, 0.0);
          } else {
            r = rv[u];
            x = xv[u];
            const double2 w = wv[u];
            const double2 uu = make_double2(r.x * mi[u].x, r.y * mi[u].y);
            double2 p, sn;
            if (first) { p = uu; sn = w; }
            else {
              p = make_double2(fma(beta, pv[u].x, uu.x), fma(beta, pv[u].y, uu.y));
              sn = make_double2(fma(beta, sv[u].x, w.x), fma(beta, sv[u].y, w.y));
            }
            x = make_double2(fma(alpha, p.x, x.x), fma(alpha, p.y, x.y));
            r = make_double2(fma(-alpha, sn.x, r.x), fma(-alpha, sn.y, r.y));
            if (have) { Pr[n] = p; Sr[n] = sn; }
          }
          if (have) { Rr[n] = r; Xr[n] = x; }
          reg[n + i / Q] = make_double2(r.x * mi[u].x, r.y * mi[u].y);
        }
      }
    } else {
      const double2* src = reinterpret_cast<const double2*>(in) + base;
#pragma unroll 4
      for (int i = 0; i < R; ++i) linb::cp16(&reg[l + L * i + i / Q], &src[l + L * i]);
      linb::cp_wait();
    }
    __syncwarp();
    C2_FT(a, gen, 1);
    c2_dst<N, 0>(reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, nullptr, nullptr);
    __syncwarp();
    C2_FT(a, gen, 2);
    if (op == 4) {
      const double2* Rr = a.res ? resR : reinterpret_cast<const double2*>(a.R) + base;
      const double2* Mr = reinterpret_cast<const double2*>(a.Mi) + base;
      const double2* Dr = reinterpret_cast<const double2*>(a.Dk) + base;
      double2* Wr = a.res ? resW : reinterpret_cast<double2*>(a.W) + base;
      constexpr int UN = (2 * kC2U) < R ? (2 * kC2U) : R;
#pragma unroll 1
      for (int i0 = 0; i0 < R; i0 += UN) {
        double2 rv[UN], mi[UN], dv[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int n = l + L * (i0 + u);
          rv[u] = Rr[n];
          mi[u] = Mr[n];
          dv[u] = Dr[n];
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int i = i0 + u, n = l + L * i;
          const double2 y = reg[n + i / Q], r = rv[u], d = dv[u];
          const double2 uu = make_double2(r.x * mi[u].x, r.y * mi[u].y);
          const double2 w = make_double2(fma(d.x, uu.x, y.x), fma(d.y, uu.y, y.y));
          if (have) {
            Wr[n] = w;
            part[0] = fma(r.x, uu.x, part[0]);
            part[0] = fma(r.y, uu.y, part[0]);
            part[1] = fma(w.x, uu.x, part[1]);
            part[1] = fma(w.y, uu.y, part[1]);
            part[2] = fma(r.x, r.x, part[2]);
            part[2] = fma(r.y, r.y, part[2]);
          }
        }
      }
    } else if (have) {
      double2* dst = reinterpret_cast<double2*>(out) + base;
#pragma unroll 8
      for (int i = 0; i < R; ++i) dst[l + L * i] = reg[l + L * i + i / Q];
    }
    __syncwarp();
    C2_FT(a, gen, 4);
  }
}

// ---- column phase: tiles of TC columns (one lane group per column pair) ----
//   op 0: out = T' in                         (PI -> PI)
//   op 1: out = T' (CT .* T' in)              (PI -> PI)
//   op 2: gx = sigma T' in                    (PI -> external layout, rows 1..m)
template <int N>
CHP_DEV void c2_cols(const Coop2Args& a, double2* sm, int op, const double* in, double* out,
                     double sigma, double2 ac, unsigned int gen = 0) {
  using F = fdst::FG<N>;
  using G2 = Coop2G<N>;
  constexpr int L = F::L, GROUPS = G2::GROUPS, TC = G2::TC;
  const int g = threadIdx.x / L, l = threadIdx.x % L;
  const double2* twl = a.wtab + N + l;
  double2* reg = sm + G2::RBASE(g);
  for (int tile = blockIdx.x; tile < N / TC; tile += gridDim.x) {
    const int j0 = tile * TC;
    // fill: (pair s, column pair c): 32 contiguous bytes of the PI field
    // op 1: the group's c'' column-pair vector is staged by cp.async under the fill and
    // the first transform (its 64 L2 loads per lane otherwise sit inside the second
    // transform's pre-processing)
    double2* cs = sm + G2::CBASE + g * G2::CS;
    if (CHP_C2_CTS && op == 1) {
      const double2* cr = reinterpret_cast<const double2*>(a.CT) +
                          (long long)(j0 / 2 + (g < GROUPS ? g : 0)) * N;
      for (int n = l; n <= N; n += L) linb::cp16(&cs[n], &cr[n]);
    }
#if CHP_C2_FB > 0
    // (kFB items' loads together: through generic pointers the compiler keeps every
    // shared-memory store in order with the next item's global loads)
    constexpr int kItems = (N / 2) * GROUPS;
    constexpr int kFB = (kItems / G2::THREADS) >= CHP_C2_FB ? CHP_C2_FB
                        : ((kItems / G2::THREADS) > 0 ? (kItems / G2::THREADS) : 1);
    constexpr bool kEven = kItems % (kFB * G2::THREADS) == 0;
    if constexpr (kEven) {
      for (int i0 = threadIdx.x; i0 < kItems; i0 += kFB * G2::THREADS) {
        double2 u[kFB], w[kFB];
#pragma unroll
        for (int e = 0; e < kFB; ++e) {
          const int idx = i0 + e * G2::THREADS;
          const int s = idx / GROUPS, c = idx % GROUPS;
          const double2* src = reinterpret_cast<const double2*>(in + ((long long)s * N + j0 + 2 * c) * 2);
          u[e] = src[0];
          w[e] = src[1];
        }
#pragma unroll
        for (int e = 0; e < kFB; ++e) {
          const int idx = i0 + e * G2::THREADS;
          const int s = idx / GROUPS, c = idx % GROUPS;
          double2* rg = sm + G2::RBASE(c);
          rg[fdst::p2<N>(2 * s)] = make_double2(u[e].x, w[e].x);
          rg[fdst::p2<N>(2 * s + 1)] = make_double2(u[e].y, w[e].y);
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < kItems; idx += G2::THREADS) {
        const int s = idx / GROUPS, c = idx % GROUPS;
        const double2* src = reinterpret_cast<const double2*>(in + ((long long)s * N + j0 + 2 * c) * 2);
        const double2 u = src[0], w = src[1];
        double2* rg = sm + G2::RBASE(c);
        rg[fdst::p2<N>(2 * s)] = make_double2(u.x, w.x);
        rg[fdst::p2<N>(2 * s + 1)] = make_double2(u.y, w.y);
      }
    }
#else
#pragma unroll 16
    for (int idx = threadIdx.x; idx < (N / 2) * GROUPS; idx += G2::THREADS) {
      const int s = idx / GROUPS, c = idx % GROUPS;
      const double2* src = reinterpret_cast<const double2*>(in + ((long long)s * N + j0 + 2 * c) * 2);
      const double2 u = src[0], w = src[1];
      double2* rg = sm + G2::RBASE(c);
      rg[fdst::p2<N>(2 * s)] = make_double2(u.x, w.x);
      rg[fdst::p2<N>(2 * s + 1)] = make_double2(u.y, w.y);
    }
#endif
    __syncthreads();
    C2_FT(a, gen, 1);
    c2_dst<N, 0>(reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, nullptr, nullptr);
    C2_FT(a, gen, 2);
    if (op == 1) {
#if CHP_C2_CTS
      linb::cp_wait();
      __syncwarp();
      c2_dst<N, 2>(reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, cs + l, cs + N - l);
#else
      __syncwarp();
      const double2* cr = reinterpret_cast<const double2*>(a.CT) +
                          (long long)(j0 / 2 + (g < GROUPS ? g : 0)) * N;
      c2_dst<N, 1>(reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, cr + l, cr + N - l);
#endif
    }
    __syncthreads();
    C2_FT(a, gen, 3);
    if (op == 2) {
      // external layout: storage row i = math row i + 1; 16 B per (row, column pair)
      for (int idx = threadIdx.x; idx < a.m * GROUPS; idx += G2::THREADS) {
        const int i = idx / GROUPS, c = idx % GROUPS;
        const double2 v = sm[G2::RBASE(c) + fdst::p2<N>(i + 1)];
        *reinterpret_cast<double2*>(out + (long long)i * N + j0 + 2 * c) =
            make_double2(v.x * sigma, v.y * sigma);
      }
    } else {
#if CHP_C2_FB > 0
      if constexpr (kEven) {
        for (int i0 = threadIdx.x; i0 < kItems; i0 += kFB * G2::THREADS) {
          double2 u[kFB], w[kFB];
#pragma unroll
          for (int e = 0; e < kFB; ++e) {
            const int idx = i0 + e * G2::THREADS;
            const int s = idx / GROUPS, c = idx % GROUPS;
            const double2* rg = sm + G2::RBASE(c);
            u[e] = rg[fdst::p2<N>(2 * s)];
            w[e] = rg[fdst::p2<N>(2 * s + 1)];
          }
#pragma unroll
          for (int e = 0; e < kFB; ++e) {
            const int idx = i0 + e * G2::THREADS;
            const int s = idx / GROUPS, c = idx % GROUPS;
            double2* dst = reinterpret_cast<double2*>(out + ((long long)s * N + j0 + 2 * c) * 2);
            dst[0] = make_double2(u[e].x, w[e].x);
            dst[1] = make_double2(u[e].y, w[e].y);
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < kItems; idx += G2::THREADS) {
          const int s = idx / GROUPS, c = idx % GROUPS;
          const double2* rg = sm + G2::RBASE(c);
          const double2 u = rg[fdst::p2<N>(2 * s)], w = rg[fdst::p2<N>(2 * s + 1)];
          double2* dst = reinterpret_cast<double2*>(out + ((long long)s * N + j0 + 2 * c) * 2);
          dst[0] = make_double2(u.x, w.x);
          dst[1] = make_double2(u.y, w.y);
        }
      }
#else
      for (int idx = threadIdx.x; idx < (N / 2) * GROUPS; idx += G2::THREADS) {
        const int s = idx / GROUPS, c = idx % GROUPS;
        const double2* rg = sm + G2::RBASE(c);
        const double2 u = rg[fdst::p2<N>(2 * s)], w = rg[fdst::p2<N>(2 * s + 1)];
        double2* dst = reinterpret_cast<double2*>(out + ((long long)s * N + j0 + 2 * c) * 2);
        dst[0] = make_double2(u.x, w.x);
        dst[1] = make_double2(u.y, w.y);
      }
#endif
    }
    __syncthreads();
    C2_FT(a, gen, 4);
  }
}

template <int N>
__global__ void __launch_bounds__(128, 2) k2d_coarse2(Coop2Args a) {
  using G2 = Coop2G<N>;
  GridBar grid{a.bar, 0u, a.trace, a.trace_cap};
  extern __shared__ __align__(16) double2 smc2[];
  __shared__ double red[64];
  const int m = a.m;
  const long long NN = (long long)N * N;           // PI field doubles
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const double sigma = 1.0 / (8.0 * N);
  const double tol2 = a.tol * a.tol;
  const double acs = a.dt * sigma * sigma;         // CT scale: a sigma^2
  const double2 acl = __ldg(&a.wtab[threadIdx.x % fdst::FG<N>::L]);   // per-lane (cos, sin)(pi l / N)
  // constant tables (PI): Dk = 1/kappa + b kappa, SK = sigma / kappa (zero on pads)
  for (long long t = gtid; t < NN; t += gstride) {
    const int s = (int)(t / (2 * N)), q = (int)((t / 2) % N), h = (int)(t & 1);
    const int p = 2 * s + h;
    double d = 0.0, sk = 0.0;
    if (p > 0 && q > 0) {
      const double kap = -(a.lam[p] + a.lam[q]);
      d = 1.0 / kap + a.b * kap;
      sk = sigma / kap;
    }
    a.Dk[t] = d;
    a.SK[t] = sk;
  }
  int pb = 0;
  for (int ic = 0; ic < a.nic; ++ic) {
    unsigned char* ch = a.changed ? a.changed + (long long)ic * (a.nsl + 1) : nullptr;
    double* Ui = a.U + ic * a.ics;
    double* Gi = a.G + ic * a.ics;
    const double* Fi = a.F ? a.F + ic * a.ics : nullptr;
    if (a.mode == 1 && (ch[0] & 2)) continue;      // IC frozen
    double dmax = 0.0;
    for (int n = a.n0; n < a.n1; ++n) {
      const double* un = Ui + (long long)n * a.sls;
      double* un1 = Ui + (long long)(n + 1) * a.sls;
      double* gn = Gi + (long long)n * a.sls;
      if (a.mode == 1 && blockIdx.x == 0 && threadIdx.x == 0) ch[n + 1] = 0;
      gbar(grid);                                   // ch[n] / U_n written by the previous slice
      const bool solve = (a.mode == 0) || (*(volatile unsigned char*)&ch[n] & 1);
      if (solve) {
        // ---- prep: rhs = v - dt L v (PI, into Y), c'' = a sigma^2 v^2 (CT), sum v^2 ----
        double sc[1] = {0.0};
        // (both loops: the loads of kPU elements are issued together; one element per
        // L2 round trip otherwise)
        constexpr int kPU = 4;
        for (long long t0 = gtid; t0 < NN / 2; t0 += kPU * gstride) {
          double v[kPU][2], vu[kPU][2], vd[kPU][2], vl[kPU][2], vr[kPU][2];
          bool in[kPU][2];
#pragma unroll
          for (int e = 0; e < kPU; ++e) {
            const long long t = t0 + e * gstride;
            const int s = (int)(t / N), j = (int)(t % N);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int i = 2 * s + h - 1;          // storage row of math row 2s+h
              in[e][h] = t < NN / 2 && j > 0 && i >= 0 && i < m;
              v[e][h] = vu[e][h] = vd[e][h] = vl[e][h] = vr[e][h] = 0.0;
              if (in[e][h]) {
                const long long o = (long long)i * N + j;
                v[e][h] = un[o];
                if (i > 0) vu[e][h] = un[o - N];
                if (i + 1 < m) vd[e][h] = un[o + N];
                if (j > 1) vl[e][h] = un[o - 1];
                if (j < m) vr[e][h] = un[o + 1];
              }
            }
          }
#pragma unroll
          for (int e = 0; e < kPU; ++e) {
            const long long t = t0 + e * gstride;
            if (t >= NN / 2) break;
            double r2[2] = {0.0, 0.0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (!in[e][h]) continue;
              const double lv = ((((vu[e][h] * a.c1 + vl[e][h] * a.c1) + v[e][h] * (-4.0 * a.c1)) +
                                  vr[e][h] * a.c1) + vd[e][h] * a.c1);
              r2[h] = v[e][h] - a.dt * lv;
              sc[0] = fma(v[e][h], v[e][h], sc[0]);
            }
            reinterpret_cast<double2*>(a.Y)[t] = make_double2(r2[0], r2[1]);
          }
        }
        for (long long t0 = gtid; t0 < NN / 2; t0 += kPU * gstride) {
          double2 vv[kPU];
#pragma unroll
          for (int e = 0; e < kPU; ++e) {
            const long long t = t0 + e * gstride;
            const int qp = (int)(t % (N / 2)), r = (int)(t / (N / 2));   // math row r, columns 2qp, 2qp+1
            vv[e] = make_double2(0.0, 0.0);
            if (t < NN / 2 && r > 0)
              vv[e] = *reinterpret_cast<const double2*>(un + (long long)(r - 1) * N + 2 * qp);
          }
#pragma unroll
          for (int e = 0; e < kPU; ++e) {
            const long long t = t0 + e * gstride;
            if (t >= NN / 2) break;
            const int qp = (int)(t % (N / 2)), r = (int)(t / (N / 2));
            double2 cv = make_double2(0.0, 0.0);
            if (r > 0) cv = make_double2(qp > 0 ? acs * (vv[e].x * vv[e].x) : 0.0, acs * (vv[e].y * vv[e].y));
            reinterpret_cast<double2*>(a.CT)[(long long)qp * N + r] = cv;
          }
        }
        double* pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
        coop_block_partials<1>(sc, red, pbuf);
        gbar(grid);
        double tc[1];
        coop_total<1>(pbuf, red, tc);
        const double acbar = a.dt * (tc[0] / ((double)m * m));
        for (long long t0 = gtid; t0 < NN / 2; t0 += 8 * gstride) {
          double2 d[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const long long t = t0 + e * gstride;
            d[e] = (t < NN / 2) ? reinterpret_cast<const double2*>(a.Dk)[t] : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const long long t = t0 + e * gstride;
            if (t < NN / 2)
              reinterpret_cast<double2*>(a.Mi)[t] =
                  make_double2((d[e].x != 0.0) ? 1.0 / (d[e].x + acbar) : 0.0,
                               (d[e].y != 0.0) ? 1.0 / (d[e].y + acbar) : 0.0);
          }
        }
        // ---- b^ = S rhs / kappa: Y = T'_i T'_j rhs (R = SK .* Y in the start phase) ----
        double nop[3] = {0.0, 0.0, 0.0};
        c2_rows<N>(a, smc2, 0, a.Y, a.Y, false, 0.0, 0.0, acl, nop, grid.gen);
        gbar(grid);
        c2_cols<N>(a, smc2, 0, a.Y, a.Y, 0.0, acl, grid.gen);
        gbar(grid);
        // ---- start (x0 = 0): r = b^, u = M^-1 r, w = A u; gamma, delta, rr0 ----
        c2_rows<N>(a, smc2, 5, a.Y, a.Y, true, 0.0, 0.0, acl, nop);
        gbar(grid);
        int it = 0;
        bool fail = false, done = false, started = false;
        double alpha = 0.0, beta = 0.0, gamma = 0.0, rr0 = 0.0;
        for (;;) {
          c2_cols<N>(a, smc2, 1, a.Y, a.Y, 0.0, acl, grid.gen);
          gbar(grid);
          double gd[3] = {0.0, 0.0, 0.0};
          c2_rows<N>(a, smc2, 4, a.Y, nullptr, false, 0.0, 0.0, acl, gd, grid.gen);
          double* pbuf = a.part + 8 * gridDim.x * (pb ^= 1);
          coop_block_partials<3>(gd, red, pbuf);
          gbar(grid);
          double t3[3];
          coop_total<3>(pbuf, red, t3);
          C2_FT(a, grid.gen, 5);
          const double gam = t3[0], del = t3[1], rr = t3[2];
          if (!started) {                                // start: alpha0 = gamma0 / delta0
            started = true;
            rr0 = rr;
            done = !(rr0 > 0.0);
            beta = 0.0;
            alpha = gam / del;
          } else {
            ++it;                                        // x, r of iteration `it` are final
            if (!(rr > tol2 * rr0)) done = true;         // also stops on NaN
            else if (it >= a.max_iter) { done = true; fail = true; }
            if (!isfinite(rr)) { done = true; fail = true; }
            beta = gam / gamma;
            alpha = gam / (del - beta * gam / alpha);
          }
          gamma = gam;
          if (done) break;
          c2_rows<N>(a, smc2, 3, nullptr, a.Y, it == 0, alpha, beta, acl, nop, grid.gen);
          gbar(grid);
        }
        if (gtid == 0) {
          a.info[ic].cg_total += it;
          a.info[ic].cg_max = max(a.info[ic].cg_max, it);
          if (fail) atomicCAS(&a.info[ic].status, CHP_SYS_OK, CHP_SYS_CG);
        }
        // ---- g = S x^ = sigma T'_i T'_j X -> gx (external layout) -----------------
        c2_rows<N>(a, smc2, 0, a.X, a.Y, false, 0.0, 0.0, acl, nop);
        gbar(grid);
        c2_cols<N>(a, smc2, 2, a.Y, a.gx, sigma, acl);
        gbar(grid);
      }
      // ---- correction / init (external layout) ------------------------------------
      const double* gsrc = solve ? a.gx : gn;
      const long long tot = (long long)m * N;
      bool any = false, bad = false;
      double* hop = (a.hop_u && n == a.n1 - 1) ? a.hop_u + ic * a.hop_stride : nullptr;
      // two points per lane and kCU lane iterations per batch of loads (t even: j even,
      // j + 1 <= m; the fields are 16-byte aligned)
      constexpr int kCU = 4;
      for (long long t0 = 2 * gtid; t0 < tot; t0 += 2 * kCU * gstride) {
        double2 g2[kCU], f2[kCU], o2[kCU], u2[kCU];
#pragma unroll
        for (int e = 0; e < kCU; ++e) {
          const long long t = t0 + 2 * e * gstride;
          if (t < tot) {
            g2[e] = *reinterpret_cast<const double2*>(gsrc + t);
            if (a.mode != 0) {
              f2[e] = *reinterpret_cast<const double2*>(Fi + (long long)n * a.sls + t);
              o2[e] = *reinterpret_cast<const double2*>(gn + t);
              u2[e] = *reinterpret_cast<const double2*>(un1 + t);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < kCU; ++e) {
          const long long t = t0 + 2 * e * gstride;
          if (t >= tot) break;
          const int j = (int)(t % N);
          const double2 gv = make_double2((j > 0) ? g2[e].x : 0.0, g2[e].y);
          if (a.mode == 0) {
            *reinterpret_cast<double2*>(un1 + t) = gv;
            *reinterpret_cast<double2*>(gn + t) = gv;
            if (hop) *reinterpret_cast<double2*>(hop + t) = gv;
            bad |= !isfinite(gv.x) || !isfinite(gv.y);
            continue;
          }
          const double2 nv = make_double2((gv.x + f2[e].x) - o2[e].x, (gv.y + f2[e].y) - o2[e].y);
          const double2 ov = u2[e];
          any |= (__double_as_longlong(nv.x) != __double_as_longlong(ov.x)) ||
                 (__double_as_longlong(nv.y) != __double_as_longlong(ov.y));
          dmax = fmax(dmax, fmax(fabs(nv.x - ov.x), fabs(nv.y - ov.y)));
          bad |= !isfinite(nv.x) || !isfinite(nv.y) || !isfinite(gv.x) || !isfinite(gv.y);
          *reinterpret_cast<double2*>(un1 + t) = nv;
          *reinterpret_cast<double2*>(gn + t) = gv;
          if (hop) *reinterpret_cast<double2*>(hop + t) = nv;
        }
      }
      if (hop) __threadfence_system();
      if (a.mode == 1) {
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
  // every block's mailbox stores are fenced and ordered before the last barrier: one
  // thread forwards the changed bits and releases the flag (frozen ICs were skipped: the
  // receiver keeps its own boundary for those)
  if (a.hop_flag && gtid == 0) {
    if (a.hop_changed && a.changed)
      for (int ic = 0; ic < a.nic; ++ic)
        a.hop_changed[ic] = a.changed[(long long)ic * (a.nsl + 1) + a.n1] & 1;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.hop_flag), "r"(a.hop_seq) : "memory");
  }
}
