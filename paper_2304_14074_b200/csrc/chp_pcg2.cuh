// Batched DST-preconditioned PCG, v2 (included inside chp_2d.cu's anonymous
// namespace after CgSys / k2d_cg_reduce).  Solves, for every active system s,
//   (I - a L diag(c_s) + b L^2) x_s = rhs_s
// exactly as the cooperative coarse kernel (chp_coarse2.cuh) does for one
// field: CG on (K^-1 + bK + a diag(c)) x^ = K^-1 rhs in the orthonormal DST
// basis, preconditioner d + a mean(c), vectors in the pair-interleaved layout,
// transforms T' = 4T of chp_fdst.cuh.  Used by the fine Newton update solve
// (schemes.py:303-304, a = 3 dt, c = Y^2) and by single-step LINEAR_A
// (schemes.py:245, a = dt, c = v^2).  One launch per phase over all systems
// (grid.y = system); converged systems skip their blocks; per-system CG
// scalars stay on the device (CgSys) and every dot product is a fixed-order
// two-level reduction.
//
// Phases per CG iteration: E3 (P = M^-1 R + beta P, streaming), T rows (Y = T'_j P),
// C cols (Y = T'_i (c'' .* T'_i Y)), T rows (Y = T'_j Y), E1 (Y = d .* P + Y, partial
// P.Y, streaming), reduce (alpha), E2 (X += alpha P, R -= alpha Y, partials), reduce (beta).
// The elementwise work runs in streaming kernels (5-6 TB/s) instead of inside the row
// transforms: fused into the transform kernels (round 1) the same loads sat on the critical
// path of a one-transform-per-group block at 8 warps/SM -- 556 + 362 us per iteration for the
// two fused row phases against 2 x (112 + 140) us unfused, although the unfused form moves
// P and Y once more (profiles/r02_c4_launches_v0.txt, all 128 config-4 systems active).

struct Pcg2 {
  int m;
  long long fs;                  // external field stride (m * N)
  const double* rhs;             // external layout, compact per system
  const double* cv;              // c, external layout
  double* out;                   // solution, external layout
  double *X, *R, *P, *Y;         // PI, stride NN per system
  double* CT;                    // [q/2][n] double2 per system, stride NN + 2
  const double* Dk;              // PI: 1/kappa + b kappa (shared)
  const double* SK;              // PI: sigma / kappa (shared)
  double a, sigma;
  CgSys* cg;
  double* partial;
  const double2* wtab;
};

template <int N> struct Pcg2G {
  using F = fdst::FG<N>;
  static constexpr int L = F::L;
  static constexpr int THREADS = 128;
  static constexpr int GPB = THREADS / L;
  static constexpr int RBLK = (N / 2 + GPB - 1) / GPB;        // row blocks per system
  static constexpr int GROUPS = (GPB < N / 2) ? GPB : N / 2;
  static constexpr int TC = 2 * GROUPS;
  static constexpr int RBASE(int c) { return c * F::RS + 2 * (c >> 1); }
  static constexpr size_t SMEM = sizeof(double2) * (size_t)(RBASE(GPB - 1) + F::RS);
};

CHP_DEV bool pcg2_skip(const CgSys& q, bool loop) { return !q.active || (loop && q.done); }

// preconditioner inverse 1 / (d + a mean(c)) on the fly from the shared d table
// (a deterministic reciprocal: float seed + two Newton steps; M need not be exact)
CHP_DEV double2 pcg2_mi(double2 d, double acb) {
  return make_double2(d.x != 0.0 ? wdst::rcp(d.x + acb) : 0.0, d.y != 0.0 ? wdst::rcp(d.y + acb) : 0.0);
}

// Dk, SK tables (PI, shared by all systems)
__global__ void k_pcg2_tables(int N, const double* lam, double b, double sigma, double* Dk,
                              double* SK) {
  const long long NN = (long long)N * N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / (2 * N)), q = (int)((t / 2) % N), h = (int)(t & 1);
    const int p = 2 * s + h;
    double d = 0.0, sk = 0.0;
    if (p > 0 && q > 0) {
      const double kap = -(lam[p] + lam[q]);
      d = 1.0 / kap + b * kap;
      sk = sigma / kap;
    }
    Dk[t] = d;
    SK[t] = sk;
  }
}

// rhs (external) -> Y (PI); c (external) -> CT (a sigma^2 c)
template <int N>
__global__ void k_pcg2_prep(Pcg2 a) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], false)) return;
  const long long NN = (long long)N * N;
  const int m = a.m;
  const double* rh = a.rhs + (long long)s * a.fs;
  const double* cv = a.cv + (long long)s * a.fs;
  double2* Y = reinterpret_cast<double2*>(a.Y + (long long)s * NN);
  double2* CT = reinterpret_cast<double2*>(a.CT + (long long)s * (NN + 2));
  const double acs = a.a * a.sigma * a.sigma;
  const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long t = i0; t < NN / 2; t += st) {
    const int sp = (int)(t / N), j = (int)(t % N);
    const int ra = 2 * sp - 1, rb = 2 * sp;        // storage rows of math rows 2sp, 2sp+1
    double ya = 0.0, yb = 0.0;
    if (j > 0) {
      if (ra >= 0) ya = rh[(long long)ra * N + j];
      if (rb < m) yb = rh[(long long)rb * N + j];
    }
    Y[t] = make_double2(ya, yb);
  }
  for (long long t = i0; t < NN / 2; t += st) {
    const int qp = (int)(t % (N / 2)), r = (int)(t / (N / 2));
    double2 c = make_double2(0.0, 0.0);
    if (r > 0) {
      const double2 v = *reinterpret_cast<const double2*>(cv + (long long)(r - 1) * N + 2 * qp);
      c = make_double2(qp > 0 ? acs * v.x : 0.0, acs * v.y);
    }
    CT[(long long)qp * N + r] = c;
  }
}

// rows (PI -> PI): OP 0: out = T'_j in
//   OP 1 (E3 fused): P = M^-1 R (+ beta P) formed while the row pair is loaded, out = T'_j P
//   OP 2 (E1 fused): out = Dk .* P + T'_j in, block partial of P . out into partial[sys * RBLK + block]
// The fused forms save one pass over P (OP 1) and one write + read of Y (OP 2) per CG iteration.
// Their elementwise loads are issued kRU elements at a time ahead of the stores: element by
// element every store may alias the next element's loads and each element then costs one
// memory round trip (the fused kernels of round 1 ran 556 + 362 us per iteration that way).
#ifndef CHP_PCG2_FUSE
#define CHP_PCG2_FUSE 1
#endif
template <int N, int OP>
__global__ void __launch_bounds__(128, 2) k_pcg2_rows(Pcg2 a, const double* in, double* out, int loop) {
  using F = fdst::FG<N>;
  using G2 = Pcg2G<N>;
  constexpr int L = F::L, R = F::R, Q = F::Q;
  constexpr int kRU = R < 8 ? R : 8;
  extern __shared__ __align__(16) double2 smp[];
  __shared__ double wpart[G2::GPB];
  const int sys = blockIdx.y;
  const CgSys& q = a.cg[sys];
  if (pcg2_skip(q, loop)) return;
  const long long NN = (long long)N * N;
  const int g = threadIdx.x / L, l = threadIdx.x % L;
  const int s = blockIdx.x * G2::GPB + g;
  const bool have = s < N / 2;
  const long long row = (long long)(have ? s : 0) * N;
  const long long base = (long long)sys * (NN / 2) + row;   // double2
  double2* reg = smp + G2::RBASE(g);
  const double2 ac = __ldg(&a.wtab[l]);
  const double2* twl = a.wtab + N + l;
  if (OP == 1) {
    const double2* Rr = reinterpret_cast<const double2*>(a.R) + base;
    const double2* Dr = reinterpret_cast<const double2*>(a.Dk) + row;
    double2* Pr = reinterpret_cast<double2*>(a.P) + base;
    const bool first = q.iters == 0;
    const double beta = q.beta, acb = q.acbar;
#pragma unroll 1
    for (int i0 = 0; i0 < R; i0 += kRU) {
      double2 rv[kRU], dv[kRU], pv[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int n = l + L * (i0 + u);
        rv[u] = Rr[n];
        dv[u] = Dr[n];
        if (!first) pv[u] = Pr[n];
      }
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int i = i0 + u, n = l + L * i;
        const double2 mi = pcg2_mi(dv[u], acb);
        double2 pn = make_double2(rv[u].x * mi.x, rv[u].y * mi.y);
        if (!first) pn = make_double2(fma(beta, pv[u].x, pn.x), fma(beta, pv[u].y, pn.y));
        if (have) Pr[n] = pn;
        reg[n + i / Q] = pn;
      }
    }
  } else {
    const double2* src = reinterpret_cast<const double2*>(in) + base;
#pragma unroll 8
    for (int i = 0; i < R; ++i) linb::cp16(&reg[l + L * i + i / Q], &src[l + L * i]);
    linb::cp_wait();
  }
  __syncwarp();
  double2* ob = fdst::out_base<N>(reg, l);
  fdst::pair_dst<N>(reg, reg, twl, l, 2.0 * ac.y, 2.0 * ac.x,
                    [&](int j, double a0, double a1, double b0, double b1) {
                      ob[2 * j] = make_double2(a0, b0);
                      ob[2 * j + 1] = make_double2(a1, b1);
                    });
  __syncwarp();
  double2* dst = reinterpret_cast<double2*>(out) + base;
  if (OP == 2) {
    const double2* Pr = reinterpret_cast<const double2*>(a.P) + base;
    const double2* Dr = reinterpret_cast<const double2*>(a.Dk) + row;
    double part = 0.0;
#pragma unroll 1
    for (int i0 = 0; i0 < R; i0 += kRU) {
      double2 pv[kRU], dv[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int n = l + L * (i0 + u);
        pv[u] = Pr[n];
        dv[u] = Dr[n];
      }
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int i = i0 + u, n = l + L * i;
        const double2 y = reg[n + i / Q];
        const double2 w = make_double2(fma(dv[u].x, pv[u].x, y.x), fma(dv[u].y, pv[u].y, y.y));
        if (have) {
          dst[n] = w;
          part = fma(pv[u].x, w.x, part);
          part = fma(pv[u].y, w.y, part);
        }
      }
    }
    // fixed-order block partial: lanes of the group (xor butterfly), then the groups in order
    for (int o = L / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o, L);
    if (l == 0) wpart[g] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < G2::GPB; ++k) t += wpart[k];
      a.partial[(long long)sys * G2::RBLK + blockIdx.x] = t;
    }
  } else if (have) {
#pragma unroll 8
    for (int i = 0; i < R; ++i) dst[l + L * i] = reg[l + L * i + i / Q];
  }
}

// cols: op 0: out = T' in ; op 1: out = T' (CT .* T' in) ; op 2: out(external) = sigma T' in
template <int N, int OP>
__global__ void __launch_bounds__(128, 2) k_pcg2_cols(Pcg2 a, const double* in, double* out, int loop) {
  using F = fdst::FG<N>;
  using G2 = Pcg2G<N>;
  constexpr int L = F::L, GROUPS = G2::GROUPS, TC = G2::TC;
  extern __shared__ __align__(16) double2 smp[];
  const int sys = blockIdx.y;
  if (pcg2_skip(a.cg[sys], loop)) return;
  const long long NN = (long long)N * N;
  const int g = threadIdx.x / L, l = threadIdx.x % L;
  const int j0 = blockIdx.x * TC;
  const double* ins = in + (long long)sys * NN;
  const double2 ac = __ldg(&a.wtab[l]);
  const double2* twl = a.wtab + N + l;
  double2* reg = smp + G2::RBASE(g);
  // (kFB items' loads are issued together, ahead of the shared-memory stores)
  constexpr int kFB = 8, kItems = (N / 2) * GROUPS;
  for (int i0 = threadIdx.x; i0 < kItems; i0 += kFB * G2::THREADS) {
    double2 u[kFB], w[kFB];
#pragma unroll
    for (int e = 0; e < kFB; ++e) {
      const int idx = i0 + e * G2::THREADS;
      if (idx < kItems) {
        const int s = idx / GROUPS, c = idx % GROUPS;
        const double2* src = reinterpret_cast<const double2*>(ins + ((long long)s * N + j0 + 2 * c) * 2);
        u[e] = src[0];
        w[e] = src[1];
      }
    }
#pragma unroll
    for (int e = 0; e < kFB; ++e) {
      const int idx = i0 + e * G2::THREADS;
      if (idx < kItems) {
        const int s = idx / GROUPS, c = idx % GROUPS;
        double2* rg = smp + G2::RBASE(c);
        rg[fdst::p2<N>(2 * s)] = make_double2(u[e].x, w[e].x);
        rg[fdst::p2<N>(2 * s + 1)] = make_double2(u[e].y, w[e].y);
      }
    }
  }
  __syncthreads();
  double2* ob = fdst::out_base<N>(reg, l);
  auto put = [&](int j, double a0, double a1, double b0, double b1) {
    ob[2 * j] = make_double2(a0, b0);
    ob[2 * j + 1] = make_double2(a1, b1);
  };
  fdst::pair_dst<N>(reg, reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, put);
  if (OP == 1) {
    __syncwarp();
    const double2* cr = reinterpret_cast<const double2*>(a.CT + (long long)sys * (NN + 2)) +
                        (long long)(j0 / 2 + (g < GROUPS ? g : 0)) * N;
    fdst::pair_dst<N, true>(reg, reg, twl, l, 2.0 * ac.y, 2.0 * ac.x, put, cr + l, cr + N - l);
  }
  __syncthreads();
  if (OP == 2) {
    double* o = out + (long long)sys * a.fs;
    const double sg = a.sigma;
    for (int idx = threadIdx.x; idx < a.m * GROUPS; idx += G2::THREADS) {
      const int i = idx / GROUPS, c = idx % GROUPS;
      const double2 v = smp[G2::RBASE(c) + fdst::p2<N>(i + 1)];
      *reinterpret_cast<double2*>(o + (long long)i * N + j0 + 2 * c) = make_double2(v.x * sg, v.y * sg);
    }
  } else {
    double* o = out + (long long)sys * NN;
    for (int i0 = threadIdx.x; i0 < kItems; i0 += kFB * G2::THREADS) {
      double2 u[kFB], w[kFB];
#pragma unroll
      for (int e = 0; e < kFB; ++e) {
        const int idx = i0 + e * G2::THREADS;
        if (idx < kItems) {
          const int s = idx / GROUPS, c = idx % GROUPS;
          const double2* rg = smp + G2::RBASE(c);
          u[e] = rg[fdst::p2<N>(2 * s)];
          w[e] = rg[fdst::p2<N>(2 * s + 1)];
        }
      }
#pragma unroll
      for (int e = 0; e < kFB; ++e) {
        const int idx = i0 + e * G2::THREADS;
        if (idx < kItems) {
          const int s = idx / GROUPS, c = idx % GROUPS;
          double2* dst = reinterpret_cast<double2*>(o + ((long long)s * N + j0 + 2 * c) * 2);
          dst[0] = make_double2(u[e].x, w[e].x);
          dst[1] = make_double2(u[e].y, w[e].y);
        }
      }
    }
  }
}

CHP_DEV void pcg2_block_pair(double v1, double v2, double* out) {
  __shared__ double w1[32], w2[32];
  for (int o = 16; o > 0; o >>= 1) {
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  if ((threadIdx.x & 31) == 0) { w1[threadIdx.x >> 5] = v1; w2[threadIdx.x >> 5] = v2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { t1 += w1[k]; t2 += w2[k]; }
    out[0] = t1;
    out[1] = t2;
  }
}

// R = SK .* Y ; X = 0 ; partials (R.Mi R, R.R)
template <int N>
__global__ void k_pcg2_init(Pcg2 a) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], false)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  double2* X = reinterpret_cast<double2*>(a.X) + o;
  double2* R = reinterpret_cast<double2*>(a.R) + o;
  const double2* Y = reinterpret_cast<const double2*>(a.Y) + o;
  const double2* Dk = reinterpret_cast<const double2*>(a.Dk);
  const double2* SK = reinterpret_cast<const double2*>(a.SK);
  const double acb = a.cg[s].acbar;
  double v1 = 0.0, v2 = 0.0;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    const double2 y = Y[t], sk = SK[t], mi = pcg2_mi(Dk[t], acb);
    const double2 r = make_double2(y.x * sk.x, y.y * sk.y);
    X[t] = make_double2(0.0, 0.0);
    R[t] = r;
    v1 = fma(r.x, r.x * mi.x, v1);
    v1 = fma(r.y, r.y * mi.y, v1);
    v2 = fma(r.x, r.x, v2);
    v2 = fma(r.y, r.y, v2);
  }
  pcg2_block_pair(v1, v2, a.partial + ((long long)s * kPB + blockIdx.x) * 2);
}

// E3: P = Mi .* R (+ beta P after the first iteration)
template <int N>
__global__ void k_pcg2_pdir(Pcg2 a) {
  const int s = blockIdx.y;
  const CgSys& q = a.cg[s];
  if (pcg2_skip(q, true)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  const double2* R = reinterpret_cast<const double2*>(a.R) + o;
  double2* P = reinterpret_cast<double2*>(a.P) + o;
  const double2* Dk = reinterpret_cast<const double2*>(a.Dk);
  const bool first = q.iters == 0;
  const double beta = q.beta, acb = q.acbar;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    const double2 r = R[t], mi = pcg2_mi(Dk[t], acb);
    double2 p = make_double2(r.x * mi.x, r.y * mi.y);
    if (!first) {
      const double2 po = P[t];
      p = make_double2(fma(beta, po.x, p.x), fma(beta, po.y, p.y));
    }
    P[t] = p;
  }
}

// E1: Y = Dk .* P + Y (Y = a S (c .* S P) on entry: Y = A P) ; partial P.Y
template <int N>
__global__ void k_pcg2_aptail(Pcg2 a, int loop) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], loop)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  const double2* P = reinterpret_cast<const double2*>(a.P) + o;
  double2* Y = reinterpret_cast<double2*>(a.Y) + o;
  const double2* Dk = reinterpret_cast<const double2*>(a.Dk);
  double v1 = 0.0;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    const double2 p = P[t], d = Dk[t], y = Y[t];
    const double2 w = make_double2(fma(d.x, p.x, y.x), fma(d.y, p.y, y.y));
    Y[t] = w;
    v1 = fma(p.x, w.x, v1);
    v1 = fma(p.y, w.y, v1);
  }
  // fixed-order block partial (single value per block, kPB blocks per system)
  __shared__ double w1[32];
  for (int of = 16; of > 0; of >>= 1) v1 += __shfl_xor_sync(0xffffffffu, v1, of);
  if ((threadIdx.x & 31) == 0) w1[threadIdx.x >> 5] = v1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t1 += w1[k];
    a.partial[(long long)s * kPB + blockIdx.x] = t1;
  }
}

// X += alpha P ; R -= alpha Y ; partials (R.Mi R, R.R)
template <int N>
__global__ void k_pcg2_update(Pcg2 a) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], true)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  double2* X = reinterpret_cast<double2*>(a.X) + o;
  double2* R = reinterpret_cast<double2*>(a.R) + o;
  const double2* P = reinterpret_cast<const double2*>(a.P) + o;
  const double2* Y = reinterpret_cast<const double2*>(a.Y) + o;
  const double2* Dk = reinterpret_cast<const double2*>(a.Dk);
  const double al = a.cg[s].alpha, acb = a.cg[s].acbar;
  double v1 = 0.0, v2 = 0.0;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    double2 x = X[t], r = R[t];
    const double2 p = P[t], y = Y[t], mi = pcg2_mi(Dk[t], acb);
    x.x = fma(al, p.x, x.x);
    x.y = fma(al, p.y, x.y);
    r.x = fma(-al, y.x, r.x);
    r.y = fma(-al, y.y, r.y);
    X[t] = x;
    R[t] = r;
    v1 = fma(r.x, r.x * mi.x, v1);
    v1 = fma(r.y, r.y * mi.y, v1);
    v2 = fma(r.x, r.x, v2);
    v2 = fma(r.y, r.y, v2);
  }
  pcg2_block_pair(v1, v2, a.partial + ((long long)s * kPB + blockIdx.x) * 2);
}

// warm start, part a: R = b^ = SK .* Y ; P = x^0 (the X left by the previous
// solve of this system) ; partial |b^|^2 (the tolerance reference, as with x0 = 0)
template <int N>
__global__ void k_pcg2_warm_a(Pcg2 a) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], false)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  const double2* X = reinterpret_cast<const double2*>(a.X) + o;
  double2* R = reinterpret_cast<double2*>(a.R) + o;
  double2* P = reinterpret_cast<double2*>(a.P) + o;
  const double2* Y = reinterpret_cast<const double2*>(a.Y) + o;
  const double2* SK = reinterpret_cast<const double2*>(a.SK);
  double v1 = 0.0;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    const double2 y = Y[t], sk = SK[t];
    const double2 r = make_double2(y.x * sk.x, y.y * sk.y);
    R[t] = r;
    P[t] = X[t];
    v1 = fma(r.x, r.x, v1);
    v1 = fma(r.y, r.y, v1);
  }
  pcg2_block_pair(v1, 0.0, a.partial + ((long long)s * kPB + blockIdx.x) * 2);
}

// warm start, part b: R = b^ - A x^0 (A x^0 in Y) ; partials (R.Mi R, R.R)
template <int N>
__global__ void k_pcg2_warm_b(Pcg2 a) {
  const int s = blockIdx.y;
  if (pcg2_skip(a.cg[s], false)) return;
  const long long NN = (long long)N * N, o = (long long)s * (NN / 2);
  double2* R = reinterpret_cast<double2*>(a.R) + o;
  const double2* Y = reinterpret_cast<const double2*>(a.Y) + o;
  const double2* Dk = reinterpret_cast<const double2*>(a.Dk);
  const double acb = a.cg[s].acbar;
  double v1 = 0.0, v2 = 0.0;
#pragma unroll 4
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NN / 2;
       t += (long long)gridDim.x * blockDim.x) {
    const double2 y = Y[t], rb = R[t], mi = pcg2_mi(Dk[t], acb);
    const double2 r = make_double2(rb.x - y.x, rb.y - y.y);
    R[t] = r;
    v1 = fma(r.x, r.x * mi.x, v1);
    v1 = fma(r.y, r.y * mi.y, v1);
    v2 = fma(r.x, r.x, v2);
    v2 = fma(r.y, r.y, v2);
  }
  pcg2_block_pair(v1, v2, a.partial + ((long long)s * kPB + blockIdx.x) * 2);
}
