// LINEAR_B fine propagator, v2 passes (schemes.py:249-267 step_linear_b):
//   x_{n+1} = S D S (x_n + dt L(x_n^3 - 3 x_n)),  S = (2/N) T_i T_j (orthonormal 2D DST-I),
//   D = 1 / (1 - 2 dt lam + eps^2 dt lam^2),  lam = lam_p + lam_q (grid.py:127-144).
//
// HBM layout of the two scratch fields per system (N x N doubles each; math
// rows 0..N, 0 and N the zero Dirichlet rows; math column q = storage column q,
// column 0 the zero pad):
//   P (state between steps; row-spectral, column-physical): "pair-interleaved",
//     rows stored two at a time, element (row pair s = rows (2s, 2s+1), column q,
//     h) at (s N + q) * 2 + h: the row pass copies a pair of rows with
//     contiguous 16-byte cp.async; the column pass writes 32 contiguous bytes
//     per (row pair, column pair).
//   Q (row-spectral rhs): row-major, math row i at storage row i: the column
//     pass fills its tile with 16-byte cp.async of (Q[i][q], Q[i][q+1]).
//
// One step = one row pass + one column pass = 32 B of HBM per grid-point-step:
//   row pass  (sliding window over a strip of row pairs, G lane groups per block):
//             phase 0: x = T'_j P for pair p0+g   (cp.async pair -> slot -> transform)
//             phase 1: rhs = x + dt L(x^3 - 3x) for the shifted pair p0-1+g from
//                      the x slots (halo rows come from the neighbouring slot),
//                      Q = T'_j rhs -> staged in the slot -> coalesced row stores
//             the slot ring has G+1 slots: the last phase-0 pair of a chunk is the
//             carried halo of the next, so each row is transformed once per phase.
//   column pass (GROUPS column pairs per block): P = T'_i (D'' .* T'_i Q), the
//             divisors applied in the forward transform's post-processing from a
//             table laid out in the post-processing's chunk order (coalesced,
//             each value read once)
// T' = 4T (chp_fdst.cuh); all normalisations live in D'' = (2/N)^2 D / 256.
#pragma once
#include "chp_fdst.cuh"

#ifndef CHP_ROW_WARPS
#define CHP_ROW_WARPS 4
#endif
#ifndef CHP_ROW_MINB
#define CHP_ROW_MINB 2
#endif
#ifndef CHP_COL_WARPS
#define CHP_COL_WARPS 4
#endif
#ifndef CHP_COL_MINB
#define CHP_COL_MINB 2
#endif

namespace linb {

template <int N> struct RowG {          // row pass geometry
  using F = fdst::FG<N>;
  static constexpr int L = F::L;
  static constexpr int WARPS = (N >= 1024) ? CHP_ROW_WARPS : (N >= 256 ? 4 : 2);
  static constexpr int THREADS = WARPS * 32;
  static constexpr int G = THREADS / L;              // lane groups = row pairs per chunk
  static constexpr int NP = N / 2;                   // row pairs per field
  // phase-1 pairs per strip: a strip of SP pairs transforms SP + 1 pairs in phase 0 in
  // ceil((SP + 1) / G) chunks of G, so SP = 63 (64 / G chunks, 1.6 % halo overhead)
  static constexpr int SP = (NP < 64) ? NP : 63;
  static constexpr int SLOTS = G + 1;
  static constexpr size_t SMEM = sizeof(double2) * (size_t)SLOTS * F::RS;
  static constexpr int MINB = (N >= 1024) ? CHP_ROW_MINB : 3;
};

template <int N> struct ColG {          // column pass geometry
  using F = fdst::FG<N>;
  static constexpr int L = F::L;
  static constexpr int WARPS = (N >= 1024) ? CHP_COL_WARPS : (N >= 256 ? 4 : 2);
  static constexpr int THREADS = WARPS * 32;
  static constexpr int GALL = THREADS / L;
  static constexpr int GROUPS = (GALL < N / 2) ? GALL : N / 2;   // column pairs per block
  static constexpr int TC = 2 * GROUPS;
  // region base of group c: c * RS + 2 (c >> 1) keeps the tile fill conflict free
  static constexpr int RBASE(int c) { return c * F::RS + 2 * (c >> 1); }
  static constexpr size_t SMEM = sizeof(double2) * (size_t)(RBASE(GALL - 1) + F::RS);
  static constexpr int MINB = (N >= 512) ? CHP_COL_MINB : 3;
};

enum { MODE_FIRST = 0, MODE_MID = 1, MODE_LAST = 2 };

struct RowArgs {
  const double* in;       // MID/LAST: P (pair-interleaved); FIRST: physical field (external layout)
  long long in_stride;
  const int* in_index;    // FIRST: system -> input field (nullable)
  double* out;            // FIRST/MID: Q (pair-interleaved); LAST: physical field (external)
  long long out_stride;
  const int* out_index;   // LAST: system -> output field (nullable)
  int m;
  double cdt;             // dt / h^2
  int mode;
  chp_sys_info* info;
  const int* info_index;
  const double2* wtab;    // (cos, sin)(pi l / N) at [l], W_N^{l k2} at [N + k2 L + l]
};

CHP_DEV void cp16(void* sdst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
CHP_DEV void cp_wait() { asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory"); }

CHP_DEV double wcub(double x) { return x * fma(x, x, -3.0); }   // x^3 - 3x

// one 32-byte global store (STG.256 on sm_100)
CHP_DEV void st256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d) : "memory");
}

// Q's column-pair order (the row pass stores from registers, the column pass fills a
// tile of consecutive positions): column pair k sits at pair position qpos(k).  Lane
// l of the row pass holds k = C l + j (j < C); runs of V = min(4, C) consecutive k
// stay adjacent and the runs of one j / V are laid out lane by lane, so a store
// instruction covers V-pair runs of consecutive lanes, and GROUPS consecutive
// positions of the column pass are whole runs of consecutive k (its P write-out
// stays 128-byte coalesced).
template <int N> struct QPos {
  static constexpr int L = fdst::FG<N>::L, C = fdst::FG<N>::C;
  static constexpr int V = C < 4 ? C : 4, G4 = C / V;
};
template <int N> CHP_DEV int qpos(int k) {
  using QP = QPos<N>;
  const int b = k / QP::V;
  return QP::V * ((b % QP::G4) * QP::L + b / QP::G4) + k % QP::V;
}
template <int N> CHP_DEV int qpos_inv(int p) {
  using QP = QPos<N>;
  const int grp = p / QP::V;
  return QP::V * ((grp % QP::L) * QP::G4 + grp / QP::L) + p % QP::V;
}

// SPV: phase-1 row pairs per strip (compile time, so the chunk loop has a fixed trip
// count); short strips for small batches are separate instantiations
template <int N, int SPV = RowG<N>::SP>
__global__ void __launch_bounds__(RowG<N>::THREADS, RowG<N>::MINB) k2d_rowb(RowArgs a) {
  using F = fdst::FG<N>;
  using RG = RowG<N>;
  constexpr int L = F::L, R = F::R, Q = F::Q, C = F::C, RS = F::RS, G = RG::G, SL = RG::SLOTS;
  extern __shared__ __align__(16) double2 slots[];
  const int tid = threadIdx.x, g = tid / L, l = tid % L;
  const int sys = blockIdx.y;
  const int sp0 = blockIdx.x * SPV;
  const int sp1 = min(sp0 + SPV, RG::NP);              // phase-1 pairs [sp0, sp1)
  constexpr int chunks = (SPV + 1 + G - 1) / G;
  const double2 ac = __ldg(&a.wtab[l]);
  const double sa2 = 2.0 * ac.y, ca2 = 2.0 * ac.x;
  const double2* twl = a.wtab + N + l;
  const int m = a.m;
  const double cdt = a.cdt;

  if (a.mode == MODE_LAST) {
    // x = T' P for pairs [sp0, sp1) -> physical rows (2s, 2s+1) = storage rows 2s-1, 2s
    const long long fo = a.out_index ? a.out_index[sys] : sys;
    const double* P = a.in + (long long)sys * a.in_stride;
    double* out = a.out + fo * a.out_stride;
    double2* reg = slots + g * RS;
    double fin = 0.0;
    for (int s0 = sp0; s0 < sp1; s0 += G) {
      const int s = s0 + g;
      const bool have = s < sp1;
      const double2* src = reinterpret_cast<const double2*>(P + (long long)(have ? s : sp0) * 2 * N);
#pragma unroll 4
      for (int i = 0; i < R; ++i) cp16(&reg[l + L * i + i / Q], &src[l + L * i]);
      cp_wait();
      __syncwarp();
      double2* ob = fdst::out_base<N>(reg, l);
      fdst::pair_dst<N>(reg, reg, twl, l, sa2, ca2, [&](int j, double a0, double a1, double b0, double b1) {
        ob[2 * j] = make_double2(a0, b0);
        ob[2 * j + 1] = make_double2(a1, b1);
      });
      __syncwarp();
      if (have) {
        // coalesced copy-out: lane covers column pairs (2c, 2c+1), c = l + L i
        const int ra = 2 * s - 1, rb = 2 * s;          // storage rows
#pragma unroll 4
        for (int i = 0; i < N / 2 / L; ++i) {
          const int c = l + L * i;
          const double2 u = reg[fdst::p2<N>(2 * c)], w = reg[fdst::p2<N>(2 * c + 1)];
          fin = fma(u.x, 0.0, fma(u.y, 0.0, fma(w.x, 0.0, fma(w.y, 0.0, fin))));
          if (ra >= 0) *reinterpret_cast<double2*>(out + (long long)ra * N + 2 * c) = make_double2(u.x, w.x);
          if (rb < m) *reinterpret_cast<double2*>(out + (long long)rb * N + 2 * c) = make_double2(u.y, w.y);
        }
      }
      __syncwarp();
    }
    if (__syncthreads_or(fin != 0.0) && tid == 0) {
      const long long fi = a.info_index ? a.info_index[sys] : sys;
      atomicCAS(&a.info[fi].status, CHP_SYS_OK, CHP_SYS_NONFINITE);
    }
    return;
  }

  double* Qo = a.out + (long long)sys * a.out_stride;
  const double* Pin = nullptr;
  const double* U = nullptr;
  if (a.mode == MODE_MID) Pin = a.in + (long long)sys * a.in_stride;
  else U = a.in + (a.in_index ? (long long)a.in_index[sys] : (long long)sys) * a.in_stride;

  for (int t = 0; t < chunks; ++t) {
    const int p0 = sp0 + t * G;
    // ---- phase 0: slot of pair s0 = p0 + g holds x rows (2 s0, 2 s0 + 1) ----
    {
      const int s0 = p0 + g;
      double2* reg = slots + ((t * G + g) % SL) * RS;
      const bool load = s0 <= sp1 && s0 < RG::NP;
      if (a.mode == MODE_MID) {
        const double2* src = reinterpret_cast<const double2*>(Pin + (long long)(load ? s0 : 0) * 2 * N);
        if (load) {
#pragma unroll 4
          for (int i = 0; i < R; ++i) cp16(&reg[l + L * i + i / Q], &src[l + L * i]);
        } else {
#pragma unroll 4
          for (int i = 0; i < R; ++i) reg[l + L * i + i / Q] = make_double2(0.0, 0.0);
        }
        cp_wait();
        __syncwarp();
        double2* ob = fdst::out_base<N>(reg, l);
        fdst::pair_dst<N>(reg, reg, twl, l, sa2, ca2, [&](int j, double a0, double a1, double b0, double b1) {
          ob[2 * j] = make_double2(a0, b0);
          ob[2 * j + 1] = make_double2(a1, b1);
        });
      } else {
        // first step: x is the physical input (storage row i-1 = math row i)
        const int ra = 2 * s0 - 1, rb = 2 * s0;
#pragma unroll 4
        for (int i = 0; i < R; ++i) {
          const int n = l + L * i;
          double xa = 0.0, xb = 0.0;
          if (load && n > 0) {
            if (ra >= 0) xa = U[(long long)ra * N + n];
            if (rb < m) xb = U[(long long)rb * N + n];
          }
          reg[l + L * i + i / Q] = make_double2(xa, xb);
        }
      }
    }
    __syncthreads();
    // ---- phase 1: rhs of rows (2 s1 + 1, 2 s1 + 2), s1 = p0 - 1 + g ----------
    const int s1 = p0 - 1 + g;
    const bool act = s1 >= sp0 && s1 < sp1;
    double2* r0 = slots + ((t * G + g + SL - 1) % SL) * RS;   // pair s1: rows 2s1, 2s1+1
    const double2* r1 = slots + ((t * G + g) % SL) * RS;      // pair s1+1: rows 2s1+2, 2s1+3
    double2 rhs[R];                                            // lane chunk n = R l + i
    {
      const int nb = R * l;
      const double2* u0 = r0 + (R + 1) * l;                    // p2(R l + i) = (R+1) l + i
      const double2* u1 = r1 + (R + 1) * l;
      // left neighbour (n = nb - 1) and right neighbour (n = nb + R)
      double2 ul = make_double2(0.0, 0.0), vl = make_double2(0.0, 0.0);
      if (l > 0) { ul = u0[-2]; vl = u1[-2]; }
      double2 ur = make_double2(0.0, 0.0), vr = make_double2(0.0, 0.0);
      if (l < L - 1) { ur = u0[R + 1]; vr = u1[R + 1]; }
      // rows: A = 2s1 (u.x), B = 2s1+1 (u.y), Cc = 2s1+2 (v.x), D = 2s1+3 (v.y)
      double wBl = wcub(ul.y), wCl = wcub(vl.x);
      double2 u = u0[0], v = u1[0];
      double wB = wcub(u.y), wC = wcub(v.x);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double2 un, vn;
        if (i + 1 < R) { un = u0[i + 1]; vn = u1[i + 1]; }
        else { un = ur; vn = vr; }
        const double wBr = wcub(un.y), wCr = wcub(vn.x);
        const double wA = wcub(u.x), wD = wcub(v.y);
        // L w at (B, n) and (C, n): up + down + left + right - 4 centre, times dt/h^2
        const double sB = fma(-4.0, wB, ((wA + wC) + (wBl + wBr)));
        const double sC = fma(-4.0, wC, ((wB + wD) + (wCl + wCr)));
        rhs[i] = make_double2(fma(cdt, sB, u.y), fma(cdt, sC, v.x));
        wBl = wB; wCl = wC; wB = wBr; wC = wCr;
        u = un; v = vn;
      }
      (void)nb;
    }
    __syncthreads();                                           // every slot's x has been read
    {
      double2* w0 = r0 + (R + 1) * l;
#pragma unroll
      for (int i = 0; i < R; ++i) w0[i] = rhs[i];
      __syncwarp();
      // Q rows 2s1+1 (a) and 2s1+2 (b, absent for the last pair) straight from the
      // post-processing registers (no staging): see qpos for the column-pair order.
      // Consecutive outputs j, j+1 of a lane are adjacent pairs: one 32-byte store.
      const int ra = 2 * s1 + 1, rb = ra + 1;
      double* qa = Qo + (long long)(act ? ra : 0) * N;
      double* qb = Qo + (long long)(act && rb < N ? rb : 0) * N;
      const bool sta = act, stb = act && rb < N;
      double pa0 = 0.0, pa1 = 0.0, pb0 = 0.0, pb1 = 0.0;
      fdst::pair_dst<N>(r0, r0, twl, l, sa2, ca2, [&](int j, double a0, double a1, double b0, double b1) {
        if ((j & 1) == 0) {
          pa0 = a0; pa1 = a1; pb0 = b0; pb1 = b1;
          return;
        }
        const int pos = qpos<N>(F::C * l + j - 1);
        if (sta) st256(qa + 2 * pos, pa0, pa1, a0, a1);
        if (stb) st256(qb + 2 * pos, pb0, pb1, b0, b1);
      });
      __syncwarp();
    }
  }
}

struct ColArgs {
  const double* qin;       // Q (row-major, math row i at row i, column pairs in qpos order)
  double* pout;            // P (pair-interleaved, pairs (2s, 2s+1))
  long long stride;        // doubles per system (N*N)
  const double2* dtab;     // [q/2][(2j+h) L + l]: (D''(p, q), D''(p, q+1)), p = 2(C l + j) + h
  const double2* wtab;
};

template <int N>
__global__ void __launch_bounds__(ColG<N>::THREADS, ColG<N>::MINB) k2d_colb(ColArgs a) {
  using F = fdst::FG<N>;
  using CG = ColG<N>;
  constexpr int L = F::L, GROUPS = CG::GROUPS, TC = CG::TC;
  extern __shared__ __align__(16) double2 tile[];
  const int tid = threadIdx.x, g = tid / L, l = tid % L;
  const int sys = blockIdx.y;
  const int j0 = blockIdx.x * TC;
  const double* Qs = a.qin + (long long)sys * a.stride;
  double* Ps = a.pout + (long long)sys * a.stride;
  // ---- fill: Q rows 1..N-1 of columns j0 .. j0+TC-1 -> region c (p2 layout) --
  {
    constexpr int ITEMS = (N - 1) * GROUPS;
#pragma unroll 4
    for (int idx = tid; idx < ITEMS; idx += CG::THREADS) {
      const int i = 1 + idx / GROUPS, c = idx % GROUPS;
      cp16(&tile[CG::RBASE(c) + fdst::p2<N>(i)], Qs + (long long)i * N + j0 + 2 * c);
    }
    cp_wait();
  }
  __syncthreads();
  // every lane group runs (groups beyond the tile, tiny N only, work on their
  // own scratch region and store nothing) so that whole warps stay converged
  double2* reg = tile + CG::RBASE(g);
  {
    const double2 ac = __ldg(&a.wtab[l]);
    const double sa2 = 2.0 * ac.y, ca2 = 2.0 * ac.x;
    const double2* twl = a.wtab + N + l;
    double2* ob = fdst::out_base<N>(reg, l);
    auto put = [&](int j, double a0, double a1, double b0, double b1) {
      ob[2 * j] = make_double2(a0, b0);
      ob[2 * j + 1] = make_double2(a1, b1);
    };
    // D'' of the column pair (j0 + 2g, j0 + 2g + 1) scales the forward transform's
    // outputs in its post-processing (chunk-layout table, each value read once)
    const double2* dr = a.dtab + (long long)qpos_inv<N>(j0 / 2 + (g < GROUPS ? g : 0)) * N + l;
    fdst::pair_dst<N, false, true>(reg, reg, twl, l, sa2, ca2, put, nullptr, nullptr, dr);
    __syncwarp();
    fdst::pair_dst<N>(reg, reg, twl, l, sa2, ca2, put);
  }
  __syncthreads();
  // ---- write-out: P pairs (2s, 2s+1), s = 0..N/2-1 -----------------------------
  {
    constexpr int ITEMS = (N / 2) * GROUPS;
#pragma unroll 4
    for (int idx = tid; idx < ITEMS; idx += CG::THREADS) {
      const int s = idx / GROUPS, c = idx % GROUPS;
      const double2* rg = tile + CG::RBASE(c);
      const double2 u = rg[fdst::p2<N>(2 * s)], w = rg[fdst::p2<N>(2 * s + 1)];
      double2* dst = reinterpret_cast<double2*>(Ps + ((long long)s * N + 2 * qpos_inv<N>(j0 / 2 + c)) * 2);
      __stcs(dst, make_double2(u.x, w.x));
      __stcs(dst + 1, make_double2(u.y, w.y));
    }
  }
}

}  // namespace linb
