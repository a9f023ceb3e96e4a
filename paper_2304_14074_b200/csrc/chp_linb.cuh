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
#include <cuda.h>            // CUtensorMap (type only; the encoder is resolved at run time)
#include "chp_fdst.cuh"

// N = 1024 block shapes (profiles/r02_linb_ab.md): row pass 4 warps x 2 blocks per SM (a 5-slot
// ring: fewer chunks per strip and fewer block barriers than 2 x 4), column pass 2 warps x 4
// blocks per SM (2-pair tiles: four independent blocks interleave their tile load / transform /
// store phases where two 4-warp blocks left the SM waiting on both tiles at once).
#ifndef CHP_ROW_WARPS
#define CHP_ROW_WARPS 4
#endif
#ifndef CHP_ROW_MINB
#define CHP_ROW_MINB 2
#endif
#ifndef CHP_COL_WARPS
#define CHP_COL_WARPS 2
#endif
#ifndef CHP_COL_MINB
#define CHP_COL_MINB 4
#endif

namespace linb {

// N = 1024 strip length.  Every block runs ceil((SP + 1) / G) chunks whatever its strip holds,
// so what counts is strips x chunks per field: 63 gives 9 x 16 = 144 chunk slots for the 512 + 9
// pairs a field needs (the ninth strip has 8 pairs and ran 13 chunks on zeros); 57 gives nine
// equal strips of 15 chunks = 135 (-6 %).  Measured per 16 steps of 512 / 256 / 64 slices:
// 63: 104.4 / 52.4 / 13.5 ms; 57: 100.4 / 50.2 / 12.9; 52: 102.0 / 51.2 / 14.1; 74: 100.0 / 50.7 /
// 14.6; 86: 100.3 / 50.5 / 14.3; 103: 99.7 / 50.1 / 15.6 (too few blocks for small batches).
#ifndef CHP_ROW_SP
#define CHP_ROW_SP 57
#endif
template <int N> struct RowG {          // row pass geometry
  using F = fdst::FG<N>;
  static constexpr int L = F::L;
  static constexpr int WARPS = (N >= 1024) ? CHP_ROW_WARPS : (N >= 256 ? 4 : 2);
  static constexpr int THREADS = WARPS * 32;
  static constexpr int G = THREADS / L;              // lane groups = row pairs per chunk
  static constexpr int NP = N / 2;                   // row pairs per field
  // phase-1 pairs per strip: a strip of SP pairs transforms SP + 1 pairs in phase 0 in
  // ceil((SP + 1) / G) chunks of G (63: 64 / G chunks, 1.6 % halo overhead; N = 1024: see
  // CHP_ROW_SP above)
  static constexpr int SP = (NP < 64) ? NP : (N >= 1024 ? CHP_ROW_SP : 63);
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

CHP_DEV unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
CHP_DEV void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
CHP_DEV void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
CHP_DEV void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra LAB_DONE_%=;\n bra LAB_WAIT_%=;\n LAB_DONE_%=:\n}" ::"r"(smem_u32(b)), "r"(parity)
      : "memory");
}
CHP_DEV void tma_load_2d(void* sdst, const CUtensorMap* map, int c0, int c1, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(sdst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(b)) : "memory");
}

// one contiguous global -> shared bulk copy (UBLKCP), completion on an mbarrier
CHP_DEV void bulk_load(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
CHP_DEV void fence_async_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// loader of a transform whose input is an unpadded pair vector (a row pair as the bulk
// copy lands it): v = src[l + L n2], mirror src[N - l - L n2] (src[N] for n = 0: discarded)
template <int N> struct PlainLd {
  const double2 *vb, *wb;
  CHP_DEV PlainLd(const double2* src, int l) : vb(src + l), wb(src + N - l) {}
  CHP_DEV double2 v(int n2) const { return vb[fdst::FG<N>::L * n2]; }
  CHP_DEV double2 w(int n2) const { return wb[-fdst::FG<N>::L * n2]; }
};

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
  // MODE_MID, one warp per pair (N = 1024): each group's row pair arrives by one bulk copy
  // (UBLKCP) on the group's mbarrier; narrower groups (two or more per warp, 4 KB pairs or
  // less) keep the per-thread cp.async fill, which measured faster there
  constexpr bool BULK = (L == 32);
  constexpr bool PADC = (Q == 1);          // pad copies for the second transform's mirror reads
  __shared__ __align__(8) unsigned long long rbar[G];
  unsigned rphase = 0;
  if (BULK && a.mode == MODE_MID) {
    if (tid == 0) {
#pragma unroll
      for (int i = 0; i < G; ++i) mbar_init(&rbar[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      fence_async_proxy();
    }
    __syncthreads();
  }

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

  double2 xo[R];                                               // the group's own x pair (phase 0 -> 1)
  // chunks this strip needs: phase 1 of chunk t covers pairs sp0 + t G - 1 ... sp0 + t G + G - 2,
  // so a short last strip (NP = 8 x 63 + 8 at N = 1024) stops after (sp1 - sp0) / G + 1 chunks
  // instead of running the remaining ones on zeros
#ifndef CHP_ROW_EARLY
#define CHP_ROW_EARLY 0
#endif
  const int nch = CHP_ROW_EARLY ? min(chunks, (sp1 - sp0) / G + 1) : chunks;
  for (int t = 0; t < nch; ++t) {
    const int p0 = sp0 + t * G;
    // ---- phase 0: slot of pair s0 = p0 + g holds x rows (2 s0, 2 s0 + 1) ----
    {
      const int s0 = p0 + g;
      double2* reg = slots + ((t * G + g) % SL) * RS;
      const bool load = s0 <= sp1 && s0 < RG::NP;
      if (a.mode == MODE_MID) {
        // the copy of chunk t > 0 was issued from the previous chunk's phase 1 (below)
        if (load) {
          if constexpr (BULK) {
            if (t == 0 && l == 0) {
              mbar_expect_tx(&rbar[g], 16u * N);
              bulk_load(reg, Pin + (long long)s0 * 2 * N, 16u * N, &rbar[g]);
            }
            mbar_wait(&rbar[g], rphase);
            rphase ^= 1;
          } else {
            const double2* src = reinterpret_cast<const double2*>(Pin + (long long)s0 * 2 * N);
#pragma unroll 4
            for (int i = 0; i < R; ++i) cp16(&reg[l + L * i], &src[l + L * i]);
            cp_wait();
          }
        } else {
#pragma unroll 4
          for (int i = 0; i < R; ++i) reg[l + L * i] = make_double2(0.0, 0.0);
        }
        __syncwarp();
        // x goes to the slot for the neighbouring group (its rows A, B) and stays in this
        // lane's registers for the group's own phase 1 (rows C, D): lane chunk n = R l + i
        double2* ob = fdst::out_base<N>(reg, l);
        fdst::pair_dst_ld<N>(PlainLd<N>(reg, l), reg, twl, l, sa2, ca2,
                             [&](int j, double a0, double a1, double b0, double b1) {
          xo[2 * j] = make_double2(a0, b0);
          xo[2 * j + 1] = make_double2(a1, b1);
          ob[2 * j] = xo[2 * j];
          ob[2 * j + 1] = xo[2 * j + 1];
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
#pragma unroll
        for (int i = 0; i < R; ++i) xo[i] = make_double2(0.0, 0.0);   // defined on every path: never live across a chunk
      }
    }
    __syncthreads();
    // ---- phase 1: rhs of rows (2 s1 + 1, 2 s1 + 2), s1 = p0 - 1 + g ----------
    const int s1 = p0 - 1 + g;
    const bool act = s1 >= sp0 && s1 < sp1;
    double2* r0 = slots + ((t * G + g + SL - 1) % SL) * RS;   // pair s1: rows 2s1, 2s1+1
    const double2* r1 = slots + ((t * G + g) % SL) * RS;      // pair s1+1: rows 2s1+2, 2s1+3
    {
      double2* u0 = r0 + (R + 1) * l;                          // p2(R l + i) = (R+1) l + i
      if (a.mode != MODE_MID) {
        // first step: x was loaded straight into the slots; pick up the group's own pair
        // before the neighbouring group rewrites that slot in place
        const double2* u1 = r1 + (R + 1) * l;
#pragma unroll
        for (int i = 0; i < R; ++i) xo[i] = u1[i];
        __syncthreads();
      }
      // Rows A = 2s1, B = 2s1+1 come from the neighbouring group's slot r0, rows C = 2s1+2,
      // D = 2s1+3 are this group's own pair, still in registers (xo).  Left neighbour
      // (n = R l - 1) and right neighbour (n = R l + R): r0's through shared memory, the own
      // pair's from the adjacent lanes' registers.  Nobody else touches r0 in this phase, so the
      // rhs replaces x in place as the sweep goes (after every lane's edge reads).
      double2 ul = make_double2(0.0, 0.0), ur = make_double2(0.0, 0.0);
      if (l > 0) ul = u0[-2];
      if (l < L - 1) ur = u0[R + 1];
      double vlx = __shfl_up_sync(0xffffffffu, xo[R - 1].x, 1, L);
      double vrx = __shfl_down_sync(0xffffffffu, xo[0].x, 1, L);
      if (l == 0) vlx = 0.0;
      if (l == L - 1) vrx = 0.0;
      __syncwarp();
      double wBl = wcub(ul.y), wCl = wcub(vlx);
      double2 u = u0[0], v = xo[0];
      double wB = wcub(u.y), wC = wcub(v.x);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double2 un;
        double vnx;
        if (i + 1 < R) { un = u0[i + 1]; vnx = xo[i + 1].x; }
        else { un = ur; vnx = vrx; }
        const double wBr = wcub(un.y), wCr = wcub(vnx);
        const double wA = wcub(u.x), wD = wcub(v.y);
        // L w at (B, n) and (C, n): up + down + left + right - 4 centre, times dt/h^2
        const double sB = fma(-4.0, wB, ((wA + wC) + (wBl + wBr)));
        const double sC = fma(-4.0, wC, ((wB + wD) + (wCl + wCr)));
        const double2 rh = make_double2(fma(cdt, sB, u.y), fma(cdt, sC, v.x));
        u0[i] = rh;
        if (PADC && i == 0 && l > 0) u0[-1] = rh;               // pad copy of the chunk's first column
        wBl = wB; wCl = wC; wB = wBr; wC = wCr;
        u = un;
        if (i + 1 < R) v = xo[i + 1];
        // keep the x loads of later columns from being hoisted over the whole sweep (their
        // registers are what the own pair occupies)
        if ((i & 3) == 3) asm volatile("" ::: "memory");
      }
    }
    {
      __syncwarp();
      // Q rows 2s1+1 (a) and 2s1+2 (b, absent for the last pair) straight from the
      // post-processing registers (no staging): see qpos for the column-pair order.
      // Consecutive outputs j, j+1 of a lane are adjacent pairs: one 32-byte store.
      const int ra = 2 * s1 + 1, rb = ra + 1;
      double* qa = Qo + (long long)(act ? ra : 0) * N;
      double* qb = Qo + (long long)(act && rb < N ? rb : 0) * N;
      const bool sta = act, stb = act && rb < N;
      double pa0 = 0.0, pa1 = 0.0, pb0 = 0.0, pb1 = 0.0;
      // r0 is this group's phase-0 slot of the next chunk: its row pair is requested as soon
      // as the transform has read its last value from the slot (the callbacks run after that)
      const int sn = p0 + G + g;
      const bool prefetch = BULK && a.mode == MODE_MID && t + 1 < chunks && sn <= sp1 && sn < RG::NP;
      fdst::pair_dst_ld<N>(fdst::SmemLd<N, PADC>(r0, l), r0, twl, l, sa2, ca2,
                           [&](int j, double a0, double a1, double b0, double b1) {
        if ((j & 1) == 0) {
          if (j == 0 && prefetch && l == 0) {
            fence_async_proxy();
            mbar_expect_tx(&rbar[g], 16u * N);
            bulk_load(r0, Pin + (long long)sn * 2 * N, 16u * N, &rbar[g]);
          }
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

// ---------------------------------------------------------------------------
// Column pass with a TMA tile (N >= 64): the block's Q tile -- rows 0..N-1 of its
// GROUPS column pairs, IB = 16 GROUPS bytes per row -- is fetched by cp.async.bulk.tensor
// (UTMALDG) boxes of up to 256 rows into a hardware-swizzled row-major tile (64- or
// 128-byte swizzle: the 16-byte chunk index is XORed with row bits, which makes a lane
// group's stride-IB column reads bank-conflict free) instead of per-thread 16-byte
// cp.async whose 32 lanes each hit a different row (one shared-memory wavefront per
// lane).  The forward transform's pre-processing reads the tile directly (TileLd); after
// a block barrier the tile's memory becomes the groups' private regions.  The inverse
// transform's outputs go to P straight from the post-processing registers: a lane holds
// rows (2k, 2k+1) of both columns of its pair = 32 contiguous bytes of P.
// ---------------------------------------------------------------------------
CHP_DEV void tma_store_3d(const CUtensorMap* map, const void* ssrc, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(ssrc)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
CHP_DEV void tma_store_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int N> struct ColT {          // TMA column pass geometry
  using F = fdst::FG<N>;
  using CG = ColG<N>;
  static constexpr int L = F::L, GROUPS = CG::GROUPS;
  static constexpr int IB = 16 * GROUPS;                 // tile row bytes: 64 or 128
  static constexpr int BR = N < 256 ? N : 256;           // rows per TMA box
  static constexpr int NBOX = N / BR;
  static constexpr size_t TILE = (size_t)N * IB;
  static constexpr size_t REGIONS = sizeof(double2) * (size_t)(CG::RBASE(CG::GALL - 1) + F::RS);
  // lane 0's mirror of n = 0 reads row N (one row past the tile; the value is discarded)
  static constexpr size_t SMEM = 1024 + (TILE + IB > REGIONS ? TILE + IB : REGIONS);
  static_assert(N >= 64 && CG::GROUPS == CG::GALL && (IB == 32 || IB == 64 || IB == 128),
                "TMA column pass geometry");
  // 16-byte chunk XOR of the hardware swizzle for tile row r (64B: bits 7-8 of the byte
  // offset = (r >> 1) & 3; 128B: bits 7-9 = r & 7)
  // (32B: bit 7 = (r >> 2) & 1)
  CHP_DEV static int swz(int r) { return IB == 32 ? ((r >> 2) & 1) : (IB == 64 ? ((r >> 1) & 3) : (r & 7)); }
  // P leaves through one TMA store (UTMASTG) when the block's pairs span 128 bytes of a P
  // row pair (GROUPS = 4: N = 1024): the inverse transform's outputs are staged in a
  // 128-byte-swizzled tile [j][l][128 B] (row pair k = C l + j at tile row j L + l, so the
  // 32 lanes of a store instruction hit 32 consecutive tile rows: conflict free), and the
  // tensor map's dimension order {columns, l, j} scatters the tile rows to P's row pairs
  // (GROUPS = 2: 64-byte tile rows with the 64-byte swizzle, XOR term (row >> 1) & 3)
  static constexpr bool PSTORE = (GROUPS == 4 || GROUPS == 2);
  static constexpr int PB = 32 * GROUPS;                  // P tile row bytes: 128 or 64
  static constexpr size_t PTILE = (size_t)(N / 2) * PB;
  CHP_DEV static int pswz(int l) { return PB == 128 ? (l & 7) : ((l >> 1) & 3); }
};

// loader of the forward transform: column pair g of the swizzled tile.  Rows l + L n2 and
// N - l - L n2 keep their swizzle term for every n2 (L n2 is a multiple of 8).
template <int N> struct TileLd {
  const unsigned char *vb, *wb;
  CHP_DEV TileLd(const unsigned char* tile, int g, int l)
      : vb(tile + l * ColT<N>::IB + ((g ^ ColT<N>::swz(l)) << 4)),
        wb(tile + (N - l) * ColT<N>::IB + ((g ^ ColT<N>::swz(N - l)) << 4)) {}
  CHP_DEV double2 v(int n2) const {
    return *reinterpret_cast<const double2*>(vb + n2 * (fdst::FG<N>::L * ColT<N>::IB));
  }
  CHP_DEV double2 w(int n2) const {
    return *reinterpret_cast<const double2*>(wb - n2 * (fdst::FG<N>::L * ColT<N>::IB));
  }
};

template <int N>
__global__ void __launch_bounds__(ColG<N>::THREADS, ColG<N>::MINB)
k2d_colt(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap pmap, ColArgs a) {
  using F = fdst::FG<N>;
  using CG = ColG<N>;
  using CT = ColT<N>;
  constexpr int L = F::L, TC = CG::TC;
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned char* tile = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, g = tid / L, l = tid % L;
  const int sys = blockIdx.y;
  const int j0 = blockIdx.x * TC;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar, (unsigned)CT::TILE);
#pragma unroll
    for (int b = 0; b < CT::NBOX; ++b)
      tma_load_2d(tile + (size_t)b * CT::BR * CT::IB, &qmap, j0, sys * N + b * CT::BR, &bar);
  }
  double* Ps = a.pout + (long long)sys * a.stride;
  const double2 ac = __ldg(&a.wtab[l]);
  const double sa2 = 2.0 * ac.y, ca2 = 2.0 * ac.x;
  const double2* twl = a.wtab + N + l;
  const int kq = qpos_inv<N>(j0 / 2 + g);               // the pair's true column pair
  const double2* dr = a.dtab + (long long)kq * N + l;
  double2* reg = reinterpret_cast<double2*>(tile) + CG::RBASE(g);
  __syncthreads();                                       // the barrier is initialised
  mbar_wait(&bar, 0);
  {
    constexpr bool PADC = (F::Q == 1);
    double2* ob = fdst::out_base<N>(reg, l);
    auto put = [&](int j, double a0, double a1, double b0, double b1) {
      ob[2 * j] = make_double2(a0, b0);
      ob[2 * j + 1] = make_double2(a1, b1);
      if (PADC && j == 0 && l > 0) ob[-1] = make_double2(a0, b0);   // pad copy (fdst::SmemLd)
    };
    // D'' of the column pair scales the forward transform's outputs in its post-processing
    fdst::pair_dst_ld<N, false, true, fdst::BlockSync<true, false>>(TileLd<N>(tile, g, l), reg, twl, l, sa2, ca2, put, nullptr,
                                            nullptr, dr);
    __syncwarp();
    // P (pair-interleaved): rows (2k, 2k+1), columns (2 kq, 2 kq + 1), k = C l + j
    if constexpr (CT::PSTORE) {
      // tile row j L + l, 16-byte chunks 2g and 2g + 1, XOR-swizzled with the row's low bits
      unsigned char* pt = tile + l * CT::PB;
      const int c0 = ((2 * g) ^ CT::pswz(l)) << 4, c1 = ((2 * g + 1) ^ CT::pswz(l)) << 4;
      fdst::pair_dst_ld<N, false, false, fdst::BlockSync<false, true>>(
          fdst::SmemLd<N, PADC>(reg, l), reg, twl, l, sa2, ca2,
          [&](int j, double a0, double a1, double b0, double b1) {
            *reinterpret_cast<double2*>(pt + j * (L * CT::PB) + c0) = make_double2(a0, a1);
            *reinterpret_cast<double2*>(pt + j * (L * CT::PB) + c1) = make_double2(b0, b1);
          });
      fence_async_proxy();
      __syncthreads();
      if (tid == 0) {
        tma_store_3d(&pmap, tile, 4 * qpos_inv<N>(j0 / 2), sys * L, 0);
        tma_store_commit_wait_read();
      }
    } else {
      double* pl = Ps + ((long long)(F::C * l) * N + 2 * kq) * 2;
      fdst::pair_dst_ld<N>(fdst::SmemLd<N, PADC>(reg, l), reg, twl, l, sa2, ca2,
                           [&](int j, double a0, double a1, double b0, double b1) {
        st256(pl + (long long)j * (2 * N), a0, a1, b0, b1);
      });
    }
  }
}

// Two-team column pass (N = 1024): one 256-thread block per SM runs two tiles, one per team
// of 4 warps, through the same phase sequence ONE PHASE APART (fdst::PhaseTick): while one
// team's warps move data through shared memory the other team's warps run their DFT on the
// FP64 pipes.  Warp w of either team sits on scheduler w % 4, so each scheduler always holds
// one warp of each kind.  Two independent 128-thread blocks per SM (k2d_colt) drift into
// lockstep instead, where both pipes idle in turn.
template <int N> struct ColT2 {
  using CT = ColT<N>;
  static constexpr int THREADS = 2 * ColG<N>::THREADS;
  static constexpr size_t TEAM = ((CT::SMEM - 1024) + 1023) / 1024 * 1024;   // per-team bytes
  static constexpr size_t SMEM = 1024 + 2 * TEAM;
  static_assert(CT::PSTORE && CT::PB == 128, "two-team column pass: N = 1024, 4-pair tiles");
};

template <int N>
__global__ void __launch_bounds__(ColT2<N>::THREADS, 1)
k2d_colt2(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap pmap, ColArgs a) {
  using F = fdst::FG<N>;
  using CG = ColG<N>;
  using CT = ColT<N>;
  using Sy = fdst::PhaseTick;
  constexpr int L = F::L, TC = CG::TC, TT = CG::THREADS;
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ __align__(8) unsigned long long bar[2];
  const int team = threadIdx.x / TT, tid = threadIdx.x % TT;
  unsigned char* tile = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u) + team * ColT2<N>::TEAM;
  const int g = tid / L, l = tid % L;
  const int sys = blockIdx.y;
  const int j0 = (blockIdx.x * 2 + team) * TC;
  if (tid == 0) {
    mbar_init(&bar[team], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_proxy();
    mbar_expect_tx(&bar[team], (unsigned)CT::TILE);
#pragma unroll
    for (int b = 0; b < CT::NBOX; ++b)
      tma_load_2d(tile + (size_t)b * CT::BR * CT::IB, &qmap, j0, sys * N + b * CT::BR, &bar[team]);
  }
  const double2 ac = __ldg(&a.wtab[l]);
  const double sa2 = 2.0 * ac.y, ca2 = 2.0 * ac.x;
  const double2* twl = a.wtab + N + l;
  const int kq = qpos_inv<N>(j0 / 2 + g);
  const double2* dr = a.dtab + (long long)kq * N + l;
  double2* reg = reinterpret_cast<double2*>(tile) + CG::RBASE(g);
  __syncthreads();                                       // both barriers are initialised
  if (team == 1) Sy::tick();                             // team 1 runs one phase behind team 0
  mbar_wait(&bar[team], 0);
  {
    double2* ob = fdst::out_base<N>(reg, l);
    auto put = [&](int j, double a0, double a1, double b0, double b1) {
      ob[2 * j] = make_double2(a0, b0);
      ob[2 * j + 1] = make_double2(a1, b1);
    };
    fdst::pair_dst_ld<N, false, true, Sy>(TileLd<N>(tile, g, l), reg, twl, l, sa2, ca2, put, nullptr,
                                          nullptr, dr);
    __syncwarp();
    unsigned char* pt = tile + l * 128;
    const int c0 = ((2 * g) ^ (l & 7)) << 4, c1 = ((2 * g + 1) ^ (l & 7)) << 4;
    fdst::pair_dst_ld<N, false, false, Sy>(
        fdst::SmemLd<N>(reg, l), reg, twl, l, sa2, ca2,
        [&](int j, double a0, double a1, double b0, double b1) {
          *reinterpret_cast<double2*>(pt + j * (L * 128) + c0) = make_double2(a0, a1);
          *reinterpret_cast<double2*>(pt + j * (L * 128) + c1) = make_double2(b0, b1);
        });
    fence_async_proxy();
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(TT) : "memory");   // the team's P tile is staged
    if (tid == 0) {
      tma_store_3d(&pmap, tile, 4 * qpos_inv<N>(j0 / 2), sys * L, 0);
      tma_store_commit_wait_read();
    }
  }
  if (team == 0) Sy::tick();                             // matches team 1's leading barrier
}

}  // namespace linb
