// Pair DST-I with compile-time shared-memory addressing (LINEAR_B fine passes).
//
// Same algebra as chp_wdst.cuh (one complex FFT of length N for two real
// DST-I of length N-1, four-step N = L x R, one lane group of L lanes per
// pair), re-laid out so that every shared-memory access of the transform is
// a per-lane base register plus a compile-time immediate and is bank-conflict
// free without XOR swizzles:
//
//   pair layout  (input/output of the transform, double2 = (a_n, b_n)):
//                p2(n) = n + floor(n / R)          (one pad slot per R values)
//   transpose    T[k2][n1] at k2 (L+1) + n1
//   Z buffer     zaddr(k) = k + floor(k / C),  C = N / (2L); Z_0 also at zaddr(N)
//
// All three live in the same group region of RS double2.  The transform is
// scaled: it returns 4 T x (T the unnormalised DST-I), the factor 2 of the
// pre-processing and of the post-processing folded into the callers' tables,
// which saves the 1/2 multiplies:
//   z_n  = (2 s_n + 1) v_n + (2 s_n - 1) v_{N-n},   s_n = sin(pi n / N)
//   Z    = FFT_N(z)
//   out: X_{2k} = (Y.y - X.y, X.x - Y.x),  c_k = (X.x + Y.x, X.y + Y.y) (c_0 halved),
//        X_{2k+1} = sum_{l <= k} c_l            (X = Z_k, Y = Z_{N-k})
// The running sums are in-lane over a contiguous chunk of C outputs plus one
// fixed-order group scan: results are bitwise reproducible run to run.
#pragma once
#include "chp_common.cuh"
#include "chp_wdst.cuh"

#ifndef CHP_TW_POW
#define CHP_TW_POW 1
#endif
#ifndef CHP_PAIR_ATTR
#define CHP_PAIR_ATTR CHP_DEV
#endif

namespace fdst {

using wdst::brev;
using wdst::ilog2;

CHP_DEV constexpr int cmax(int a, int b) { return a > b ? a : b; }

// cos / sin (pi k / 32), k = 0..31 (cos(pi/2) = 0 exactly)
CHP_DEV constexpr double cpi32(int k) {
  constexpr double c[32] = {1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 0.0, -0.0980171403295606, -0.19509032201612828, -0.2902846772544624, -0.3826834323650898, -0.47139673682599764, -0.5555702330196022, -0.6343932841636455, -0.7071067811865476, -0.773010453362737, -0.8314696123025452, -0.881921264348355, -0.9238795325112867, -0.9569403357322088, -0.9807852804032304, -0.9951847266721969};
  return c[k & 31];
}
CHP_DEV constexpr double spi32(int k) {
  constexpr double s[32] = {0.0, 0.0980171403295606, 0.19509032201612828, 0.2902846772544624, 0.3826834323650898, 0.47139673682599764, 0.5555702330196022, 0.6343932841636455, 0.7071067811865476, 0.773010453362737, 0.8314696123025452, 0.881921264348355, 0.9238795325112867, 0.9569403357322088, 0.9807852804032304, 0.9951847266721969, 1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606};
  return s[k & 31];
}

template <int N> struct FG {
  static constexpr int L = wdst::Geo<N>::L, R = wdst::Geo<N>::R;
  static constexpr int Q = R / L;                 // stage-2 DFTs per lane (1 or 2)
  static constexpr int C = N / (2 * L);           // outputs k per lane in the post-processing
  static constexpr int LB = ilog2(L), RB = ilog2(R);
  static constexpr int P2N = N + N / R;           // p2(N)
  static constexpr int ZN = N + 2 * L;            // zaddr(N)
  static constexpr int RS = cmax(cmax(P2N + 1, ZN + 1), R * (L + 1));   // region (double2)
  static_assert(Q == 1 || Q == 2, "geometry");
};

template <int N> CHP_DEV constexpr int p2(int n) { return n + n / FG<N>::R; }

// Pair DST-I of the pair vector read through `ld`.  reg: the group's scratch region (RS
// double2; the input may live there).
// twl = twiddle table + l (W_N^{l k2} at twl[k2 L]); sa2 / ca2 = 2 sin / 2 cos (pi l / N).
// out(j, A2k, A2k1, B2k, B2k1) for k = C l + j (j compile-time after unrolling);
// out runs after the group has finished reading reg (it may write there).
// dsc (optional): per-row diagonal scale applied to the input (a column pair's
// spectral divisors, D[n] = (d_a(n), d_b(n)), n = 0..N), read coalesced:
// dsc points at D + l, dsm at D + N - l.
// dpo (optional, PS = true): per-output scale, chunk layout: dpo points at
// T + l, and T[(2j + h) L + l] scales output row 2(C l + j) + h (coalesced; each
// value read once; the loads are issued after the second DFT so their latency
// overlaps the post-processing).
// Input loaders of the pre-processing: v(n2) = pair value at n = l + L n2, w(n2) = its
// mirror at N - n.  SmemLd: a group-private pair region in p2 layout; other loaders
// (chp_linb.cuh TileLd: the column pass's TMA tile) only change the addressing.
// PADCOPY (Q == 1 geometries): the writer of the region also stored every element n = R q
// (q >= 1) into the pad slot in front of it, p2(n) - 1.  Lane 0's mirror values are exactly
// those elements; reading the copies keeps the 32 lanes of a mirror load on 32 consecutive
// slots (4 wavefronts) where lane 0 would otherwise sit one slot off and cost a fifth.
template <int N, bool PADCOPY = false> struct SmemLd {
  const double2 *sd, *sm0, *sm1;
  static_assert(!PADCOPY || FG<N>::Q == 1, "pad copies: one DFT per lane geometries");
  CHP_DEV SmemLd(const double2* src, int l)
      : sd(src + l), sm0(src + p2<N>(N - l) - ((PADCOPY && l == 0) ? 1 : 0)),
        // Q == 2: lane 0's mirror offsets differ by one for odd n2 (see header)
        sm1((FG<N>::Q == 2 && l == 0) ? src + p2<N>(N - l) - 1 : src + p2<N>(N - l)) {}
  CHP_DEV double2 v(int n2) const { return sd[FG<N>::L * n2 + n2 / FG<N>::Q]; }
  CHP_DEV double2 w(int n2) const {
    return ((n2 & 1) ? sm1 : sm0)[p2<N>(N - 1 - FG<N>::L * n2) - p2<N>(N - 1)];
  }
};

// Synchronisation policy of the transform's five phase boundaries.  The phases alternate
// between shared-memory traffic (L) and FP64 arithmetic (F):
//   P0 input loads + pre-processing (L) | loaded()      | P1 first DFT + twiddles (F) |
//   inputs_done() | P2 transpose (L) | transposed() | P3 second DFT (F) | dft2_done() |
//   P4 Z staging + post-processing + scan (L) | z_read() | P5 out() callbacks (L)
// WarpSync: the group's data is private, only the warp-level barriers the reuse of reg needs.
struct WarpSync {
  CHP_DEV static void loaded() {}
  CHP_DEV static void inputs_done() { __syncwarp(); }   // input reads done before reg is written
  CHP_DEV static void transposed() { __syncwarp(); }    // transposed reads done before Z is written
  CHP_DEV static void dft2_done() {}
  CHP_DEV static void z_read() { __syncwarp(); }        // Z reads done before out() writes reg
};
// BlockIn / BlockOut / BlockInOut: the input is shared by the whole block and reg overlays it
// (column pass tile) and/or out() writes memory other groups' regions overlay (P tile).
template <bool IN, bool OUT> struct BlockSync : WarpSync {
  CHP_DEV static void inputs_done() { if constexpr (IN) __syncthreads(); else __syncwarp(); }
  CHP_DEV static void z_read() { if constexpr (OUT) __syncthreads(); else __syncwarp(); }
};
// PhaseTick: every boundary is a block-wide barrier.  Two teams of warps that run the same
// transform sequence one phase apart (one team executes one extra barrier first) then always
// pair one team's L phase with the other's F phase: the shared-memory pipe and the FP64
// pipes work at the same time instead of in lockstep.
struct PhaseTick {
  CHP_DEV static void tick() { asm volatile("bar.sync 0;" ::: "memory"); }
  CHP_DEV static void loaded() { tick(); }
  CHP_DEV static void inputs_done() { tick(); }
  CHP_DEV static void transposed() { tick(); }
  CHP_DEV static void dft2_done() { tick(); }
  CHP_DEV static void z_read() { tick(); }
};

// DS: 0 no input scale; 1 scale table in global memory (read with ld.global.cg); 2 scale
// table anywhere (plain loads: a copy staged in shared memory).
template <int N, int DS = 0, bool PS = false, class Sy = WarpSync, class Ld, class Out>
CHP_PAIR_ATTR void pair_dst_ld(const Ld ld, double2* reg, const double2* __restrict__ twl, int l,
                      double sa2, double ca2, Out out,
                      const double2* __restrict__ dsc = nullptr,
                      const double2* __restrict__ dsm = nullptr,
                      const double2* __restrict__ dpo = nullptr) {
  using G = FG<N>;
  constexpr int L = G::L, R = G::R, Q = G::Q, C = G::C, LB = G::LB, RB = G::RB;
  // Global loads (divisors, twiddles) must not be hoisted across the
  // preceding code: dozens of independent loads in flight would push the
  // kernel past its register budget.  Laundering the pointers through an empty
  // asm with a memory clobber pins them in program order.
  if constexpr (DS) {
    asm volatile("" : "+l"(dsc), "+l"(dsm)::"memory");
  }
  double2 z[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    double2 v = ld.v(n2);
    double2 w = ld.w(n2);
    if constexpr (DS) {
      const double2 dv = (DS == 2) ? dsc[L * n2] : __ldcg(dsc + L * n2);
      const double2 dw = (DS == 2) ? dsm[-L * n2] : __ldcg(dsm - L * n2);
      v = make_double2(v.x * dv.x, v.y * dv.y);
      w = make_double2(w.x * dw.x, w.y * dw.y);
    }
    const double cc = cpi32(n2 * (32 / R)), ss = spi32(n2 * (32 / R));
    // sp = 2 sin(pi (l + L n2) / N) + 1 ; sm = sp - 2
    double sp;
    if (cc == 0.0) sp = fma(ca2, ss, 1.0);
    else if (ss == 0.0) sp = fma(sa2, cc, 1.0);
    else sp = fma(sa2, cc, fma(ca2, ss, 1.0));
    const double smn = sp - 2.0;
    z[n2] = make_double2(fma(sp, v.x, smn * w.x), fma(sp, v.y, smn * w.y));
  }
  if (l == 0) z[0] = make_double2(0.0, 0.0);      // x_0 = x_N = 0 (pad slots may hold anything)
  Sy::loaded();
  wdst::dft<R>(z);
  asm volatile("" : "+l"(twl)::"memory");
#if CHP_TW_POW
  // W^{l k2} from the table entries at powers of two and at most popcount(k2) - 1
  // products (<= 4 roundings): 5 loads instead of R - 1 through L1
  double2 tw[R];
#pragma unroll
  for (int k2 = 1; k2 < R; ++k2) {
    const int hb = k2 >= 16 ? 16 : (k2 >= 8 ? 8 : (k2 >= 4 ? 4 : (k2 >= 2 ? 2 : 1)));
    tw[k2] = (hb == k2) ? __ldg(&twl[k2 * L]) : wdst::cmul(tw[hb], tw[k2 - hb]);
  }
#pragma unroll
  for (int k2 = 1; k2 < R; ++k2) z[brev(k2, RB)] = wdst::cmul(z[brev(k2, RB)], tw[k2]);
#else
#pragma unroll
  for (int k2 = 1; k2 < R; ++k2) z[brev(k2, RB)] = wdst::cmul(z[brev(k2, RB)], __ldg(&twl[k2 * L]));
#endif
  Sy::inputs_done();
  double2* tp = reg + l;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) tp[k2 * (L + 1)] = z[brev(k2, RB)];
  __syncwarp();
  double2 v[Q][L];
  const double2* tr = reg + l * (L + 1);
#pragma unroll
  for (int t = 0; t < Q; ++t) {
#pragma unroll
    for (int n1 = 0; n1 < L; ++n1) v[t][n1] = tr[t * L * (L + 1) + n1];
  }
  Sy::transposed();
#pragma unroll
  for (int t = 0; t < Q; ++t) wdst::dft<L>(v[t]);
  Sy::dft2_done();
  // Z[k2 + R k1], k2 = l + L t  ->  zaddr = zb + L t + (R + 2) k1 (+ t when Q == 2)
  double2* zw = reg + l + ((Q == 1) ? l / C : 0);
#pragma unroll
  for (int t = 0; t < Q; ++t) {
#pragma unroll
    for (int k1 = 0; k1 < L; ++k1) zw[L * t + (R + 2) * k1 + ((Q == 2) ? t : 0)] = v[t][brev(k1, LB)];
  }
  if (l == 0) reg[G::ZN] = v[0][0];               // Z_0 again at zaddr(N)
  double2 dd[PS ? 2 * C : 1];
  if constexpr (PS) {
    asm volatile("" : "+l"(dpo)::"memory");
#pragma unroll
    for (int r = 0; r < 2 * C; ++r) dd[r] = __ldcg(dpo + r * L);
  }
  __syncwarp();
  const double2* xr = reg + (C + 1) * l;
  const double2* yr = reg + (N + 2 * L - 1 - (C + 1) * l);
  const double h0 = (l == 0) ? 0.5 : 1.0;
  double ea[C], eb[C], ca[C], cb[C];
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const double2 X = xr[j];
    const double2 Y = yr[(j == 0) ? 1 : -j];
    ea[j] = Y.y - X.y;
    eb[j] = X.x - Y.x;
    double xa = X.x + Y.x, xb = X.y + Y.y;
    if (j == 0) { xa *= h0; xb *= h0; }
    sa += xa;
    sb += xb;
    ca[j] = sa;
    cb[j] = sb;
  }
  double ia = sa, ib = sb;
#pragma unroll
  for (int o = 1; o < L; o <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, ia, o, L);
    const double yb = __shfl_up_sync(0xffffffffu, ib, o, L);
    if (l >= o) { ia += ya; ib += yb; }
  }
  const double offa = ia - sa, offb = ib - sb;
  Sy::z_read();
#pragma unroll
  for (int j = 0; j < C; ++j) {
    if constexpr (PS)
      out(j, ea[j] * dd[2 * j].x, (ca[j] + offa) * dd[2 * j + 1].x, eb[j] * dd[2 * j].y,
          (cb[j] + offb) * dd[2 * j + 1].y);
    else
      out(j, ea[j], ca[j] + offa, eb[j], cb[j] + offb);
  }
}

// Pair DST-I of the pair vector held in `src` (p2 layout, group-private, may alias `reg`).
template <int N, int DS = 0, bool PS = false, class Out>
CHP_PAIR_ATTR void pair_dst(const double2* src, double2* reg, const double2* __restrict__ twl, int l,
                      double sa2, double ca2, Out out,
                      const double2* __restrict__ dsc = nullptr,
                      const double2* __restrict__ dsm = nullptr,
                      const double2* __restrict__ dpo = nullptr) {
  pair_dst_ld<N, DS, PS, WarpSync>(SmemLd<N>(src, l), reg, twl, l, sa2, ca2, out, dsc, dsm, dpo);
}

// store the transform output into a pair region in p2 layout (k = C l + j):
// p2(2k) = (2C + 1) l + 2j, p2(2k + 1) = p2(2k) + 1
template <int N>
CHP_DEV double2* out_base(double2* reg, int l) { return reg + (2 * FG<N>::C + 1) * l; }

}  // namespace fdst
