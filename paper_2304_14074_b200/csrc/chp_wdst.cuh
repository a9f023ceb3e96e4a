// Register-resident DST-I for pairs of real vectors: one lane group per pair.
//
// Unnormalised DST-I of length N-1 (N = 2^p, 8 <= N <= 1024) of two real
// vectors a, b via one complex FFT of length N (algebra in chp_dst.cuh):
//   y_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2,  z = y^a + i y^b,
//   Z = FFT_N(z),  R^a_k = (Z_k + conj Z_{N-k})/2,  R^b_k = (Z_k - conj Z_{N-k})/(2i),
//   X_{2k} = -Im R_k,  X_{2k+1} = sum_{l<=k} c_l  (c_0 = Re R_0 / 2, c_l = Re R_l).
//
// Four-step FFT, N = L x R: a group of L lanes (a full warp for N = 1024) with
// R complex values per lane in registers.
//   load + pre-processing (x_n and x_{N-n} both come from the caller's in())
//   stage 1: lane l: R-point DFT of z[l + L n2], twiddle W_N^{l k2} (smem table)
//   transpose through shared memory (XOR swizzle, conflict free)
//   stage 2: L-point DFT(s) for k2 = l + L t -> Z[k2 + R k1]
//   Z back to shared memory in natural order; post-processing on contiguous
//   chunks of k per lane: in-lane running sums + one warp scan of the chunk
//   totals (fixed order: results are bit-reproducible run to run).
#pragma once
#include "chp_common.cuh"

namespace wdst {

CHP_DEV constexpr double c64(int k) {
  constexpr double c[64] = {1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 2.0670321098263988e-43, -0.0980171403295606, -0.19509032201612828, -0.2902846772544624, -0.3826834323650898, -0.47139673682599764, -0.5555702330196022, -0.6343932841636455, -0.7071067811865476, -0.773010453362737, -0.8314696123025452, -0.881921264348355, -0.9238795325112867, -0.9569403357322088, -0.9807852804032304, -0.9951847266721969, -1.0, -0.9951847266721969, -0.9807852804032304, -0.9569403357322088, -0.9238795325112867, -0.881921264348355, -0.8314696123025452, -0.773010453362737, -0.7071067811865476, -0.6343932841636455, -0.5555702330196022, -0.47139673682599764, -0.3826834323650898, -0.2902846772544624, -0.19509032201612828, -0.0980171403295606, 2.2338764406549882e-41, 0.0980171403295606, 0.19509032201612828, 0.2902846772544624, 0.3826834323650898, 0.47139673682599764, 0.5555702330196022, 0.6343932841636455, 0.7071067811865476, 0.773010453362737, 0.8314696123025452, 0.881921264348355, 0.9238795325112867, 0.9569403357322088, 0.9807852804032304, 0.9951847266721969};
  constexpr double s[64] = {0.0, 0.0980171403295606, 0.19509032201612828, 0.2902846772544624, 0.3826834323650898, 0.47139673682599764, 0.5555702330196022, 0.6343932841636455, 0.7071067811865476, 0.773010453362737, 0.8314696123025452, 0.881921264348355, 0.9238795325112867, 0.9569403357322088, 0.9807852804032304, 0.9951847266721969, 1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 4.1340642196527976e-43, -0.0980171403295606, -0.19509032201612828, -0.2902846772544624, -0.3826834323650898, -0.47139673682599764, -0.5555702330196022, -0.6343932841636455, -0.7071067811865476, -0.773010453362737, -0.8314696123025452, -0.881921264348355, -0.9238795325112867, -0.9569403357322088, -0.9807852804032304, -0.9951847266721969, -1.0, -0.9951847266721969, -0.9807852804032304, -0.9569403357322088, -0.9238795325112867, -0.881921264348355, -0.8314696123025452, -0.773010453362737, -0.7071067811865476, -0.6343932841636455, -0.5555702330196022, -0.47139673682599764, -0.3826834323650898, -0.2902846772544624, -0.19509032201612828, -0.0980171403295606};
  return c[k & 63];
}
CHP_DEV constexpr double s64(int k) {
  constexpr double c[64] = {1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 2.0670321098263988e-43, -0.0980171403295606, -0.19509032201612828, -0.2902846772544624, -0.3826834323650898, -0.47139673682599764, -0.5555702330196022, -0.6343932841636455, -0.7071067811865476, -0.773010453362737, -0.8314696123025452, -0.881921264348355, -0.9238795325112867, -0.9569403357322088, -0.9807852804032304, -0.9951847266721969, -1.0, -0.9951847266721969, -0.9807852804032304, -0.9569403357322088, -0.9238795325112867, -0.881921264348355, -0.8314696123025452, -0.773010453362737, -0.7071067811865476, -0.6343932841636455, -0.5555702330196022, -0.47139673682599764, -0.3826834323650898, -0.2902846772544624, -0.19509032201612828, -0.0980171403295606, 2.2338764406549882e-41, 0.0980171403295606, 0.19509032201612828, 0.2902846772544624, 0.3826834323650898, 0.47139673682599764, 0.5555702330196022, 0.6343932841636455, 0.7071067811865476, 0.773010453362737, 0.8314696123025452, 0.881921264348355, 0.9238795325112867, 0.9569403357322088, 0.9807852804032304, 0.9951847266721969};
  constexpr double s[64] = {0.0, 0.0980171403295606, 0.19509032201612828, 0.2902846772544624, 0.3826834323650898, 0.47139673682599764, 0.5555702330196022, 0.6343932841636455, 0.7071067811865476, 0.773010453362737, 0.8314696123025452, 0.881921264348355, 0.9238795325112867, 0.9569403357322088, 0.9807852804032304, 0.9951847266721969, 1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898, 0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 4.1340642196527976e-43, -0.0980171403295606, -0.19509032201612828, -0.2902846772544624, -0.3826834323650898, -0.47139673682599764, -0.5555702330196022, -0.6343932841636455, -0.7071067811865476, -0.773010453362737, -0.8314696123025452, -0.881921264348355, -0.9238795325112867, -0.9569403357322088, -0.9807852804032304, -0.9951847266721969, -1.0, -0.9951847266721969, -0.9807852804032304, -0.9569403357322088, -0.9238795325112867, -0.881921264348355, -0.8314696123025452, -0.773010453362737, -0.7071067811865476, -0.6343932841636455, -0.5555702330196022, -0.47139673682599764, -0.3826834323650898, -0.2902846772544624, -0.19509032201612828, -0.0980171403295606};
  return s[k & 63];
}

template <int N> struct Geo;
template <> struct Geo<8>    { static constexpr int L = 2,  R = 4;  };
template <> struct Geo<16>   { static constexpr int L = 4,  R = 4;  };
template <> struct Geo<32>   { static constexpr int L = 4,  R = 8;  };
template <> struct Geo<64>   { static constexpr int L = 8,  R = 8;  };
template <> struct Geo<128>  { static constexpr int L = 8,  R = 16; };
template <> struct Geo<256>  { static constexpr int L = 16, R = 16; };
template <> struct Geo<512>  { static constexpr int L = 16, R = 32; };
#ifndef CHP_L1024
#define CHP_L1024 32
#endif
template <> struct Geo<1024> { static constexpr int L = CHP_L1024, R = 1024 / CHP_L1024; };  // 64: two warps per pair

CHP_DEV constexpr int brev(int k, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((k >> i) & 1) << (bits - 1 - i);
  return r;
}
CHP_DEV constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

CHP_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
CHP_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
CHP_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// d * W_64^idx, trivial cases folded (idx is a compile-time constant after unrolling)
CHP_DEV double2 tw64(double2 d, int idx) {
  idx &= 63;
  if (idx == 0) return d;
  if (idx == 16) return make_double2(d.y, -d.x);       // * (-i)
  if (idx == 32) return make_double2(-d.x, -d.y);
  if (idx == 48) return make_double2(-d.y, d.x);       // * (+i)
  const double c = c64(idx), s = -s64(idx);             // W = exp(-2 pi i idx/64)
  return make_double2(fma(d.x, c, -d.y * s), fma(d.x, s, d.y * c));
}

// In-register radix-2 DIF DFT of size R (R <= 32): X[k] ends in v[brev(k)].
template <int R>
CHP_DEV void dft(double2 (&v)[R]) {
#pragma unroll
  for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * span) {
#pragma unroll
      for (int j = 0; j < span; ++j) {
        const double2 u = v[b + j], w = v[b + j + span];
        v[b + j] = cadd(u, w);
        v[b + j + span] = tw64(csub(u, w), j * (32 / span));
      }
    }
  }
}

// Swizzle of the natural-order Z buffer (double2 units): chunk reads of stride
// C and consecutive writes are both bank-conflict free.
template <int N>
CHP_DEV int zsw(int k) {
  constexpr int C = N / 2 / Geo<N>::L;
  constexpr int CB = ilog2(C);
  return k ^ ((k >> CB) & 7);
}

// Swizzle of a shared-memory row of N doubles that is read by consecutive
// lanes and written in double2 chunks of stride 2C (keeps (2k, 2k+1) adjacent).
CHP_DEV int rsw(int e) { return e ^ (((e >> 5) & 15) << 1); }

// Twiddle table W_N^{l k2} laid out [k2][l] (R*L = N double2), built on the host.
// plus W_64^k (k < 64) at twt[N + k] for the 64-lane (N = 1024) second stage
template <int N>
CHP_DEV void load_twiddles(double2* twt, const double2* __restrict__ g) {
  for (int i = threadIdx.x; i < N + 64; i += blockDim.x) twt[i] = __ldg(&g[i]);
}

// named barrier of one 64-thread lane group (two warps)
CHP_DEV void group_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// synchronise one lane group (a warp or part of one; two warps when LG = 64)
template <int N, int LG = Geo<N>::L>
CHP_DEV void group_sync() {
  if constexpr (LG == 64) group_bar(1 + (int)(threadIdx.x / 64));
  else __syncwarp();
}

// N = 1024 with 64-lane groups: R = 16 complex per lane, three register stages
// (16-point, 4 x 4-point, 16-point) and two swizzled shared-memory transposes;
// half the registers per lane of a 32 x 32 split, so twice the warps per SM.
template <int N, class In, class Out>
CHP_DEV void pair_dst64(In in, Out out, double2* scr, const double2* twt, int l, double2 ac) {
  constexpr int L = 64, R = 16, C = N / 2 / L;
  static_assert(N == 1024, "pair_dst64 is the N = 1024 geometry");
  const int bar = 1 + (int)(threadIdx.x / L);
  double2 z[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    double a, am, b, bm;
    in(l + L * n2, a, am, b, bm);
    const double s = fma(ac.y, c64(n2 * (32 / R)), ac.x * s64(n2 * (32 / R)));
    const double sa = s * (a + am), da = 0.5 * (a - am);
    const double sb = s * (b + bm), db = 0.5 * (b - bm);
    z[n2] = make_double2(sa + da, sb + db);
  }
  dft<R>(z);
#pragma unroll
  for (int k2 = 1; k2 < R; ++k2) z[brev(k2, 4)] = cmul(z[brev(k2, 4)], twt[k2 * L + l]);
  group_bar(bar);
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) scr[k2 * L + (l ^ k2)] = z[brev(k2, 4)];
  group_bar(bar);
  // stage 2a: lane -> (k2 = l >> 2, la = 4 (l & 3) + t), 4-point DFTs over lb
  const int k2 = l >> 2, q = l & 3;
  double2 v[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
#pragma unroll
    for (int lb = 0; lb < 4; ++lb) v[t][lb] = scr[k2 * L + ((4 * q + t + 16 * lb) ^ k2)];
  }
  group_bar(bar);
  const double2* w64 = twt + N;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    dft<4>(v[t]);
#pragma unroll
    for (int k1a = 1; k1a < 4; ++k1a)
      v[t][brev(k1a, 2)] = cmul(v[t][brev(k1a, 2)], w64[((4 * q + t) * k1a) & 63]);
#pragma unroll
    for (int k1a = 0; k1a < 4; ++k1a)
      scr[k2 * L + ((4 * (4 * q + t) + k1a) ^ k2)] = v[t][brev(k1a, 2)];
  }
  group_bar(bar);
  // stage 2b: lane -> (k2 = l >> 2, k1a = l & 3), 16-point DFT over la
  const int k1a = l & 3;
  double2 w[16];
#pragma unroll
  for (int la = 0; la < 16; ++la) w[la] = scr[k2 * L + ((4 * la + k1a) ^ k2)];
  group_bar(bar);
  dft<16>(w);
#pragma unroll
  for (int k1b = 0; k1b < 16; ++k1b) scr[zsw<N>(k2 + 16 * k1a + 64 * k1b)] = w[brev(k1b, 4)];
  group_bar(bar);
  // post-processing on the chunk [l*C, l*C + C)
  double ea[C], eb[C], ca[C], cb[C];
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int k = l * C + j;
    const double2 X = scr[zsw<N>(k)];
    const double2 Y = scr[zsw<N>((N - k) & (N - 1))];
    ea[j] = 0.5 * (Y.y - X.y);
    eb[j] = 0.5 * (X.x - Y.x);
    double xa = 0.5 * (X.x + Y.x);
    double xb = 0.5 * (X.y + Y.y);
    if (j == 0 && l == 0) { xa *= 0.5; xb *= 0.5; ea[0] = 0.0; eb[0] = 0.0; }
    sa += xa;
    sb += xb;
    ca[j] = sa;
    cb[j] = sb;
  }
  // exclusive scan of the chunk totals over the 64 lanes (fixed order)
  double ia = sa, ib = sb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, ia, o);
    const double yb = __shfl_up_sync(0xffffffffu, ib, o);
    if ((l & 31) >= o) { ia += ya; ib += yb; }
  }
  group_bar(bar);                                    // scr reads done
  double* tot = reinterpret_cast<double*>(scr);
  if (l == 31) { tot[0] = ia; tot[1] = ib; }
  group_bar(bar);
  if (l >= 32) { ia += tot[0]; ib += tot[1]; }
  const double offa = ia - sa, offb = ib - sb;
  group_bar(bar);                                    // before out() may write scr
#pragma unroll
  for (int j = 0; j < C; ++j) out(l * C + j, ea[j], ca[j] + offa, eb[j], cb[j] + offb);
}

// Unnormalised DST-I of the pair (a, b).
//   in(n, a, am, b, bm): x_n and x_{N-n} of both vectors, n = l + L*n2
//                        (return zeros for n == 0);
//   out(k, A2k, A2k1, B2k, B2k1): for k in the lane's chunk [l*C, l*C + C),
//                        C = N/(2L), A_0 := 0;
//   scr: R*L double2 of group-private shared memory (free when out() runs;
//        in() must have consumed any data kept there before the transpose);
//   twt: block-shared twiddle table; ac = (cos, sin)(pi l / N).
//   LG: lanes per group -- Geo<N>::L, or 64 for the two-warp N = 1024 variant
//        (its own twiddle layout, see the host tables).
template <int N, int LG = Geo<N>::L, class In, class Out>
CHP_DEV void pair_dst(In in, Out out, double2* scr, const double2* twt, int l, double2 ac) {
  if constexpr (LG == 64) {
    pair_dst64<N>(in, out, scr, twt, l, ac);
    return;
  } else {
  constexpr int L = Geo<N>::L, R = Geo<N>::R, Q = R / L;
  constexpr int LB = ilog2(L), RB = ilog2(R);
  constexpr int C = N / 2 / L;
  double2 z[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    double a, am, b, bm;
    in(l + L * n2, a, am, b, bm);
    // sin(pi (l + L n2)/N) = sin(pi l/N) cos(pi n2/R) + cos(pi l/N) sin(pi n2/R)
    const double s = fma(ac.y, c64(n2 * (32 / R)), ac.x * s64(n2 * (32 / R)));
    const double sa = s * (a + am), da = 0.5 * (a - am);
    const double sb = s * (b + bm), db = 0.5 * (b - bm);
    z[n2] = make_double2(sa + da, sb + db);
  }
  dft<R>(z);
#pragma unroll
  for (int k2 = 1; k2 < R; ++k2) z[brev(k2, RB)] = cmul(z[brev(k2, RB)], twt[k2 * L + l]);
  __syncwarp();
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) scr[k2 * L + (l ^ (k2 & (L - 1)))] = z[brev(k2, RB)];
  __syncwarp();
  double2 v[Q][L];
#pragma unroll
  for (int t = 0; t < Q; ++t) {
#pragma unroll
    for (int n1 = 0; n1 < L; ++n1) v[t][n1] = scr[(l + L * t) * L + (n1 ^ l)];
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < Q; ++t) dft<L>(v[t]);
#pragma unroll
  for (int t = 0; t < Q; ++t) {
#pragma unroll
    for (int k1 = 0; k1 < L; ++k1) scr[zsw<N>(l + L * t + R * k1)] = v[t][brev(k1, LB)];
  }
  __syncwarp();
  // post-processing on the chunk [l*C, l*C + C)
  double ea[C], eb[C], ca[C], cb[C];
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int k = l * C + j;
    const double2 X = scr[zsw<N>(k)];
    const double2 Y = scr[zsw<N>((N - k) & (N - 1))];
    ea[j] = 0.5 * (Y.y - X.y);           // -Im R^a_k
    eb[j] = 0.5 * (X.x - Y.x);           // -Im R^b_k
    double xa = 0.5 * (X.x + Y.x);       //  Re R^a_k
    double xb = 0.5 * (X.y + Y.y);       //  Re R^b_k
    if (j == 0 && l == 0) { xa *= 0.5; xb *= 0.5; ea[0] = 0.0; eb[0] = 0.0; }
    sa += xa;
    sb += xb;
    ca[j] = sa;
    cb[j] = sb;
  }
  // exclusive scan of the chunk totals across the group (fixed order)
  double ia = sa, ib = sb;
#pragma unroll
  for (int o = 1; o < L; o <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, ia, o, L);
    const double yb = __shfl_up_sync(0xffffffffu, ib, o, L);
    if (l >= o) { ia += ya; ib += yb; }
  }
  const double offa = ia - sa, offb = ib - sb;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < C; ++j) out(l * C + j, ea[j], ca[j] + offa, eb[j], cb[j] + offb);
  }
}

// fast reciprocal: float seed + two Newton steps (relative error ~1e-16)
CHP_DEV double rcp(double x) {
  double y = (double)__frcp_rn((float)x);
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

}  // namespace wdst
