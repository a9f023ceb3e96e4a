// Shared-memory DST-I for pairs of real vectors (the 2D spectral solves).
//
// Unnormalised DST-I of length m = N-1 (N a power of two):
//   X_k = sum_{j=1}^{N-1} x_j sin(pi j k / N),   k = 1..N-1,
// computed for two vectors a, b at once with ONE complex FFT of length N:
//   y_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2     (x_0 = x_N = 0)
//   z   = y^a + i y^b,  Z = FFT_N(z)
//   R^a_k = (Z_k + conj Z_{N-k})/2,  R^b_k = (Z_k - conj Z_{N-k})/(2i)
//   X_{2k} = -Im R_k,  X_{2k+1} = X_{2k-1} + Re R_k,  X_1 = Re R_0 / 2.
// The odd outputs are a prefix sum, evaluated with a fixed-order blocked scan
// (deterministic: the same input bits always give the same output bits).
//
// Memory: a pair occupies 2N doubles of shared memory: A[0..N) then B[0..N)
// (index = math index; A[0] is ignored and written as 0).  The transform is
// in place: the same 2N doubles hold z as N double2 during the FFT.
//
// A "group" of T threads (T a multiple of 32, T <= N/4 or T == 32) works on
// one pair; groups synchronise with named barrier `bar_id`.
#pragma once
#include "chp_common.cuh"

namespace chpdst {

struct Tables {          // per-N device tables (built once per context)
  const double2* tw;     // tw[k] = exp(-2 pi i k / N), k < N
  const double* sj;      // sj[j] = sin(pi j / N), j <= N
};

CHP_DEV void group_sync(int bar_id, int T) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(T) : "memory");
}

CHP_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
CHP_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
CHP_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i
CHP_DEV double2 cmi(double2 a) { return make_double2(a.y, -a.x); }

// In-place forward FFT of Z[N] (Stockham radix-4, radix-2 tail), group of T.
template <int N, int T>
CHP_DEV void fft_inplace(double2* Z, const double2* __restrict__ tw, int t, int bar) {
  constexpr int Q = N / 4;                       // radix-4 butterflies per pass
  constexpr int BPT = (Q + T - 1) / T;           // butterflies per thread
  int Ns = 1;
#pragma unroll 1
  for (; Ns * 4 <= N; Ns *= 4) {
    double2 v[BPT][4];
#pragma unroll
    for (int u = 0; u < BPT; ++u) {
      const int j = t + u * T;
      if (j < Q) {
        const int k = j % Ns;
        const int tstep = (N / (Ns * 4)) * k;    // twiddle index step
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double2 x = Z[j + r * Q];
          if (r) x = cmul(x, __ldg(&tw[(r * tstep) & (N - 1)]));
          v[u][r] = x;
        }
      }
    }
    group_sync(bar, T);
#pragma unroll
    for (int u = 0; u < BPT; ++u) {
      const int j = t + u * T;
      if (j < Q) {
        const double2 t0 = cadd(v[u][0], v[u][2]);
        const double2 t1 = csub(v[u][0], v[u][2]);
        const double2 t2 = cadd(v[u][1], v[u][3]);
        const double2 t3 = cmi(csub(v[u][1], v[u][3]));
        const int k = j % Ns;
        const int d = (j / Ns) * Ns * 4 + k;
        Z[d] = cadd(t0, t2);
        Z[d + Ns] = cadd(t1, t3);
        Z[d + 2 * Ns] = csub(t0, t2);
        Z[d + 3 * Ns] = csub(t1, t3);
      }
    }
    group_sync(bar, T);
  }
  if (Ns < N) {  // one radix-2 pass (N = 2 * 4^p)
    constexpr int H = N / 2;
    constexpr int BPT2 = (H + T - 1) / T;
    double2 v[BPT2][2];
#pragma unroll
    for (int u = 0; u < BPT2; ++u) {
      const int j = t + u * T;
      if (j < H) {
        const int k = j % Ns;
        v[u][0] = Z[j];
        v[u][1] = cmul(Z[j + H], __ldg(&tw[(N / (Ns * 2)) * k]));
      }
    }
    group_sync(bar, T);
#pragma unroll
    for (int u = 0; u < BPT2; ++u) {
      const int j = t + u * T;
      if (j < H) {
        const int k = j % Ns;
        const int d = (j / Ns) * Ns * 2 + k;
        Z[d] = cadd(v[u][0], v[u][1]);
        Z[d + Ns] = csub(v[u][0], v[u][1]);
      }
    }
    group_sync(bar, T);
  }
}

// Fixed-order exclusive scan of one double per thread across a group of T
// threads (T multiple of 32).  `ws` is scratch of T/32 doubles for the group.
template <int T>
CHP_DEV double group_exclusive_scan(double v, double* ws, int t, int bar) {
  const int lane = t & 31, w = t >> 5;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (T > 32) {
    if (lane == 31) ws[w] = incl;
    group_sync(bar, T);
    double off = 0.0;
    for (int q = 0; q < w; ++q) off += ws[q];
    group_sync(bar, T);
    return off + incl - v;
  }
  return incl - v;
}

// Unnormalised DST-I of the pair stored at P (2N doubles), in place.
// Values are scaled by `scale` on output.  `ws`: T/32 doubles scratch.
template <int N, int T>
CHP_DEV void dst_pair(double* P, const Tables& tb, double scale, double* ws, int t, int bar) {
  double* A = P;
  double* B = P + N;
  double2* Z = reinterpret_cast<double2*>(P);
  // --- pre-processing: (j, N-j) pairs, j = 1..N/2
  constexpr int H = N / 2;
  constexpr int PPT = (H + T - 1) / T;
  double2 zj[PPT], zn[PPT];
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const int j = 1 + t + u * T;
    if (j <= H) {
      const double s = __ldg(&tb.sj[j]);
      const double a1 = A[j], a2 = A[N - j], b1 = B[j], b2 = B[N - j];
      const double sa = s * (a1 + a2), da = 0.5 * (a1 - a2);
      const double sb = s * (b1 + b2), db = 0.5 * (b1 - b2);
      zj[u] = make_double2(sa + da, sb + db);
      zn[u] = make_double2(sa - da, sb - db);
    }
  }
  group_sync(bar, T);
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const int j = 1 + t + u * T;
    if (j <= H) {
      Z[j] = zj[u];
      if (j != H) Z[N - j] = zn[u];
    }
  }
  if (t == 0) Z[0] = make_double2(0.0, 0.0);
  group_sync(bar, T);
  fft_inplace<N, T>(Z, tb.tw, t, bar);
  // --- post-processing: thread owns k in [t*C, (t+1)*C), C = H / T (>= 1)
  constexpr int C = (H >= T) ? H / T : 1;
  const bool owner = (t * C) < H;
  double ea[C], eb[C], ca[C], cb[C];
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int u = 0; u < C; ++u) {
    const int k = t * C + u;
    ea[u] = eb[u] = ca[u] = cb[u] = 0.0;
    if (owner) {
      const double2 X = Z[k];
      const double2 Y = Z[(N - k) & (N - 1)];
      ea[u] = 0.5 * (Y.y - X.y);             // -Im R^a_k
      eb[u] = 0.5 * (X.x - Y.x);             // -Im R^b_k
      ca[u] = 0.5 * (X.x + Y.x);             //  Re R^a_k
      cb[u] = 0.5 * (X.y + Y.y);             //  Re R^b_k
      if (k == 0) { ca[u] *= 0.5; cb[u] *= 0.5; }
      sa += ca[u];
      sb += cb[u];
      ca[u] = sa;   // local inclusive prefix
      cb[u] = sb;
    }
  }
  const double offa = group_exclusive_scan<T>(owner ? sa : 0.0, ws, t, bar);
  const double offb = group_exclusive_scan<T>(owner ? sb : 0.0, ws, t, bar);
  group_sync(bar, T);   // all reads of Z done before overwriting
  if (owner) {
#pragma unroll
    for (int u = 0; u < C; ++u) {
      const int k = t * C + u;
      if (k > 0) {
        A[2 * k] = scale * ea[u];
        B[2 * k] = scale * eb[u];
      }
      A[2 * k + 1] = scale * (offa + ca[u]);
      B[2 * k + 1] = scale * (offb + cb[u]);
    }
  }
  if (t == 0) { A[0] = 0.0; B[0] = 0.0; }
  group_sync(bar, T);
}

}  // namespace chpdst
