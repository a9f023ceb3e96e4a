// Neumann-Neumann fine step (Scheme.NN_LINEAR_A) on sm_100a -- the B200
// restatement of the reference's ddm.py (1D only, as the reference).
//
// One time step (ddm.py:268-340, _nn_solve) on a field of `nodes` grid points
// split into S subdomains of `step` cells sharing their end points:
//   * per subdomain, the Dirichlet solve of the mixed (u, v) system with zero
//     traces plus its response to the four local traces (ddm.py:147-203), and
//     the Neumann solve's interface values per unit load (ddm.py:205-256);
//   * the relaxed interface iteration on the traces g (u) and h (v)
//     (ddm.py:293-330), stopping once both cell-weighted L2 increments are
//     <= tol, or NNConvergenceError after max_iter sweeps (ddm.py:331-332);
//   * assembly of u^{n+1} = Dirichlet solution at the converged traces, with
//     the traces themselves at the interface nodes (ddm.py:334-340).
//
// Mapping: one warp segment of W = next_pow2(S) lanes per system, lane i =
// subdomain i; 32/W systems per warp.  The interface iteration exchanges the
// edge values and Neumann loads with the neighbouring subdomains by warp
// shuffles inside the segment -- no shared or global memory in the sweep loop.
//
// The reference factors each 2k x 2k mixed matrix by dense LAPACK LU.  Here
// the same matrix, ordered node by node as x_k = (u_k, v_k), is block
// tridiagonal with 2x2 blocks.  The interface iteration needs only the END
// values of the Dirichlet/Neumann solutions (edge responses), which a forward
// and a reverse block elimination deliver without storing anything; only the
// final assembly solve keeps G_k, z_k (6 doubles per node) in a per-lane
// global scratch column for its back substitution (x_k = z_k - G_k x_{k+1}).
// Same system, different rounding: parity against the reference is by
// tolerance (tests/test_gpu_nn.py; measured <= 2e-15).
#include <math.h>

#include "chp_common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRow = 6;   // assembly scratch doubles per node: G (4) + z (2)
constexpr int kQ = 4;     // register-queue depth of the field loads

struct NNConst {
  double dt, eps2, hh, hgrid, theta, tol;
  double au, av;    // regular couplings: u-row to v_{k+-1}, v-row to u_{k+-1}
  double bu, bv0;   // regular diagonal block [[1, bu], [bv0 - c2, 1]]
  double iu, iv0;   // Neumann interface diagonal [[0.5, iu], [iv0 - 0.5 c2, 0.5]]
  double cu, cv;    // Neumann interface couplings
  double rg, rh;    // Dirichlet trace loads: v-row (g), u-row (h)
  int nodes, step, S, W, max_iter, warm, steps, nsys;
};

struct B2 {  // [[a, b], [c, d]]
  double a, b, c, d;
};

CHP_DEV B2 inv2(const B2& m) {
  const double r = 1.0 / (m.a * m.d - m.b * m.c);
  return {m.d * r, -m.b * r, -m.c * r, m.a * r};
}

// Off-diagonal blocks are anti-diagonal: [[0, p], [q, 0]].
// D - A*G with A = [[0,p],[q,0]]
CHP_DEV B2 schur(const B2& D, double p, double q, const B2& G) {
  return {D.a - p * G.c, D.b - p * G.d, D.c - q * G.a, D.d - q * G.b};
}
// Dinv * [[0,p],[q,0]]
CHP_DEV B2 times_anti(const B2& Di, double p, double q) {
  return {Di.b * q, Di.a * p, Di.d * q, Di.c * p};
}

struct Scratch {
  double* base;
  size_t nl;   // lanes in the launch (column stride)
  size_t gl;   // this lane's column
  CHP_DEV double& at(int k, int f) const { return base[((size_t)k * kRow + f) * nl + gl]; }
};

// Block elimination of one subdomain system, nodes k = 0..K-1 (first_node +
// k), in direction kDir (+1: from k = 0, -1: from k = K-1), carrying NC
// right-hand-side columns; returns the solution at the LAST processed node for
// every column (x_{K-1} forward, x_0 reverse) -- no storage.  Row k:
//   A_k x_{k-1} + B_k x_k + C_k x_{k+1} = r_k,   A, C = [[0, p], [q, 0]].
// Processing order j: D_j = B - P G_{j-1}, G_j = D_j^-1 Nx, z_j = D_j^-1
// (r - P z_{j-1}), with P the coupling to the previously processed node and Nx
// the coupling to the next one.  `kNeu`: Neumann rows (ddm.py:218-236).
template <bool kNeu>
struct NodeRow {   // diagonal block and couplings of row k
  B2 D;
  double ap, aq, cp, cq;
};

template <bool kNeu>
CHP_DEV NodeRow<kNeu> node_row(const NNConst& c, double c2, int k, int K, bool lo_if,
                               bool hi_if) {
  NodeRow<kNeu> n;
  const bool iface = kNeu && ((k == 0 && lo_if) || (k == K - 1 && hi_if));
  n.D = iface ? B2{0.5, c.iu, c.iv0 - 0.5 * c2, 0.5} : B2{1.0, c.bu, c.bv0 - c2, 1.0};
  const bool a_if = kNeu && (k == K - 1 && hi_if);   // A_k of the right interface row
  const bool c_if = kNeu && (k == 0 && lo_if);       // C_k of the left interface row
  n.ap = a_if ? c.cu : c.au;
  n.aq = a_if ? c.cv : c.av;
  n.cp = c_if ? c.cu : c.au;
  n.cq = c_if ? c.cv : c.av;
  return n;
}

// One elimination step of a chain: D = B - P G, G = D^-1 Nx, z = D^-1 (r - P z).
template <int NC>
CHP_DEV void chain_step(bool first, B2 D, double pp, double pq, double np, double nq,
                        double (&r)[NC][2], B2& G, double (&x)[NC][2]) {
  if (!first) {
    D = schur(D, pp, pq, G);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      r[j][0] -= pp * x[j][1];
      r[j][1] -= pq * x[j][0];
    }
  }
  const B2 Di = inv2(D);
  G = times_anti(Di, np, nq);
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double z0 = Di.a * r[j][0] + Di.b * r[j][1];
    const double z1 = Di.c * r[j][0] + Di.d * r[j][1];
    x[j][0] = z0;
    x[j][1] = z1;
  }
}

// Block elimination of one subdomain system (nodes k = 0..K-1 = first_node +
// k) from BOTH ends at once, carrying NC right-hand-side columns: the forward
// chain (from k = 0) ends with x_{K-1}, the reverse chain (from k = K-1) with
// x_0 -- the only values the interface iteration needs, so nothing is stored;
// the two independent chains interleave for ILP.  Row k:
//   A_k x_{k-1} + B_k x_k + C_k x_{k+1} = r_k,   A, C = [[0, p], [q, 0]];
// the forward chain's coupling to the previous node is A_k (next: C_k), the
// reverse chain's C_k (next: A_k).  `kNeu`: Neumann rows (ddm.py:218-236).
// (Interleaving the Neumann and Dirichlet systems too -- four chains -- was
// measured slower: 198 registers, 2.33 vs 2.12 ms per config-2-shaped launch.)
template <int NC, bool kNeu, typename Rhs>
CHP_DEV void solve_ends(const NNConst& c, const double* u, int first_node, int K, bool lo_if,
                        bool hi_if, Rhs rhs, double (&xf)[NC][2], double (&xr)[NC][2]) {
  B2 Gf = {0, 0, 0, 0}, Gr = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < NC; ++j) xf[j][0] = xf[j][1] = xr[j][0] = xr[j][1] = 0.0;
  // field values enter a register queue kQ nodes ahead of their use, so the
  // loads overlap the dependent elimination chain instead of stalling it
  const double* uf0 = u + first_node - 1;        // node k -> uf0[k]
  double qf[kQ], qr[kQ];
#pragma unroll
  for (int t = 0; t < kQ; ++t) {
    qf[t] = t < K ? uf0[t] : 0.0;
    qr[t] = t < K ? uf0[K - 1 - t] : 0.0;
  }
  for (int s = 0; s < K; ++s) {
    const int kf = s, kr = K - 1 - s;
    const double uf = qf[0], ur = qr[0];
#pragma unroll
    for (int t = 0; t + 1 < kQ; ++t) {
      qf[t] = qf[t + 1];
      qr[t] = qr[t + 1];
    }
    qf[kQ - 1] = s + kQ < K ? uf0[s + kQ] : 0.0;
    qr[kQ - 1] = s + kQ < K ? uf0[K - 1 - s - kQ] : 0.0;
    const NodeRow<kNeu> nf = node_row<kNeu>(c, uf * uf, kf, K, lo_if, hi_if);
    const NodeRow<kNeu> nr = node_row<kNeu>(c, ur * ur, kr, K, lo_if, hi_if);
    double rf[NC][2], rr[NC][2];
    rhs(kf, uf, rf);
    rhs(kr, ur, rr);
    chain_step<NC>(s == 0, nf.D, nf.ap, nf.aq, nf.cp, nf.cq, rf, Gf, xf);
    chain_step<NC>(s == 0, nr.D, nr.cp, nr.cq, nr.ap, nr.aq, rr, Gr, xr);
  }
}

__global__ void __launch_bounds__(128) k_nn_propagate(
    NNConst c, const double* in, long long in_stride, double* out,
    long long out_stride, const int* __restrict__ sys_index, const double* traces_in,
    double* traces_out, SysInfo* info, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int W = c.W, S = c.S;
  const int i = lane & (W - 1);            // subdomain
  const int spw = 32 / W;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long s = warp * spw + lane / W;   // system within the launch
  const bool valid = s < c.nsys;
  const bool lane_on = valid && i < S;
  const int idx = valid ? (sys_index ? sys_index[s] : (int)s) : 0;
  const Scratch sc{scratch, (size_t)gridDim.x * blockDim.x,
                   (size_t)(blockIdx.x * blockDim.x + threadIdx.x)};
  const int step = c.step;
  const int a = i * step, b = (i + 1) * step;
  const bool lo_if = a > 0, hi_if = i < S - 1;
  const bool owns_if = lane_on && hi_if;   // lane i owns interface i (node b)

  SysInfo* si = valid ? info + idx : nullptr;
  bool live = valid && si->status == CHP_SYS_OK;
  double g = 0.0, h = 0.0;
  if (owns_if && traces_in) {
    g = traces_in[(size_t)idx * 2 * (S - 1) + i];
    h = traces_in[(size_t)idx * 2 * (S - 1) + (S - 1) + i];
  }
  long long sweeps_total = 0;
  int sweeps_max = 0;
  double res_max = 0.0;
  int steps_done = 0;

  for (int st = 0; st < c.steps; ++st) {
    const double* u = st == 0 ? in + (size_t)idx * in_stride : out + (size_t)idx * out_stride;
    double* o = out + (size_t)idx * out_stride;
    if (st > 0 && !c.warm) g = h = 0.0;

    // ---- Neumann interface responses (ddm.py:205-256) and Dirichlet edge
    // values + trace responses (ddm.py:147-203): only the end values of each
    // solve are needed, so each system is eliminated once from either end ----
    double ner[4][4] = {};   // rows (phi_L, phi_R, psi_L, psi_R), cols (L_u, L_v, R_u, R_v)
    double edge0[4] = {}, er[4][4] = {};  // rows (u_first, u_last, v_first, v_last)
    double unode = 0.0, c2node = 0.0;
    if (lane_on && live) {
      const int an = lo_if ? a : a + 1, bn = hi_if ? b : b - 1;
      const int Kn = bn - an + 1;
      auto neu_rhs = [&](int k, double, double (&r)[4][2]) {
        const bool L0 = k == 0 && lo_if, R1 = k == Kn - 1 && hi_if;
        r[0][0] = L0 ? 1.0 : 0.0; r[0][1] = 0.0;
        r[1][0] = 0.0;            r[1][1] = L0 ? 1.0 : 0.0;
        r[2][0] = R1 ? 1.0 : 0.0; r[2][1] = 0.0;
        r[3][0] = 0.0;            r[3][1] = R1 ? 1.0 : 0.0;
      };
      const int K = step - 1;
      auto dir_rhs = [&](int k, double un, double (&r)[5][2]) {
        const bool f = k == 0, l = k == K - 1;
        r[0][0] = un;             r[0][1] = -un;
        r[1][0] = 0.0;            r[1][1] = f ? c.rg : 0.0;   // g_left  (v-row)
        r[2][0] = f ? c.rh : 0.0; r[2][1] = 0.0;              // h_left  (u-row)
        r[3][0] = 0.0;            r[3][1] = l ? c.rg : 0.0;   // g_right (v-row)
        r[4][0] = l ? c.rh : 0.0; r[4][1] = 0.0;              // h_right (u-row)
      };
      double xf[4][2], xr[4][2];
      solve_ends<4, true>(c, u, an, Kn, lo_if, hi_if, neu_rhs, xf, xr);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ner[0][j] = xr[j][0]; ner[1][j] = xf[j][0];
        ner[2][j] = xr[j][1]; ner[3][j] = xf[j][1];
      }
      double yf[5][2], yr[5][2];
      solve_ends<5, false>(c, u, a + 1, K, false, false, dir_rhs, yf, yr);
      edge0[0] = yr[0][0]; edge0[1] = yf[0][0]; edge0[2] = yr[0][1]; edge0[3] = yf[0][1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        er[0][j] = yr[j + 1][0]; er[1][j] = yf[j + 1][0];
        er[2][j] = yr[j + 1][1]; er[3][j] = yf[j + 1][1];
      }
      if (hi_if) {
        unode = u[b - 1];
        c2node = unode * unode;
      }
    }
    __syncwarp();

    // ---- interface iteration (ddm.py:293-332) ----
    bool done = !live;
    int sweep = 0;
    double gi = INFINITY, hi = INFINITY;
    while (__any_sync(kFull, !done)) {
      if (!done) ++sweep;   // other segments of the warp may still be sweeping
      const double gL0 = __shfl_up_sync(kFull, g, 1, W), hL0 = __shfl_up_sync(kFull, h, 1, W);
      const double tr[4] = {i > 0 ? gL0 : 0.0, i > 0 ? hL0 : 0.0, hi_if ? g : 0.0,
                            hi_if ? h : 0.0};
      double e[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        e[r] = edge0[r] + (er[r][0] * tr[0] + er[r][1] * tr[1] + er[r][2] * tr[2] +
                           er[r][3] * tr[3]);
      const double uf_next = __shfl_down_sync(kFull, e[0], 1, W);
      const double vf_next = __shfl_down_sync(kFull, e[2], 1, W);
      double ju = 0.0, jv = 0.0;
      if (owns_if) {
        ju = g - c.dt * (e[3] + vf_next - 2.0 * h) / c.hh - unode;
        jv = c.eps2 * (e[1] + uf_next - 2.0 * g) / c.hh - c2node * g + h + unode;
      }
      const double juL = __shfl_up_sync(kFull, ju, 1, W), jvL = __shfl_up_sync(kFull, jv, 1, W);
      const double ld[4] = {i > 0 ? -juL : 0.0, i > 0 ? -jvL : 0.0, hi_if ? ju : 0.0,
                            hi_if ? jv : 0.0};
      double p[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        p[r] = ner[r][0] * ld[0] + ner[r][1] * ld[1] + ner[r][2] * ld[2] + ner[r][3] * ld[3];
      const double phiL_next = __shfl_down_sync(kFull, p[0], 1, W);
      const double psiL_next = __shfl_down_sync(kFull, p[2], 1, W);
      double dg = 0.0, dh = 0.0;
      if (owns_if && !done) {
        dg = c.theta * (p[1] - phiL_next);
        dh = c.theta * (p[3] - psiL_next);
        g -= dg;
        h -= dh;
      }
      double sg = dg * dg, sh = dh * dh;
      for (int off = W >> 1; off > 0; off >>= 1) {
        sg += __shfl_xor_sync(kFull, sg, off, W);
        sh += __shfl_xor_sync(kFull, sh, off, W);
      }
      if (!done) {
        gi = sqrt(c.hgrid * sg);
        hi = sqrt(c.hgrid * sh);
        if (gi <= c.tol && hi <= c.tol) {
          done = true;
        } else if (sweep >= c.max_iter) {
          done = true;
          live = false;
          if (i == 0) {
            sysinfo_fail(si, CHP_SYS_NN, c.max_iter, gi);
            si->newton_maxres = hi;   // h increment of the failed step (chp.h)
          }
        }
      }
    }
    __syncwarp();

    // ---- assembly (ddm.py:334-340) ----
    // left neighbour's traces (all lanes participate)
    const double gLa = __shfl_up_sync(kFull, g, 1, W), hLa = __shfl_up_sync(kFull, h, 1, W);
    if (lane_on && live) {
      const double tg = i > 0 ? gLa : 0.0, th = i > 0 ? hLa : 0.0;
      const double rgv = hi_if ? g : 0.0, rhv = hi_if ? h : 0.0;
      const int K = step - 1;
      bool fin = true;
      // Dirichlet solve at the converged traces (= dir_sol0 + dir_response @
      // traces): forward elimination storing G_k, z_k, then back substitution
      B2 G = {0, 0, 0, 0};
      double z0 = 0.0, z1 = 0.0;
      const double* ua = u + a;                 // node a+1+k -> ua[k]
      double q[kQ];
#pragma unroll
      for (int t = 0; t < kQ; ++t) q[t] = t < K ? ua[t] : 0.0;
      for (int k = 0; k < K; ++k) {
        const double un = q[0];
#pragma unroll
        for (int t = 0; t + 1 < kQ; ++t) q[t] = q[t + 1];
        q[kQ - 1] = k + kQ < K ? ua[k + kQ] : 0.0;
        const double c2 = un * un;
        B2 D = B2{1.0, c.bu, c.bv0 - c2, 1.0};
        double r0 = un + ((k == 0 ? th * c.rh : 0.0) + (k == K - 1 ? rhv * c.rh : 0.0));
        double r1 = -un + ((k == 0 ? tg * c.rg : 0.0) + (k == K - 1 ? rgv * c.rg : 0.0));
        if (k > 0) {
          D = schur(D, c.au, c.av, G);
          r0 -= c.au * z1;
          r1 -= c.av * z0;
        }
        const B2 Di = inv2(D);
        G = times_anti(Di, c.au, c.av);
        z0 = Di.a * r0 + Di.b * r1;
        z1 = Di.c * r0 + Di.d * r1;
        sc.at(k, 0) = G.a; sc.at(k, 1) = G.b; sc.at(k, 2) = G.c; sc.at(k, 3) = G.d;
        sc.at(k, 4) = z0; sc.at(k, 5) = z1;
      }
      double x0 = z0, x1 = z1;
      o[a + K - 1] = x0;
      fin &= isfinite(x0);
      // back substitution; node k-1's G, z are loaded while node k is solved
      double gz[6];
      if (K >= 2) {
#pragma unroll
        for (int f = 0; f < 6; ++f) gz[f] = sc.at(K - 2, f);
      }
      for (int k = K - 2; k >= 0; --k) {
        double cur[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) cur[f] = gz[f];
        if (k >= 1) {
#pragma unroll
          for (int f = 0; f < 6; ++f) gz[f] = sc.at(k - 1, f);
        }
        const double n0 = cur[4] - (cur[0] * x0 + cur[1] * x1);
        const double n1 = cur[5] - (cur[2] * x0 + cur[3] * x1);
        x0 = n0;
        x1 = n1;
        o[a + k] = x0;
        fin &= isfinite(x0);
      }
      if (hi_if) {
        o[b - 1] = g;
        fin &= isfinite(g);
      }
      if (!fin) {
        sysinfo_fail(si, CHP_SYS_NONFINITE, st + 1, 0.0);
      }
      if (i == 0) {
        sweeps_total += sweep;
        sweeps_max = max(sweeps_max, sweep);
        res_max = fmax(res_max, fmax(gi, hi));
        ++steps_done;
      }
    }
    __syncwarp();
    // a non-finite lane stops its whole system (segment-uniform)
    if (valid) {
      const unsigned seg = __ballot_sync(kFull, lane_on && si->status != CHP_SYS_OK);
      const unsigned mine = (W == 32 ? kFull : ((1u << W) - 1u)) << ((lane / W) * W);
      if (seg & mine) live = false;
    } else {
      __ballot_sync(kFull, false);
    }
  }
  if (lane_on && i < S - 1 && traces_out) {
    traces_out[(size_t)idx * 2 * (S - 1) + i] = g;
    traces_out[(size_t)idx * 2 * (S - 1) + (S - 1) + i] = h;
  }
  if (valid && i == 0 && steps_done > 0) {
    si->newton_steps += steps_done;
    si->newton_total += sweeps_total;
    si->newton_max = max(si->newton_max, sweeps_max);
    si->newton_maxres = fmax(si->newton_maxres, res_max);
  }
}

}  // namespace

size_t chp_nn_scratch_bytes(int step, int nsys, int S) {
  int W = 1;
  while (W < S) W <<= 1;
  const int spw = 32 / W;
  const long long warps = (nsys + spw - 1) / spw;
  const long long blocks = (warps + 3) / 4;
  return (size_t)(step + 1) * kRow * (size_t)(blocks * 128) * sizeof(double);
}

cudaError_t chp_nn_launch(const chp_grid& gr, const chp_nn_params& p, double dt, double eps2,
                          int steps, int nsys, const double* in, long long in_stride,
                          double* out, long long out_stride, const int* sys_index,
                          const double* traces_in, double* traces_out, chp_sys_info* info,
                          double* scratch, cudaStream_t st) {
  NNConst c;
  const double hh = p.h2;
  c.dt = dt;
  c.eps2 = eps2;
  c.hh = hh;
  c.hgrid = gr.h;
  c.theta = p.theta;
  c.tol = p.tol;
  c.au = -dt * (1.0 / hh);
  c.av = eps2 * (1.0 / hh);
  c.bu = -dt * (-2.0 / hh);
  c.bv0 = eps2 * (-2.0 / hh);
  c.iu = dt / hh;
  c.iv0 = -eps2 / hh;
  c.cu = -dt / hh;
  c.cv = eps2 / hh;
  c.rg = -eps2 / hh;
  c.rh = dt / hh;
  c.nodes = gr.nx;
  c.S = p.n_subdomains;
  c.step = (gr.nx - 1) / p.n_subdomains;
  int W = 1;
  while (W < c.S) W <<= 1;
  c.W = W;
  c.max_iter = p.max_iter;
  c.warm = p.warm_start;
  c.steps = steps;
  c.nsys = nsys;
  const int spw = 32 / W;
  const long long warps = (nsys + spw - 1) / spw;
  const long long blocks = (warps + 3) / 4;
  k_nn_propagate<<<(unsigned)blocks, 128, 0, st>>>(c, in, in_stride, out, out_stride, sys_index,
                                                   traces_in, traces_out,
                                                   reinterpret_cast<SysInfo*>(info), scratch);
  return cudaGetLastError();
}
