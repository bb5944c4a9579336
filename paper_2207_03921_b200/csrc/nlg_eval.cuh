// nlg_eval.cuh -- per element-pair integrals on the device (FP64, CUDA cores).
//
// One ordered visit (k, l) of root k produces the reference's B block of
// _engine._visit_pair (:374-425): rows on k's local hats, column half 0 on
// k's hats ("kk") and half 1 on l's hats ("kl"), from an outer-on-k sweep
// (mode 0) and an outer-on-l sweep (mode 1); an identical pair runs mode 2
// (_engine._sweep :46-185, _pyengine._sweep :48-152 for P != Q).
//
// Two device paths compute it:
//  * full pairs (dist + r_k + r_l <= delta, no truncation): the reference
//    integrates the same 7x7 point pairs (x_p on k, y_q on l) in both
//    sweeps, so one 7x7 matrix of kernel values gives the whole block:
//        kk[a,b] = 2 c sum_p w_p H_pa H_pb sum_q w_q P_pq
//        kl[a,b] = -2 c sum_{p,q} w_p w_q Q_pq H_pa H_qb,   c = 2A_k 2A_l
//    (P = kernel(x_p, y_q), Q = kernel(y_q, x_p)); half the kernel
//    evaluations of the reference and ~1/8 of its flops;
//  * clipped pairs: the reference's two truncated sweeps, with the clip /
//    fan / drop predicates in exact reference arithmetic (nlg_geom.cuh)
//    and FMA-contracted accumulation.
#pragma once
#include <cstdint>

#include "nlg_geom.cuh"
#include "nlg_math.cuh"

namespace nlg {

struct Rule7 {
  double op[7][2], ow[7], oh[7][3], ip[7][2], iw[7];
  double wh[7][3];   // w_p * H_pa
  double whh[7][9];  // w_p * H_pa * H_pb
  double iws;        // sum of the inner weights
};

struct Params {
  // mesh (device)
  const double2* __restrict__ vtx;
  const int4* __restrict__ elem;  // x, y, z vertex ids; w = label | outer << 4
  const int4* __restrict__ dofs;  // x, y, z scalar dof bases
  const double2* __restrict__ ctr;
  const double* __restrict__ rad;
  int K, V;
  int nc, kid, ball, path, sym, is_dg;
  double s, kexp, cst, delta, prer, rskip2, drop2, kp0, kp1;
  long long J, row_lo, row_hi;
  int narrow;  // COO keys of this batch are written as 32-bit (rows x J < 2^32)
  // full pairs of the constant / affine kernels (kid 2, 3 on the standard
  // path) factor into per-element terms (ftab): merge stage R forms their
  // blocks, no per-record storage
  int analytic;
  const double4* __restrict__ ftab;  // [K] (A2 psi_0, A2 psi_1, A2 psi_2, A2)
  int dbg;  // NLG_DEBUG bit mask (experiments only; 0 in production)
  // label-dependent kernels (KernelSpec.value's label_x, label_y arguments,
  // kernels.py:21-35): value = lab[label_x][label_y] x the built-in's value,
  // with a symmetric table -- so both visits of a pair, and its P and Q
  // terms, carry the same factor and a record is scaled once when emitted
  int has_lab;
  double lab[9];
};

// label factor of the pair of elements with records' w fields wk, wl
__device__ __forceinline__ double lab_scale(const Params& P, int wk, int wl) {
  return P.has_lab ? P.lab[(wk & 15) * 3 + (wl & 15)] : 1.0;
}

// the 7-point rule and its weighted hat products (identical for every plan:
// QuadratureConfig only accepts "7point", quadrature.py:20)
__constant__ Rule7 c_rule;
__constant__ PowTab c_powtab;  // pow_tab tables (nlg_math.cuh)

template <int KID> struct KTraits {
  static constexpr int NC = KID == 1 ? 2 : 1;
  static constexpr bool SYM = KID != 3;
  static constexpr int NC2 = NC * NC;
  static constexpr int E = 9 * NC2;  // entries of one 3nc x 3nc block
};

// kernel matrix at offset d = x - y (r2 = |d|^2): _engine._kernel_mat :30-43;
// id 3 returns P = value(x, y) and Q = value(y, x) (_pyengine._pq :38-45).
// tab: pow tables in shared memory (pow_tab) for the fractional kernel, or
// nullptr for the polynomial fast_pow_pos
template <int KID, bool CBANK = true, bool TAB = false>
__device__ __forceinline__ void kval(const Params& P, double x0, double y0, double d0, double d1,
                                     double r2, double* p, double* q, const PowTab* tab = nullptr) {
  if constexpr (KID == 0) {
    if constexpr (TAB)
      p[0] = P.cst * pow_tab(r2, P.kexp, tab->rc, tab->lc, tab->e2);
    else
      p[0] = P.cst * fast_pow_pos<CBANK>(r2, P.kexp);
  } else if constexpr (KID == 1) {
    const double f = P.cst / (r2 * sqrt(r2));
    const double v01 = f * d0 * d1;
    p[0] = f * d0 * d0;
    p[1] = v01;
    p[2] = v01;
    p[3] = f * d1 * d1;
  } else if constexpr (KID == 2) {
    p[0] = P.cst;
  } else {
    p[0] = (1.0 + P.kp0 * x0) * P.kp1;
    q[0] = (1.0 + P.kp0 * y0) * P.kp1;
  }
}

__device__ __forceinline__ void load_tri(const Params& P, int e, double* tx, double* ty) {
  const int4 el = __ldg(&P.elem[e]);
  const double2 a = __ldg(&P.vtx[el.x]), b = __ldg(&P.vtx[el.y]), c = __ldg(&P.vtx[el.z]);
  tx[0] = a.x; ty[0] = a.y;
  tx[1] = b.x; ty[1] = b.y;
  tx[2] = c.x; ty[2] = c.y;
}

// twice the signed area, reference order (_engine.py:58)
__device__ __forceinline__ double twice_area(const double* tx, const double* ty) {
  return cross2(tx[1] - tx[0], ty[2] - ty[0], ty[1] - ty[0], tx[2] - tx[0]);
}

// physical 7-point positions on a triangle in the reference's order
// (_engine.py:68-69): T0 + (T1 - T0) * xi0 + (T2 - T0) * xi1, unfused.
__device__ __forceinline__ void rule_points(const Params& P, const double* tx, const double* ty,
                                            double* px, double* py) {
  const double e1x = tx[1] - tx[0], e2x = tx[2] - tx[0];
  const double e1y = ty[1] - ty[0], e2y = ty[2] - ty[0];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    px[p] = __dadd_rn(__dadd_rn(tx[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
    py[p] = __dadd_rn(__dadd_rn(ty[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
  }
}

// ---------------------------------------------------------------------
// full (untruncated) non-identical pair, both visits from one 7x7 pass.
// With P_pq = kernel(x_p, y_q), Q_pq = kernel(y_q, x_p) (x on k, y on l),
// w the 7-point weights, H the hat table and c2 = 2 (2A_k)(2A_l):
//   visit (k, l): kkA[a,b] = c2 sum_p w_p H_pa H_pb sum_q w_q P_pq
//                 klA[a,b] = -c2 sum_pq w_p w_q Q_pq H_pa H_qb
//   visit (l, k): kkB[a,b] = c2 sum_q w_q H_qa H_qb sum_p w_p Q_pq
//                 klB[a,b] = -c2 sum_pq w_p w_q P_pq H_qa H_pb
// (rows a on the visit's root, columns b on its neighbour).
// ---------------------------------------------------------------------
template <int KID>
__device__ __forceinline__ void full_pair2(const Params& P, const double* kx, const double* ky,
                                           const double* lx, const double* ly, double rs2, double* kkA,
                                           double* klA, double* kkB, double* klB, long long& n_eval,
                                           const PowTab* tab) {
  using T = KTraits<KID>;
  constexpr int NC = T::NC, NC2 = T::NC2;
  double xk[7], yk[7], xl[7], yl[7];
  rule_points(P, kx, ky, xk, yk);
  rule_points(P, lx, ly, xl, yl);
  const double c2 = 2.0 * twice_area(kx, ky) * twice_area(lx, ly);
  if constexpr (KID == 2 || KID == 3) {
    if (!(rs2 > 0.0)) {
      // P_pq = P(x_p) and Q_pq = Q(y_q) (constant kernel: both constant): the
      // 7 x 7 sums factor into 7-term sums (same quantities, other rounding)
      //   kkA = c2 (sum_q w_q) sum_p w_p H_pa H_pb P_p    klA = -c2 (sum_p w_p H_pa)(sum_q w_q H_qb Q_q)
      //   kkB = c2 (sum_p w_p) sum_q w_q H_qa H_qb Q_q    klB = -c2 (sum_q w_q H_qa)(sum_p w_p H_pb P_p)
      double sw = 0.0, whs[3] = {0.0, 0.0, 0.0}, ph[3] = {0.0, 0.0, 0.0}, qh[3] = {0.0, 0.0, 0.0};
      double php[9], qhq[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) php[e] = qhq[e] = 0.0;
#pragma unroll
      for (int p = 0; p < 7; ++p) {
        const double Pp = KID == 2 ? P.cst : (1.0 + P.kp0 * xk[p]) * P.kp1;
        const double Qq = KID == 2 ? P.cst : (1.0 + P.kp0 * xl[p]) * P.kp1;
        sw += c_rule.ow[p];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          whs[a] += c_rule.wh[p][a];
          ph[a] = fma(c_rule.wh[p][a], Pp, ph[a]);
          qh[a] = fma(c_rule.wh[p][a], Qq, qh[a]);
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          php[e] = fma(c_rule.whh[p][e], Pp, php[e]);
          qhq[e] = fma(c_rule.whh[p][e], Qq, qhq[e]);
        }
      }
      n_eval += 49;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int e = a * 3 + b;
          kkA[e] = (c2 * sw) * php[e];
          kkB[e] = (c2 * sw) * qhq[e];
          klA[e] = -c2 * whs[a] * qh[b];
          klB[e] = -c2 * whs[a] * ph[b];
        }
      return;
    }
  }
  double colq[7][NC2];
#pragma unroll
  for (int e = 0; e < 9 * NC2; ++e) kkA[e] = klA[e] = klB[e] = 0.0;
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int i = 0; i < NC2; ++i) colq[q][i] = 0.0;
#pragma unroll 1
  for (int p = 0; p < 7; ++p) {
    double rp[NC2], g[3][NC2], gp[T::SYM ? 1 : 3][NC2];
#pragma unroll
    for (int i = 0; i < NC2; ++i) {
      rp[i] = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        g[b][i] = 0.0;
        if (!T::SYM) gp[T::SYM ? 0 : b][i] = 0.0;
      }
    }
    const double wp = c_rule.ow[p];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const double d0 = xk[p] - xl[q], d1 = yk[p] - yl[q];
      const double r2 = sumsq(d0, d1);
      if (rs2 > 0.0 && r2 < rs2) continue;
      double pv[NC2], qv[NC2];
      kval<KID, false, true>(P, xk[p], xl[q], d0, d1, r2, pv, qv, tab);
      ++n_eval;
      const double wq = c_rule.iw[q];
#pragma unroll
      for (int i = 0; i < NC2; ++i) {
        const double qq = T::SYM ? pv[i] : qv[i];
        rp[i] = fma(wq, pv[i], rp[i]);
        colq[q][i] = fma(wp, qq, colq[q][i]);
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          g[b][i] = fma(c_rule.wh[q][b], qq, g[b][i]);
          if (!T::SYM) gp[T::SYM ? 0 : b][i] = fma(c_rule.wh[q][b], pv[i], gp[T::SYM ? 0 : b][i]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int d = 0; d < NC; ++d) {
            const int e = ((a * NC + c) * 3 + b) * NC + d;
            const int cd = c * NC + d;
            kkA[e] = fma(c_rule.whh[p][a * 3 + b], rp[cd], kkA[e]);
            klA[e] = fma(c_rule.wh[p][a], g[b][cd], klA[e]);
            // klB rows a on l (inner hat via g' over q), columns b on k (outer point p)
            klB[e] = fma(c_rule.wh[p][b], T::SYM ? g[a][cd] : gp[T::SYM ? 0 : a][cd], klB[e]);
          }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int d = 0; d < NC; ++d) {
          const int e = ((a * NC + c) * 3 + b) * NC + d;
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < 7; ++q) s = fma(c_rule.whh[q][a * 3 + b], colq[q][c * NC + d], s);
          kkB[e] = s * c2;
          kkA[e] *= c2;
          klA[e] *= -c2;
          klB[e] *= -c2;
        }
}

// full non-identical pair of the peridynamic kernel (kid 1, nc = 2), in the
// unique components only: the kernel matrix P_pq = c dd^T / |d|^3 is
// symmetric (u = 00, 01, 11) and even in d, so Q = P, both own blocks are
// symmetric in (a, b) and (c, d), and klB is the transpose of klA:
//   K [ab][u] = sum_p whh_p[ab] sum_q w_q P_pq[u]     kkA = c2 K
//   K2[ab][u] = sum_q whh_q[ab] sum_p w_p P_pq[u]     kkB = c2 K2
//   G[a][b][u] = sum_pq wh_p[a] wh_q[b] P_pq[u]        klA[(a,c),(b,d)] = -c2 G[a][b][u(c,d)]
//                                                      klB[(a,c),(b,d)] = -c2 G[b][a][u(c,d)]
// (ab: 00 01 02 11 12 22).  66 accumulators instead of four 36-entry blocks.
__device__ __forceinline__ int sym3i(int a, int b) {
  const int i = a < b ? a : b, j = a < b ? b : a;
  return i == 0 ? j : (i == 1 ? 2 + j : 5);
}
__device__ __forceinline__ void full_pair_peri(const Params& P, const double* kx, const double* ky,
                                               const double* lx, const double* ly, double rs2, double (*K)[3],
                                               double (*K2)[3], double (*G)[3][3], long long& n_eval) {
  double xk[7], yk[7], xl[7], yl[7];
  rule_points(P, kx, ky, xk, yk);
  rule_points(P, lx, ly, xl, yl);
  double colq[7][3];
#pragma unroll
  for (int i = 0; i < 6; ++i) K[i][0] = K[i][1] = K[i][2] = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) G[a][b][0] = G[a][b][1] = G[a][b][2] = 0.0;
#pragma unroll
  for (int q = 0; q < 7; ++q) colq[q][0] = colq[q][1] = colq[q][2] = 0.0;
#pragma unroll 1
  for (int p = 0; p < 7; ++p) {
    double rp[3] = {0.0, 0.0, 0.0}, g[3][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) g[b][0] = g[b][1] = g[b][2] = 0.0;
    const double wp = c_rule.ow[p];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const double d0 = xk[p] - xl[q], d1 = yk[p] - yl[q];
      const double r2 = sumsq(d0, d1);
      if (rs2 > 0.0 && r2 < rs2) continue;
      ++n_eval;
      const double f = P.cst / (r2 * sqrt(r2));
      const double pu[3] = {f * d0 * d0, f * d0 * d1, f * d1 * d1};
      const double wq = c_rule.iw[q];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        rp[u] = fma(wq, pu[u], rp[u]);
        colq[q][u] = fma(wp, pu[u], colq[q][u]);
#pragma unroll
        for (int b = 0; b < 3; ++b) g[b][u] = fma(c_rule.wh[q][b], pu[u], g[b][u]);
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b)
#pragma unroll
        for (int u = 0; u < 3; ++u) K[sym3i(a, b)][u] = fma(c_rule.whh[p][a * 3 + b], rp[u], K[sym3i(a, b)][u]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int u = 0; u < 3; ++u) G[a][b][u] = fma(c_rule.wh[p][a], g[b][u], G[a][b][u]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b)
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q) v = fma(c_rule.whh[q][a * 3 + b], colq[q][u], v);
        K2[sym3i(a, b)][u] = v;
      }
}

// full non-identical pair of a symmetric scalar kernel (kid 0): P_pq =
// kernel(|x_p - y_q|) = Q_pq, so klB = klA^T and both own blocks are
// symmetric: K[ab] = sum_p whh_p[ab] sum_q w_q P_pq (kkA = c2 K), K2 from the
// column sums (kkB = c2 K2), G[a][b] = sum_pq wh_p[a] wh_q[b] P_pq
// (klA = -c2 G, klB = -c2 G^T).  22 accumulators instead of four 9-entry
// blocks plus the column sums.
__device__ __forceinline__ void full_pair_sym1(const Params& P, const double* kx, const double* ky,
                                               const double* lx, const double* ly, double* K, double* K2,
                                               double (*G)[3], long long& n_eval, const PowTab* tab) {
  double xk[7], yk[7], xl[7], yl[7];
  rule_points(P, kx, ky, xk, yk);
  rule_points(P, lx, ly, xl, yl);
  double colq[7];
#pragma unroll
  for (int i = 0; i < 6; ++i) K[i] = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) G[a][0] = G[a][1] = G[a][2] = 0.0;
#pragma unroll
  for (int q = 0; q < 7; ++q) colq[q] = 0.0;
#pragma unroll 1
  for (int p = 0; p < 7; ++p) {
    double rp = 0.0, g[3] = {0.0, 0.0, 0.0};
    const double wp = c_rule.ow[p];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const double d0 = xk[p] - xl[q], d1 = yk[p] - yl[q];
      const double r2 = sumsq(d0, d1);
      double pv[1], qv[1];
      kval<0, false, true>(P, xk[p], xl[q], d0, d1, r2, pv, qv, tab);
      rp = fma(c_rule.iw[q], pv[0], rp);
      colq[q] = fma(wp, pv[0], colq[q]);
#pragma unroll
      for (int b = 0; b < 3; ++b) g[b] = fma(c_rule.wh[q][b], pv[0], g[b]);
    }
    n_eval += 49 / 7;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b) K[sym3i(a, b)] = fma(c_rule.whh[p][a * 3 + b], rp, K[sym3i(a, b)]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) G[a][b] = fma(c_rule.wh[p][a], g[b], G[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 7; ++q) v = fma(c_rule.whh[q][a * 3 + b], colq[q], v);
      K2[sym3i(a, b)] = v;
    }
}

// full identical pair (k == l, mode 2): both column halves land on k's dofs;
// returned as the two halves so the presence test matches the reference's
// per-triplet `v != 0` (_engine.py:403-424).
template <int KID>
__device__ __forceinline__ void full_identical(const Params& P, const double* kx, const double* ky,
                                               double rs2, double* h0, double* h1, long long& n_eval,
                                               const PowTab* tab) {
  using T = KTraits<KID>;
  constexpr int NC = T::NC, NC2 = T::NC2;
  double xk[7], yk[7];
  rule_points(P, kx, ky, xk, yk);
  const double ta = twice_area(kx, ky);
  const double c = ta * ta;
  double colq[7][NC2];
#pragma unroll
  for (int e = 0; e < 9 * NC2; ++e) { h0[e] = 0.0; h1[e] = 0.0; }
  for (int q = 0; q < 7; ++q)
    for (int i = 0; i < NC2; ++i) colq[q][i] = 0.0;
  for (int p = 0; p < 7; ++p) {
    double rp[NC2], gq[3][NC2], gp[3][NC2];
    for (int i = 0; i < NC2; ++i) { rp[i] = 0.0; for (int b = 0; b < 3; ++b) gq[b][i] = gp[b][i] = 0.0; }
    for (int q = 0; q < 7; ++q) {
      const double d0 = xk[p] - xk[q], d1 = yk[p] - yk[q];
      const double r2 = sumsq(d0, d1);
      if (rs2 > 0.0 && r2 < rs2) continue;
      double pv[NC2], qv[NC2];
      kval<KID, true, true>(P, xk[p], xk[q], d0, d1, r2, pv, qv, tab);
      ++n_eval;
      for (int i = 0; i < NC2; ++i) {
        const double qq = T::SYM ? pv[i] : qv[i];
        rp[i] += c_rule.iw[q] * pv[i];
        colq[q][i] += c_rule.ow[p] * qq;
        for (int b = 0; b < 3; ++b) {
          gq[b][i] += c_rule.wh[q][b] * qq;
          gp[b][i] += c_rule.wh[q][b] * pv[i];
        }
      }
    }
    for (int a = 0; a < 3; ++a)
      for (int cc = 0; cc < NC; ++cc)
        for (int b = 0; b < 3; ++b)
          for (int d = 0; d < NC; ++d) {
            const int e = ((a * NC + cc) * 3 + b) * NC + d;
            const int i = cc * NC + d;
            h0[e] += c_rule.whh[p][a * 3 + b] * rp[i];
            h1[e] -= c_rule.wh[p][a] * gq[b][i] + c_rule.wh[p][b] * gp[a][i];
          }
  }
  for (int q = 0; q < 7; ++q)
    for (int a = 0; a < 3; ++a)
      for (int cc = 0; cc < NC; ++cc)
        for (int b = 0; b < 3; ++b)
          for (int d = 0; d < NC; ++d) {
            const int e = ((a * NC + cc) * 3 + b) * NC + d;
            h0[e] += c_rule.whh[q][a * 3 + b] * colq[q][cc * NC + d];
          }
  for (int e = 0; e < 9 * NC2; ++e) { h0[e] *= c; h1[e] *= c; }
}

}  // namespace nlg
