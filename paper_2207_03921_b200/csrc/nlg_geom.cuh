// nlg_geom.cuh -- device clipping of an inner triangle against the
// interaction ball of one outer quadrature point.
//
// Every predicate that decides the sparsity pattern must reproduce the
// reference's floating-point decisions exactly, so these routines restate
// /root/reference/pkg/src/nlfem/_geom_scalar.py operation for operation
// (clip_circle :27-115, insert_caps :118-181, clip_square :184-266):
// products that feed a sum go through __dmul_rn so nvcc cannot contract
// them into FMAs (numba does not fuse), sqrt and division are IEEE.
#pragma once
#include <cstdint>

namespace nlg {

constexpr double kBallTieRel = 1e-12;    // _geom_scalar.py:15
constexpr double kDedupRel = 1e-13;      // _geom_scalar.py:18
constexpr double kChordSkipRel = 1e-10;  // _geom_scalar.py:21
constexpr double kCapMemberRel = 1e-12;  // _geom_scalar.py:24
constexpr int kMaxPoly = 12;             // triangle -> <= 6 clip rows, <= 9 with caps

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
// a*a + b*b without contraction
__device__ __forceinline__ double sumsq(double a, double b) { return __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)); }
// a*b - c*d without contraction
__device__ __forceinline__ double cross2(double a, double b, double c, double d) {
  return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
}

struct Poly {
  double x[kMaxPoly], y[kMaxPoly];
  int n;
};

// clip_circle: vertices of the convex CCW triangle (tx, ty) inside the
// closed disk around (cx, cy) plus edge/circle crossings, with crossing
// flags; returns the row count (< 3 means empty/degenerate).
__device__ __forceinline__ int clip_circle(const double* tx, const double* ty, double cx, double cy,
                                           double delta, double* ox, double* oy, bool* oflag) {
  const double rad = mul(delta, 1.0 + kBallTieRel);
  const double r2 = mul(rad, rad);
  const double dtol = mul(kDedupRel, delta);
  int n = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = i == 2 ? 0 : i + 1;
    const double ax = tx[i], ay = ty[i], bx = tx[j], by = ty[j];
    const double dax = ax - cx, day = ay - cy;
    const double qa = __dsub_rn(sumsq(dax, day), r2);
    const double dbx = bx - cx, dby = by - cy;
    const double qb = __dsub_rn(sumsq(dbx, dby), r2);
    if (qa <= 0.0) {
      if (n == 0 || fabs(ox[n - 1] - ax) > dtol || fabs(oy[n - 1] - ay) > dtol) {
        ox[n] = ax; oy[n] = ay; oflag[n] = false; ++n;
      }
    }
    const double ex = bx - ax, ey = by - ay;
    const double aa = sumsq(ex, ey);
    if (aa <= 0.0) continue;
    if (qa <= 0.0 && qb <= 0.0) continue;
    const double bb = mul(2.0, __dadd_rn(mul(ex, dax), mul(ey, day)));
    const double disc = __dsub_rn(mul(bb, bb), mul(mul(4.0, aa), qa));
    if (disc <= 0.0) continue;
    const double sq = sqrt(disc);
    const double den = mul(2.0, aa);
    const double t1 = (-bb - sq) / den;
    const double t2 = (-bb + sq) / den;
    if (qa <= 0.0) {
      if (0.0 < t2 && t2 < 1.0) {
        const double px = __dadd_rn(ax, mul(t2, ex)), py = __dadd_rn(ay, mul(t2, ey));
        if (n == 0 || fabs(ox[n - 1] - px) > dtol || fabs(oy[n - 1] - py) > dtol) {
          ox[n] = px; oy[n] = py; oflag[n] = true; ++n;
        }
      }
    } else if (qb <= 0.0) {
      if (0.0 < t1 && t1 < 1.0) {
        const double px = __dadd_rn(ax, mul(t1, ex)), py = __dadd_rn(ay, mul(t1, ey));
        if (n == 0 || fabs(ox[n - 1] - px) > dtol || fabs(oy[n - 1] - py) > dtol) {
          ox[n] = px; oy[n] = py; oflag[n] = true; ++n;
        }
      }
    } else if (0.0 < t1 && t2 < 1.0 && t1 < t2) {
      double px = __dadd_rn(ax, mul(t1, ex)), py = __dadd_rn(ay, mul(t1, ey));
      if (n == 0 || fabs(ox[n - 1] - px) > dtol || fabs(oy[n - 1] - py) > dtol) {
        ox[n] = px; oy[n] = py; oflag[n] = true; ++n;
      }
      px = __dadd_rn(ax, mul(t2, ex));
      py = __dadd_rn(ay, mul(t2, ey));
      if (fabs(ox[n - 1] - px) > dtol || fabs(oy[n - 1] - py) > dtol) {
        ox[n] = px; oy[n] = py; oflag[n] = true; ++n;
      }
    }
  }
  if (n >= 2 && fabs(ox[0] - ox[n - 1]) <= dtol && fabs(oy[0] - oy[n - 1]) <= dtol) --n;
  return n;
}

// insert_caps: add the arc midpoint behind every chord between consecutive
// crossings when it lies inside the triangle; result in p.
__device__ __forceinline__ void insert_caps(const double* tx, const double* ty, const double* bx,
                                            const double* by, const bool* bflag, int nb, double cx,
                                            double cy, double delta, Poly& p) {
  const double rad = mul(delta, 1.0 + kBallTieRel);
  if (nb < 2) {
    for (int i = 0; i < nb; ++i) { p.x[i] = bx[i]; p.y[i] = by[i]; }
    p.n = nb;
    return;
  }
  double el[3];
  double href = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = i == 2 ? 0 : i + 1;
    const double ex = tx[j] - tx[i], ey = ty[j] - ty[i];
    el[i] = sqrt(sumsq(ex, ey));
    if (el[i] > href) href = el[i];
  }
  int n = 0;
  for (int i = 0; i < nb; ++i) {
    const int j = i + 1 == nb ? 0 : i + 1;
    p.x[n] = bx[i]; p.y[n] = by[i]; ++n;
    if (!bflag[i] || !bflag[j]) continue;
    const double chx = bx[j] - bx[i], chy = by[j] - by[i];
    const double chord = sqrt(sumsq(chx, chy));
    if (chord < mul(kChordSkipRel, delta)) continue;
    const double mx = __dsub_rn(mul(0.5, __dadd_rn(bx[i], bx[j])), cx);
    const double my = __dsub_rn(mul(0.5, __dadd_rn(by[i], by[j])), cy);
    const double nd = sqrt(sumsq(mx, my));
    if (nd < mul(1e-14, delta)) continue;
    const double capx = __dadd_rn(cx, mul(rad, mx) / nd);
    const double capy = __dadd_rn(cy, mul(rad, my) / nd);
    bool inside = true;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const int f = e == 2 ? 0 : e + 1;
      const double ex = tx[f] - tx[e], ey = ty[f] - ty[e];
      const double cr = cross2(ex, capy - ty[e], ey, capx - tx[e]);
      if (cr < mul(mul(-kCapMemberRel, href), el[e])) { inside = false; break; }
    }
    if (inside) { p.x[n] = capx; p.y[n] = capy; ++n; }
  }
  p.n = n;
}

// clip_square: Sutherland-Hodgman against the box of half width delta.
__device__ __forceinline__ void clip_square(const double* tx, const double* ty, double cx, double cy,
                                            double delta, Poly& out) {
  double bx[kMaxPoly], by[kMaxPoly];
  const double bounds[4] = {cx - delta, cx + delta, cy - delta, cy + delta};
  int n = 3;
  for (int i = 0; i < 3; ++i) { bx[i] = tx[i]; by[i] = ty[i]; }
  for (int plane = 0; plane < 4; ++plane) {
    const bool axis1 = plane >= 2;
    const bool keep_ge = (plane & 1) == 0;
    const double bound = bounds[plane];
    int nn = 0;
    for (int i = 0; i < n; ++i) {
      const int j = i + 1 == n ? 0 : i + 1;
      const double c0 = bx[i], c1 = by[i], d0 = bx[j], d1 = by[j];
      const double cv = axis1 ? c1 : c0, dv = axis1 ? d1 : d0;
      const bool cin = keep_ge ? cv >= bound : cv <= bound;
      const bool din = keep_ge ? dv >= bound : dv <= bound;
      if (cin) { out.x[nn] = c0; out.y[nn] = c1; ++nn; }
      if (cin != din) {
        const double t = (bound - cv) / (dv - cv);
        out.x[nn] = __dadd_rn(c0, mul(t, d0 - c0));
        out.y[nn] = __dadd_rn(c1, mul(t, d1 - c1));
        ++nn;
      }
    }
    n = nn;
    for (int i = 0; i < n; ++i) { bx[i] = out.x[i]; by[i] = out.y[i]; }
    if (n == 0) break;
  }
  const double dtol = mul(kDedupRel, delta);
  int nn = 0;
  for (int i = 0; i < n; ++i) {
    if (nn > 0 && fabs(bx[i] - out.x[nn - 1]) <= dtol && fabs(by[i] - out.y[nn - 1]) <= dtol) continue;
    out.x[nn] = bx[i]; out.y[nn] = by[i]; ++nn;
  }
  if (nn >= 2 && fabs(out.x[0] - out.x[nn - 1]) <= dtol && fabs(out.y[0] - out.y[nn - 1]) <= dtol) --nn;
  out.n = nn < 3 ? 0 : nn;
}

// The truncated inner region of triangle (tx, ty) seen from outer point
// (cx, cy): _engine._sweep :70-91.  ball 0 = nocaps, 1 = approxcaps, 2 = inf.
__device__ __forceinline__ void truncate_inner(const double* tx, const double* ty, double cx, double cy,
                                               double delta, int ball, Poly& p) {
  if (ball == 2) {
    clip_square(tx, ty, cx, cy, delta, p);
    return;
  }
  double bx[kMaxPoly], by[kMaxPoly];
  bool bf[kMaxPoly];
  const int nb = clip_circle(tx, ty, cx, cy, delta, bx, by, bf);
  if (ball == 0) {
    for (int i = 0; i < nb; ++i) { p.x[i] = bx[i]; p.y[i] = by[i]; }
    p.n = nb;
  } else {
    insert_caps(tx, ty, bx, by, bf, nb, cx, cy, delta, p);
  }
}

}  // namespace nlg
