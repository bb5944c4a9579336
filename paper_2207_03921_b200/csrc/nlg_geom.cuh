// nlg_geom.cuh -- device clipping of an inner triangle against the
// interaction ball of one outer quadrature point.
//
// Every predicate that decides the sparsity pattern must reproduce the
// reference's floating-point decisions exactly, so these routines restate
// /root/reference/pkg/src/nlfem/_geom_scalar.py operation for operation
// (clip_circle :27-115, insert_caps :118-181, clip_square :184-266):
// products that feed a sum go through __dmul_rn so nvcc cannot contract
// them into FMAs (numba does not fuse), sqrt and division are IEEE.
//
// Output goes to caller-provided rows (shared memory in the clipped-pair
// kernel) instead of local arrays, and the code is kept compact (no loop
// unrolling): the clipped-pair kernel is instruction-cache bound otherwise.
#pragma once
#include <cstdint>

namespace nlg {

constexpr double kBallTieRel = 1e-12;    // _geom_scalar.py:15
constexpr double kDedupRel = 1e-13;      // _geom_scalar.py:18
constexpr double kChordSkipRel = 1e-10;  // _geom_scalar.py:21
constexpr double kCapMemberRel = 1e-12;  // _geom_scalar.py:24
constexpr int kMaxPoly = 9;              // triangle -> <= 6 clip rows, <= 9 with (<= 3) caps
constexpr int kMaxBase = 7;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
// a*a + b*b without contraction
__device__ __forceinline__ double sumsq(double a, double b) { return __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)); }
// a*b - c*d without contraction
__device__ __forceinline__ double cross2(double a, double b, double c, double d) {
  return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
}

// A triangle passed by value so it stays in registers across the
// (non-inlined) clip calls; vertex i is selected without local memory.
struct Tri {
  double x0, x1, x2, y0, y1, y2;
  __device__ __forceinline__ double x(int i) const { return i == 0 ? x0 : (i == 1 ? x1 : x2); }
  __device__ __forceinline__ double y(int i) const { return i == 0 ? y0 : (i == 1 ? y1 : y2); }
};

__device__ __forceinline__ Tri make_tri(const double* tx, const double* ty) {
  return Tri{tx[0], tx[1], tx[2], ty[0], ty[1], ty[2]};
}

// append (px, py) unless it repeats the previous row within dtol
__device__ __forceinline__ void push_dedup(double* ox, double* oy, unsigned& flags, int& n, double px,
                                           double py, bool crossing, double dtol, bool first_ok) {
  if ((first_ok && n == 0) || fabs(ox[n - 1] - px) > dtol || fabs(oy[n - 1] - py) > dtol) {
    ox[n] = px;
    oy[n] = py;
    if (crossing) flags |= 1u << n;
    ++n;
  }
}

// The rows of a clip in progress: the last (and first) row stay in
// registers, so the dedup test of a push reads no memory.
struct ClipRows {
  double* ox;
  double* oy;
  double dtol, lx, ly, fx, fy;
  unsigned flags;
  int n;
  __device__ __forceinline__ void push(bool on, double px, double py, bool crossing, bool first_ok) {
    if (on && ((first_ok && n == 0) || fabs(lx - px) > dtol || fabs(ly - py) > dtol)) {
      ox[n] = px;
      oy[n] = py;
      if (n == 0) { fx = px; fy = py; }
      lx = px;
      ly = py;
      if (crossing) flags |= 1u << n;
      ++n;
    }
  }
};

// clip_circle: vertices of the convex CCW triangle T inside the closed disk
// around (cx, cy) plus edge/circle crossings; bit i of *flags_out marks row i
// as a crossing.  Returns the row count (< 3: empty/degenerate).
// The reference's three cases per edge (leaving / entering / through the
// disk, _geom_scalar.py:75-108) run as one predicated sequence -- lanes of a
// warp clip different triangles, and a branch per case would run every case
// in turn: one square root, the first root's division for every crossing
// edge, the second root's only for "through" edges.  Same operations on the
// same operands as the reference; rows pushed in the same order.
__device__ __forceinline__ int clip_circle(Tri T, double cx, double cy, double delta, double* ox, double* oy,
                                        unsigned* flags_out) {
  const double rad = mul(delta, 1.0 + kBallTieRel);
  const double r2 = mul(rad, rad);
  const double q0 = __dsub_rn(sumsq(T.x0 - cx, T.y0 - cy), r2);
  const double q1 = __dsub_rn(sumsq(T.x1 - cx, T.y1 - cy), r2);
  const double q2 = __dsub_rn(sumsq(T.x2 - cx, T.y2 - cy), r2);
  ClipRows R{ox, oy, mul(kDedupRel, delta), 0.0, 0.0, 0.0, 0.0, 0u, 0};
  if (q0 <= 0.0 && q1 <= 0.0 && q2 <= 0.0) {
    // every edge runs inside: the general loop would only append the vertices
    R.push(true, T.x0, T.y0, false, true);
    R.push(true, T.x1, T.y1, false, true);
    R.push(true, T.x2, T.y2, false, true);
  } else {
#pragma unroll 1  // (unrolled: +7 % kernel time on config 5 -- code size)
    for (int i = 0; i < 3; ++i) {
      const int j = i == 2 ? 0 : i + 1;
      const double ax = T.x(i), ay = T.y(i), bx = T.x(j), by = T.y(j);
      const double qa = i == 0 ? q0 : (i == 1 ? q1 : q2);
      const double qb = j == 0 ? q0 : (j == 1 ? q1 : q2);
      const bool ina = qa <= 0.0, inb = qb <= 0.0;
      const double dax = ax - cx, day = ay - cy;
      R.push(ina, ax, ay, false, true);
      const double ex = bx - ax, ey = by - ay;
      const double aa = sumsq(ex, ey);
      const double bb = mul(2.0, __dadd_rn(mul(ex, dax), mul(ey, day)));
      const double disc = __dsub_rn(mul(bb, bb), mul(mul(4.0, aa), qa));
      const bool cross = !(aa <= 0.0) && !(ina && inb) && !(disc <= 0.0);
      if (!cross) continue;
      const double sq = sqrt(disc);
      const double den = mul(2.0, aa);
      // first root of the edge: the exit root when leaving, else the entry root
      const double ta = (ina ? -bb + sq : -bb - sq) / den;
      const bool through = !ina && !inb;
      double tb = 0.0;
      if (through) tb = (-bb + sq) / den;
      const bool ok = through ? (0.0 < ta && tb < 1.0 && ta < tb) : (0.0 < ta && ta < 1.0);
      R.push(ok, __dadd_rn(ax, mul(ta, ex)), __dadd_rn(ay, mul(ta, ey)), true, true);
      R.push(ok && through, __dadd_rn(ax, mul(tb, ex)), __dadd_rn(ay, mul(tb, ey)), true, false);
    }
  }
  int n = R.n;
  if (n >= 2 && fabs(R.fx - R.lx) <= R.dtol && fabs(R.fy - R.ly) <= R.dtol) --n;
  *flags_out = R.flags & ((1u << n) - 1u);
  return n;
}

// insert_caps: copy the clip rows to (px, py), adding the arc midpoint behind
// every chord between consecutive crossings when it lies inside the triangle.
// The (<= 3) chords are evaluated first, one per trip of a short loop -- so
// lanes clipping different triangles do their square roots and divisions
// together -- and the rows are copied afterwards.
__device__ __forceinline__ int insert_caps(Tri T, const double* bx, const double* by, unsigned bflag, int nb,
                                        double cx, double cy, double delta, double* px, double* py) {
  if (nb < 2) {
    for (int i = 0; i < nb; ++i) { px[i] = bx[i]; py[i] = by[i]; }
    return nb;
  }
  const double rad = mul(delta, 1.0 + kBallTieRel);
  // a cap needs a crossing followed (cyclically) by a crossing
  const unsigned next = (bflag >> 1) | ((bflag & 1u) << (nb - 1));
  unsigned cand = bflag & next, capmask = 0;
  double capx0 = 0.0, capy0 = 0.0, capx1 = 0.0, capy1 = 0.0, capx2 = 0.0, capy2 = 0.0;
  if (cand) {
    const double el0 = sqrt(sumsq(T.x1 - T.x0, T.y1 - T.y0));
    const double el1 = sqrt(sumsq(T.x2 - T.x1, T.y2 - T.y1));
    const double el2 = sqrt(sumsq(T.x0 - T.x2, T.y0 - T.y2));
    double href = el0;
    if (el1 > href) href = el1;
    if (el2 > href) href = el2;
    const double tol = mul(-kCapMemberRel, href);
    int c = 0;
#pragma unroll 1
    while (cand) {
      const int i = __ffs(cand) - 1;
      cand &= cand - 1;
      const int j = i + 1 == nb ? 0 : i + 1;
      const double bix = bx[i], biy = by[i], bjx = bx[j], bjy = by[j];
      const double chx = bjx - bix, chy = bjy - biy;
      const double chord = sqrt(sumsq(chx, chy));
      const double mx = __dsub_rn(mul(0.5, __dadd_rn(bix, bjx)), cx);
      const double my = __dsub_rn(mul(0.5, __dadd_rn(biy, bjy)), cy);
      const double nd = sqrt(sumsq(mx, my));
      if (chord < mul(kChordSkipRel, delta) || nd < mul(1e-14, delta)) continue;
      const double capx = __dadd_rn(cx, mul(rad, mx) / nd);
      const double capy = __dadd_rn(cy, mul(rad, my) / nd);
      // membership against the three edges (the reference stops at the first miss)
      const bool inside = cross2(T.x1 - T.x0, capy - T.y0, T.y1 - T.y0, capx - T.x0) >= mul(tol, el0) &&
                          cross2(T.x2 - T.x1, capy - T.y1, T.y2 - T.y1, capx - T.x1) >= mul(tol, el1) &&
                          cross2(T.x0 - T.x2, capy - T.y2, T.y0 - T.y2, capx - T.x2) >= mul(tol, el2);
      if (inside) {
        capmask |= 1u << i;
        if (c == 0) { capx0 = capx; capy0 = capy; }
        else if (c == 1) { capx1 = capx; capy1 = capy; }
        else { capx2 = capx; capy2 = capy; }
        ++c;
      }
    }
  }
  // rows in order, each followed by its cap ((px, py) may alias (bx - 3, by - 3):
  // row i lands at i + caps so far <= 3 + i, never ahead of an unread row)
  int n = 0, c = 0;
#pragma unroll 1
  for (int i = 0; i < nb; ++i) {
    const double rx = bx[i], ry = by[i];
    px[n] = rx;
    py[n] = ry;
    ++n;
    if ((capmask >> i) & 1u) {
      px[n] = c == 0 ? capx0 : (c == 1 ? capx1 : capx2);
      py[n] = c == 0 ? capy0 : (c == 1 ? capy1 : capy2);
      ++n;
      ++c;
    }
  }
  return n;
}

// clip_square: Sutherland-Hodgman against the box of half width delta;
// (bx, by) is scratch of kMaxPoly rows, the result lands in (px, py).
__device__ __noinline__ int clip_square(Tri T, double cx, double cy, double delta, double* bx, double* by,
                                        double* px, double* py) {
  int n = 3;
  bx[0] = T.x0; bx[1] = T.x1; bx[2] = T.x2;
  by[0] = T.y0; by[1] = T.y1; by[2] = T.y2;
#pragma unroll 1
  for (int plane = 0; plane < 4; ++plane) {
    const bool axis1 = plane >= 2;
    const bool keep_ge = (plane & 1) == 0;
    const double bound = plane == 0 ? cx - delta : plane == 1 ? cx + delta : plane == 2 ? cy - delta : cy + delta;
    int nn = 0;
    for (int i = 0; i < n; ++i) {
      const int j = i + 1 == n ? 0 : i + 1;
      const double c0 = bx[i], c1 = by[i], d0 = bx[j], d1 = by[j];
      const double cv = axis1 ? c1 : c0, dv = axis1 ? d1 : d0;
      const bool cin = keep_ge ? cv >= bound : cv <= bound;
      const bool din = keep_ge ? dv >= bound : dv <= bound;
      if (cin) { px[nn] = c0; py[nn] = c1; ++nn; }
      if (cin != din) {
        const double t = (bound - cv) / (dv - cv);
        px[nn] = __dadd_rn(c0, mul(t, d0 - c0));
        py[nn] = __dadd_rn(c1, mul(t, d1 - c1));
        ++nn;
      }
    }
    n = nn;
    for (int i = 0; i < n; ++i) { bx[i] = px[i]; by[i] = py[i]; }
    if (n == 0) break;
  }
  const double dtol = mul(kDedupRel, delta);
  int nn = 0;
  for (int i = 0; i < n; ++i) {
    if (nn > 0 && fabs(bx[i] - px[nn - 1]) <= dtol && fabs(by[i] - py[nn - 1]) <= dtol) continue;
    px[nn] = bx[i];
    py[nn] = by[i];
    ++nn;
  }
  if (nn >= 2 && fabs(px[0] - px[nn - 1]) <= dtol && fabs(py[0] - py[nn - 1]) <= dtol) --nn;
  return nn < 3 ? 0 : nn;
}

// Balls 0 / 1 without scratch rows: clip_circle writes its (<= 6) rows at
// offset 3 of (px, py) and insert_caps compacts them to the front, adding
// (<= 3) caps.  Row i's output lands at i + (caps so far) <= 3 + i, and a cap
// after it needs caps so far <= 2, so no input row is overwritten before it
// is read (row 0 is kept in registers).
__device__ __forceinline__ int truncate_inner_inplace(Tri T, double cx, double cy, double delta, int ball,
                                                      double* px, double* py) {
  unsigned f;
  if (ball == 0) return clip_circle(T, cx, cy, delta, px, py, &f);
  const int nb = clip_circle(T, cx, cy, delta, px + 3, py + 3, &f);
  return insert_caps(T, px + 3, py + 3, f, nb, cx, cy, delta, px, py);
}

// The truncated inner region of triangle T seen from outer point (cx, cy),
// _engine._sweep :70-91 (ball 0 = nocaps, 1 = approxcaps, 2 = inf).
// (sx, sy) is scratch of kMaxPoly rows; the polygon lands in (px, py).
__device__ __forceinline__ int truncate_inner(Tri T, double cx, double cy, double delta, int ball, double* sx,
                                              double* sy, double* px, double* py) {
  if (ball == 2) return clip_square(T, cx, cy, delta, sx, sy, px, py);
  unsigned f;
  if (ball == 0) return clip_circle(T, cx, cy, delta, px, py, &f);
  const int nb = clip_circle(T, cx, cy, delta, sx, sy, &f);
  return insert_caps(T, sx, sy, f, nb, cx, cy, delta, px, py);
}

__device__ __forceinline__ int truncate_inner(const double* tx, const double* ty, double cx, double cy,
                                              double delta, int ball, double* sx, double* sy, double* px,
                                              double* py) {
  return truncate_inner(make_tri(tx, ty), cx, cy, delta, ball, sx, sy, px, py);
}

}  // namespace nlg
