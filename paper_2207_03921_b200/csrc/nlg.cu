// nlg.cu -- B200 (sm_100a) nonlocal stiffness assembly: kernels, the
// per-batch pipeline and the C ABI declared in include/nlg.h.
//
// Pipeline of one nlg_assemble call (rows [row_lo, row_hi)):
//   prep      k_bounds (barycentre/radius, assembly.py:130-134),
//             k_cell + radix sort + k_cell_ranges: uniform grid of
//             barycentres, pitch (prer + 2 r_max)/2 (replaces the BFS of
//             _engine.py:530-599 with the exhaustive "brute" semantics,
//             _engine.py:486-529, which the reference equals bitwise under
//             its Assumption 4)
//   batch     k_mark_*: owner-computes root selection for the row range
//             k_candidates<count / fill>: pair records per root (each
//             unordered pair once, serving both visits), split into full and
//             clipped lists, plus singular (identical / edge / vertex) lists
//             k_full: one thread per full record (7x7 point matrix)
//             k_clipped: block-cooperative clipped records (clip queue,
//             sub-triangle queue, fold)
//             k_singular<U>: one CTA per touching pair, tensor rules
//   merge     k_root_reduce (stage R): per-root block sort-reduce of the
//             record blocks -> COO runs; radix sort of the (row, col) keys
//             + k_seg_*: deterministic segmented sums -> CSR (replaces
//             _merge_triplets, assembly.py:137-173)
#include <cub/cub.cuh>
#include <type_traits>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/nlg.h"
#include "nlg_eval.cuh"

using namespace nlg;

namespace {

thread_local std::string g_err;
const bool g_trace = getenv("NLG_TRACE") != nullptr;
double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define TRACE(tag)                                                                  \
  do {                                                                              \
    if (g_trace) fprintf(stderr, "[nlg %10.3f] %s\n", host_ms(), tag);             \
  } while (0)
std::atomic<long long> g_launches{0};

void set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      set_err("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));             \
      return NLG_ERR_CUDA;                                                                 \
    }                                                                                      \
  } while (0)

#define LAUNCHED()                                                                         \
  do {                                                                                     \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                    \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess) {                                                               \
      set_err("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_));             \
      return NLG_ERR_CUDA;                                                                 \
    }                                                                                      \
  } while (0)

constexpr unsigned long long kSentinel = ~0ull;
constexpr int kCnt = 7;  // per-root counters: full, partial, sing id/edge/vertex, epi, emit-kk
enum { C_FULL = 0, C_PART = 1, C_SID = 2, C_SED = 3, C_SVX = 4, C_EPI = 5, C_KK = 6 };

// device counters (FLOP accounting), indices
enum {
  K_EVAL_FULL0 = 0,  // inner evals the reference makes for full pairs: mode0 + mode1 (2 x 49)
  K_EVAL_FULL2,      // identical full pairs, mode 2
  K_OUT_FULL0,       // outer points (7 per sweep)
  K_OUT_FULL2,
  K_EVAL_M0, K_EVAL_M1, K_EVAL_M2,
  K_OUT_M0, K_OUT_M1, K_OUT_M2,
  K_SPTS3, K_SPTS4, K_SPTS5, K_SPTS6,
  K_DBG_SUBTRI, K_DBG_ROUNDS, K_DBG_CHUNKS, K_DBG_ITEMS, K_DBG_FAR, K_DBG_INSIDE, K_DBG_NONEMPTY,
  K_NCOUNTERS
};

__device__ __forceinline__ unsigned long long d2ord(double v) {
  unsigned long long b = __double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double ord2d(unsigned long long o) {
  unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  double v;
  memcpy(&v, &b, 8);
  return v;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__constant__ int g_trace_dev;  // NLG_TRACE: device-side debug counters

// ---------------------------------------------------------------- prep
__global__ void k_convert(const double* __restrict__ vin, const long long* __restrict__ ein,
                          const long long* __restrict__ lab, const long long* __restrict__ outer,
                          const long long* __restrict__ dof, int V, int K, double2* vtx, int4* elem,
                          int4* dofs) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < V) vtx[i] = make_double2(vin[2 * i], vin[2 * i + 1]);
  if (i < K) {
    const int flags = (int)lab[i] | ((outer[i] != 0) << 4);
    elem[i] = make_int4((int)ein[3 * i], (int)ein[3 * i + 1], (int)ein[3 * i + 2], flags);
    dofs[i] = make_int4((int)dof[3 * i], (int)dof[3 * i + 1], (int)dof[3 * i + 2], 0);
  }
}

// barycentre ((v0 + v1) + v2) / 3 and bounding radius, numpy's order
// (assembly.py:130-134); bbox/rmax over active elements via ordered atomics
__global__ void k_bounds(Params P, double2* ctr, double* rad, unsigned long long* ext) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  // bbox / max radius of the active elements: warp reductions, one atomic
  // per warp and word
  unsigned long long mn0 = ~0ull, mn1 = ~0ull, mx0 = 0, mx1 = 0, mr = 0;
  if (k < P.K) {
    const int4 e = P.elem[k];
    const double2 a = P.vtx[e.x], b = P.vtx[e.y], c = P.vtx[e.z];
    const double cx = __dadd_rn(__dadd_rn(a.x, b.x), c.x) / 3.0;
    const double cy = __dadd_rn(__dadd_rn(a.y, b.y), c.y) / 3.0;
    const double ra = sqrt(sumsq(a.x - cx, a.y - cy));
    const double rb = sqrt(sumsq(b.x - cx, b.y - cy));
    const double rc = sqrt(sumsq(c.x - cx, c.y - cy));
    const double r = fmax(fmax(ra, rb), rc);
    ctr[k] = make_double2(cx, cy);
    rad[k] = r;
    if ((e.w & 15) != 0) {
      mn0 = mx0 = d2ord(cx);
      mn1 = mx1 = d2ord(cy);
      mr = d2ord(r);
    }
  }
  for (int o = 16; o; o >>= 1) {
    mn0 = min(mn0, __shfl_xor_sync(0xffffffffu, mn0, o));
    mn1 = min(mn1, __shfl_xor_sync(0xffffffffu, mn1, o));
    mx0 = max(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = max(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
  }
  if (lane_id() == 0 && mr) {
    atomicMin(&ext[0], mn0);
    atomicMin(&ext[1], mn1);
    atomicMax(&ext[2], mx0);
    atomicMax(&ext[3], mx1);
    atomicMax(&ext[4], mr);
  }
}

struct Grid {
  double ox, oy, cs;
  double reach;  // candidate radius around a barycentre: prer + 2 r_max (widened)
  double rmax;   // largest element radius
  int nx, ny, span;
  const int* __restrict__ start;  // [ncell + 1]
  const int* __restrict__ items;  // active element ids sorted by cell
  // the items' element records, barycentres and radii in the same order
  // (the candidate scans read them coalesced)
  const int4* __restrict__ gel;
  const double2* __restrict__ gctr;
  const double* __restrict__ grad;
  const double4* __restrict__ gft;  // analytic: (A2 psi_0, A2 psi_1, A2 psi_2, A2) in scan order
  const int4* __restrict__ gdof;    // analytic: dof bases in scan order
  const double* __restrict__ gcsum; // analytic: per cell, the sum of its elements' A2 (scan order)
  // analytic: the dof bases (columns) on the same cells, by their position
  const int* __restrict__ cstart;   // [ncell + 1]
  const int* __restrict__ cid;      // dof base of each slot
  const double4* __restrict__ cpos; // (x, y, H, H present): H = sum over the incident active elements n of
                                    // A2_n psi_n[corner], the column's factor when all its elements are full partners
};

__global__ void k_grid_gather(Params P, const int* __restrict__ items, int n, int4* gel, double2* gctr, double* grad,
                              double4* gft, int4* gdof) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int l = items[j];
  gel[j] = P.elem[l];
  gctr[j] = P.ctr[l];
  grad[j] = P.rad[l];
  if (gft) {  // analytic: the partners' factors and dofs in scan order
    gft[j] = P.ftab[l];
    gdof[j] = P.dofs[l];
  }
}

// analytic: the summed A2 of each cell's elements, in scan order (one thread per cell)
__global__ void k_cell_sums(const int* __restrict__ start, int ncell, const double4* __restrict__ gft, double* csum) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  double sacc = 0.0;
  for (int j = start[c]; j < start[c + 1]; ++j) sacc += gft[j].w;
  csum[c] = sacc;
}

__global__ void k_cell(Params P, Grid G, unsigned* key, int* val) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P.K) return;
  const int4 e = P.elem[k];
  unsigned cell = (unsigned)(G.nx * G.ny);
  if ((e.w & 15) != 0) {
    const double2 c = P.ctr[k];
    int ix = (int)floor((c.x - G.ox) / G.cs), iy = (int)floor((c.y - G.oy) / G.cs);
    ix = min(max(ix, 0), G.nx - 1);
    iy = min(max(iy, 0), G.ny - 1);
    cell = (unsigned)(iy * G.nx + ix);
  }
  key[k] = cell;
  val[k] = k;
}

// analytic rows: each dof base's position (a corner of an incident element),
// its factor H (sum over the incident active elements, fixed order) and cell
__global__ void k_col_keys(Params P, Grid G, const int* __restrict__ de_start, const int* __restrict__ de_items,
                           int nb, unsigned* key, int* val, double4* cpos) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double h = 0.0, px = 0.0, py = 0.0;
  bool any = false, pres = false;
  for (int i = de_start[b]; i < de_start[b + 1]; ++i) {
    const int it = de_items[i], n = it >> 2, a = it & 3;
    const int4 el = P.elem[n];
    if (!any) {
      const double2 v = P.vtx[a == 0 ? el.x : (a == 1 ? el.y : el.z)];
      px = v.x;
      py = v.y;
      any = true;
    }
    if ((el.w & 15) == 0) continue;
    const double4 f = P.ftab[n];
    const double fa = a == 0 ? f.x : (a == 1 ? f.y : f.z);
    h += fa;
    pres |= fa != 0.0;
  }
  unsigned cell = (unsigned)(G.nx * G.ny);
  if (any) {
    int ix = (int)floor((px - G.ox) / G.cs), iy = (int)floor((py - G.oy) / G.cs);
    ix = min(max(ix, 0), G.nx - 1);
    iy = min(max(iy, 0), G.ny - 1);
    cell = (unsigned)(iy * G.nx + ix);
  }
  key[b] = cell;
  val[b] = b;
  cpos[b] = make_double4(px, py, h, pres ? 1.0 : 0.0);
}

__global__ void k_col_gather(const int* __restrict__ ids, int n, const double4* __restrict__ cpos_by_id, double4* cpos) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) cpos[j] = cpos_by_id[ids[j]];
}

__global__ void k_cell_ranges(const unsigned* __restrict__ skey, int K, int ncell, int* start) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > ncell) return;
  int lo = 0, hi = K;  // lower_bound
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (skey[mid] < (unsigned)c) lo = mid + 1; else hi = mid;
  }
  start[c] = lo;
}

// (dof base, element * 4 + local vertex) of every element corner
__global__ void k_dof_keys(Params P, unsigned* key, int* val) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 3LL * P.K) return;
  const int e = (int)(i / 3), a = (int)(i % 3);
  const int4 d = P.dofs[e];
  key[i] = (unsigned)(a == 0 ? d.x : (a == 1 ? d.y : d.z));
  val[i] = e * 4 + a;
}

// ---------------------------------------------------------------- batch marking
__device__ __forceinline__ bool row_in(const Params& P, long long base) {
  // any component row nc*base + c in [row_lo, row_hi)
  const long long r0 = (long long)P.nc * base;
  return r0 + P.nc - 1 >= P.row_lo && r0 < P.row_hi;
}

__global__ void k_mark_a(Params P, unsigned char* needA) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P.K) return;
  const int4 d = P.dofs[k];
  needA[k] = row_in(P, d.x) || row_in(P, d.y) || row_in(P, d.z);
}

__global__ void k_mark_vertices(Params P, const unsigned char* needA, unsigned char* vmark) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P.K || !needA[k]) return;
  const int4 e = P.elem[k];
  vmark[e.x] = 1;
  vmark[e.y] = 1;
  vmark[e.z] = 1;
}

// root flag: outer element that emits its own rows (A) or may own a singular
// pair reaching the range (touches an A element, path 2 only)
__global__ void k_mark_roots(Params P, const unsigned char* needA, const unsigned char* vmark,
                             int* flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P.K) return;
  const int4 e = P.elem[k];
  bool f = false;
  if (e.w & 16) {
    f = needA[k];
    if (!f && P.path == 2 && vmark) f = vmark[e.x] || vmark[e.y] || vmark[e.z];
  }
  flag[k] = f;
}

// ---------------------------------------------------------------- candidates
// Each unordered non-singular pair {k, l} is integrated ONCE: the two
// directed halves (outer k / inner l clipped, and the reverse) serve both the
// reference's visit (k, l) of root k and its visit (l, k) of root l.  A pair
// record is (k, l | emitA << 30 | emitB << 31): side A = visit (k, l) (rows of
// k), side B = visit (l, k) (rows of l).  The record is produced by the
// smaller root of the batch when both visits exist with the same category
// ("shared"); otherwise root k produces a solo record (side A only).  The
// reject/full predicates are evaluated in each visit's own operand order
// ((dist - r_root) - r_nb, _engine.py:224, :227) so rounding ties never
// differ from the reference.
constexpr int kEmitA = 1 << 30;
constexpr int kEmitB = (int)(1u << 31);
constexpr int kIdMask = (1 << 30) - 1;

constexpr int kFixBits = 72;  // bound x 2^S = 2^72: 2^23 contributions per cell below 2^95
// Fixed point: t = rint(v 2^S), |t| <= 2^72, summed exactly as a 96-bit two's
// complement integer (three 32-bit limbs in shared memory -- native 32-bit
// atomics; 64-bit shared atomics are CAS loops -- with the carries propagated
// by the adding thread; __int128 in registers), so a sum does not depend on
// the order of its terms.  (The bound can exceed the largest term by a few
// powers of two -- the analytic own terms -- so the resolution 2^-72 of the
// bound keeps ~2^-60 of every row's entries.)
using fix_t = __int128;
__device__ __forceinline__ fix_t fix_of(double v, double scale) {
  const double t = rint(v * scale);
  const double hd = floor(t * 0x1p-40);
  const long long h = __double2ll_rz(hd);
  const long long l = __double2ll_rz(fma(hd, -0x1p40, t));  // exact: t and hd 2^40 share the grid of t
  return ((fix_t)h << 40) + (fix_t)l;
}
__device__ __forceinline__ double fix_val3(const unsigned* c, double inv) {
  const double v = fma((double)(int)c[2], 0x1p64, fma((double)c[1], 0x1p32, (double)c[0]));
  return v * inv;
}
__device__ __forceinline__ void fix_atomic(unsigned* c, fix_t x) {
  unsigned x0 = (unsigned)x, x1 = (unsigned)(x >> 32), x2 = (unsigned)(x >> 64);
  if (x0) {
    const unsigned o = atomicAdd(&c[0], x0);
    if (o + x0 < o && ++x1 == 0) ++x2;
  }
  if (x1) {
    const unsigned o = atomicAdd(&c[1], x1);
    if (o + x1 < o) ++x2;
  }
  if (x2) atomicAdd(&c[2], x2);
}
// Sum over a group of lanes of 96-bit two's complement values (exact, so mod
// 2^96): four 24-bit limbs, each summed by one warp reduction (32 x 2^24 <
// 2^32), recombined with their carries.  Every lane of the group gets the total.
__device__ __forceinline__ fix_t fix_group_sum(unsigned mask, fix_t a) {  // (called by exactly the lanes of mask)
  const unsigned long long lo = (unsigned long long)a;
  const unsigned hi = (unsigned)(a >> 64);
  const unsigned s0 = __reduce_add_sync(mask, (unsigned)lo & 0xffffffu);
  const unsigned s1 = __reduce_add_sync(mask, (unsigned)(lo >> 24) & 0xffffffu);
  const unsigned s2 = __reduce_add_sync(mask, ((unsigned)(lo >> 48) | (hi << 16)) & 0xffffffu);
  const unsigned s3 = __reduce_add_sync(mask, hi >> 8);
  unsigned __int128 r = (unsigned __int128)s0 + ((unsigned __int128)s1 << 24) + ((unsigned __int128)s2 << 48) +
                        ((unsigned __int128)s3 << 72);
  r <<= 32;  // drop the bits above 96, then sign-extend
  return (fix_t)r >> 32;
}
// The 7 rule points of a triangle (reference arithmetic, as rule_points).
__device__ __forceinline__ void tri_points(const double* tx, const double* ty, double* px, double* py) {
  const double e1x = tx[1] - tx[0], e2x = tx[2] - tx[0], e1y = ty[1] - ty[0], e2y = ty[2] - ty[0];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    px[p] = __dadd_rn(__dadd_rn(tx[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
    py[p] = __dadd_rn(__dadd_rn(ty[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
  }
}

// Every vertex of l inside the widened ball of every outer point of k, and
// vice versa: both sweeps' clips return the whole inner triangle
// (_geom_scalar.py:53-66).  Symmetric in (k, l); exact reference predicates.
__device__ __forceinline__ bool pair_all_in(const Params& P, const double* kx, const double* ky, const double* xk,
                                            const double* yk, const double* lx, const double* ly, const double* xl,
                                            const double* yl) {
  const double rad = mul(P.delta, 1.0 + kBallTieRel);
  const double r2 = mul(rad, rad);
  // The rule points are convex combinations of the vertices, and the
  // distance to a point is convex: the 9 vertex-vertex distances decide the
  // 42 reference tests except within a relative 1e-10 of the radius (the
  // rule points' rounding is ~1e-16).  Only such near-ties run the exact tests.
  {
    const double hi = r2 * (1.0 + 1e-10), lo = r2 * (1.0 - 1e-10);
    bool clear = true;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double d2 = sumsq(lx[i] - kx[a], ly[i] - ky[a]);
        if (d2 > hi) return false;
        clear = clear && d2 < lo;
      }
    if (clear) return true;
  }
  // the vertex points (p = 1..3) first: a pair that fails usually fails there
#pragma unroll 1
  for (int q = 0; q < 7; ++q) {
    const int p = q < 6 ? q + 1 : 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (__dsub_rn(sumsq(lx[i] - xk[p], ly[i] - yk[p]), r2) > 0.0) return false;
      if (__dsub_rn(sumsq(kx[i] - xl[p], ky[i] - yl[p]), r2) > 0.0) return false;
    }
  }
  return true;
}

// Truncation class of a clipped pair, in two parts with the reference's
// exact predicates: "inside" -- every inner vertex inside the widened ball of
// every outer point, both ways (the clips return the triangles themselves,
// _geom_scalar.py:53-66) -- and "far" -- the inner element's bounding disk
// beyond the ball of every outer point by a margin no rounding can bridge
// (every clip is empty).  Out of line: only pairs near the ball's rim get here.
__device__ __noinline__ bool pair_inside(const Params& P, const double* kx, const double* ky, const double* xk,
                                         const double* yk, const double* lx, const double* ly) {
  if (P.ball == 2) return false;
  const double rad = mul(P.delta, 1.0 + kBallTieRel);
  const double r2 = mul(rad, rad), hi = r2 * (1.0 + 1e-10), lo = r2 * (1.0 - 1e-10);
  bool clear = true;  // (see pair_all_in: the vertex distances decide all but near-ties)
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double d2 = sumsq(lx[i] - kx[a], ly[i] - ky[a]);
      if (d2 > hi) return false;
      clear = clear && d2 < lo;
    }
  if (clear) return true;
  double xl[7], yl[7];
  tri_points(lx, ly, xl, yl);
  return pair_all_in(P, kx, ky, xk, yk, lx, ly, xl, yl);
}

__device__ __noinline__ bool pair_far(const Params& P, const double* xk, const double* yk, double2 ck, double rk,
                                      const double* lx, const double* ly, double2 cl, double rl) {
  if (P.ball == 2) return false;
  {
    // every rule point of k lies within r_k of c_k (and of l within r_l of
    // c_l): the barycentre distance decides "all far" outside a band of width
    // 2 min(r_k, r_l) (margins 1e-9 relative cover the roundings)
    const double d2 = (cl.x - ck.x) * (cl.x - ck.x) + (cl.y - ck.y) * (cl.y - ck.y);
    const double fo = P.delta * (1.0 + 1e-6) + rl + rk, fi = P.delta * (1.0 + 1e-6) + rl - rk;
    const double gi = P.delta * (1.0 + 1e-6) + rk - rl;
    if (d2 > fo * fo * (1.0 + 1e-9)) return true;
    if ((fi > 0.0 && d2 < fi * fi * (1.0 - 1e-9)) || (gi > 0.0 && d2 < gi * gi * (1.0 - 1e-9))) return false;
  }
  const double far2k = (P.delta * (1.0 + 1e-6) + rk) * (P.delta * (1.0 + 1e-6) + rk);
  const double far2l = (P.delta * (1.0 + 1e-6) + rl) * (P.delta * (1.0 + 1e-6) + rl);
  double xl[7], yl[7];
  tri_points(lx, ly, xl, yl);
  bool all_far = true;
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    // outer point on k, inner l / outer point on l, inner k
    const double dkx = cl.x - xk[p], dky = cl.y - yk[p];
    const double dlx = ck.x - xl[p], dly = ck.y - yl[p];
    all_far = all_far && dkx * dkx + dky * dky > far2l && dlx * dlx + dly * dly > far2k;
  }
  return all_far;
}

// pair_all_in of root k (vertices, rule points) and element el, out of line
// (rare: only pairs within the ball's rim reach it)
__device__ __noinline__ bool pair_all_in_el(const Params& P, const double* kx, const double* ky, const double* xk,
                                            const double* yk, int4 el) {
  double lx[3], ly[3], xl[7], yl[7];
  const double2 v0 = __ldg(&P.vtx[el.x]), v1 = __ldg(&P.vtx[el.y]), v2 = __ldg(&P.vtx[el.z]);
  lx[0] = v0.x; ly[0] = v0.y; lx[1] = v1.x; ly[1] = v1.y; lx[2] = v2.x; ly[2] = v2.y;
  tri_points(lx, ly, xl, yl);
  return pair_all_in(P, kx, ky, xk, yk, lx, ly, xl, yl);
}

// Distance predicates of a visit in the reference's operand order
// (_engine.py:219-227): reject  (dist - r_root) - r_nb > prer  and
// full  (dist + r_root) + r_nb <= delta, with dist = sqrt(d2).  Pairs far
// from either threshold are decided from d2 alone -- a relative margin of
// 1e-12 dwarfs every rounding of the thresholds -- so the square root (and
// the exact test) only runs in thin shells around them.
struct VisitDist {
  double d2, dist;
  __device__ __forceinline__ explicit VisitDist(double d2_) : d2(d2_), dist(-1.0) {}
  __device__ __forceinline__ double get() {
    if (dist < 0.0) dist = sqrt(d2);
    return dist;
  }
  // (get() - a) - b > t
  __device__ __forceinline__ bool reject(double a, double b, double t) {
    const double th = t + a + b, eta = 1e-12 * th;
    if (d2 > (th + eta) * (th + eta)) return true;
    if (d2 < (th - eta) * (th - eta)) return false;
    return __dsub_rn(__dsub_rn(get(), a), b) > t;
  }
  // (get() + a) + b <= t
  __device__ __forceinline__ bool within(double a, double b, double t) {
    const double th = t - a - b, eta = 1e-12 * (t + a + b);
    if (th - eta > 0.0 && d2 < (th - eta) * (th - eta)) return true;
    if (th + eta <= 0.0 || d2 > (th + eta) * (th + eta)) return false;
    return __dadd_rn(__dadd_rn(get(), a), b) <= t;
  }
};

//  -1 none here, 0 full record, 1 clipped record, 2/3/4 singular id/edge/vertex.
// *visited: the reference would count the visit (k, l) (EPI); *flags: record sides.
// Clipped pairs whose every sweep item is untruncated take the full path (same
// arithmetic: the fan of the untruncated triangle is the triangle); pairs
// whose every item is empty contribute nothing and produce no record.
// Analytic mode (P.analytic): a visit of category 0 ("full", by distance or
// by truncation class) has no record at all -- the row merge enumerates such
// visits itself (k_row_asm) -- and *an reports it (the fill pass sums the
// partners' areas of the root's own block).
template <bool LIGHT>
__device__ __forceinline__ int classify(const Params& P, int k, int4 ek, double2 ck, double rk,
                                        const double* kx, const double* ky, const double* xk, const double* yk,
                                        bool needAk, const unsigned char* __restrict__ needA,
                                        const int* __restrict__ inR, int l, int4 el, double2 cl, double rl,
                                        bool& visited, int& flags, bool& an) {
  visited = false;
  flags = 0;
  an = false;
  VisitDist D(sumsq(ck.x - cl.x, ck.y - cl.y));
  // a shared vertex lies within r of both barycentres: dist <= r_k + r_l
  const double rs = (rk + rl) * (1.0 + 1e-9);
  const int ns = D.d2 > rs * rs ? 0
                                : (ek.x == el.x) + (ek.x == el.y) + (ek.x == el.z) + (ek.y == el.x) + (ek.y == el.y) +
                                      (ek.y == el.z) + (ek.z == el.x) + (ek.z == el.y) + (ek.z == el.z);
  const bool touching = (k == l) || ns > 0;
  if (!touching && D.reject(rk, rl, P.prer)) return -1;
  visited = true;
  if (touching && P.path == 2) {
    if (l != k && (el.w & 16) && l < k) return -1;  // owned by the smaller root (_engine.py:233)
    if (!(needAk || needA[l])) return -1;
    return k == l ? 2 : (ns == 2 ? 3 : 4);
  }
  const bool full = D.within(rk, rl, P.delta);
  const bool lroot = k != l && (el.w & 16);
  bool full_lk = full, rej_lk = false;
  if (lroot) {  // root l's view of the same pair
    rej_lk = !touching && D.reject(rl, rk, P.prer);
    full_lk = D.within(rl, rk, P.delta);
  }
  if (P.analytic) {
    // records only for category-1 visits; category 0 = full or all-inside
    if (k == l) {
      if (LIGHT) return needAk ? 1 : -1;
    } else if (full) {
      an = true;  // (a clipped visit (l, k) is root l's own record)
      return -1;
    } else if (LIGHT) {
      // an upper bound: possibly clipped, and not the shared record root l makes
      if (!full_lk && lroot && !rej_lk && l < k && inR[l] >= 0) return -1;
      if (!(needAk || (lroot && needA[l]))) return -1;
      return 1;
    }
  }
  // When both views agree on `full`, both get the same category whatever the
  // truncation class, so whether the pair is shared -- and then produced by
  // the smaller root of the batch -- is known before the (costly) class.
  const bool l_makes = full == full_lk && lroot && !rej_lk && l < k && inR[l] >= 0;
  if (l_makes && !P.analytic) return -1;
  if (LIGHT) {  // upper bounds for the count pass: 0 full, 1 possibly clipped
    if (!(needAk || (lroot && needA[l]))) return -1;
    return full ? 0 : 1;
  }
  // exact truncation class of the pair (symmetric in k, l): "inside" now,
  // "far" only if this root would make the record
  const bool lgeom = k != l && (!full || !full_lk) && P.ball != 2;
  double lx[3], ly[3];
  bool tin = false;
  if (lgeom) {
    const double2 a = __ldg(&P.vtx[el.x]), b = __ldg(&P.vtx[el.y]), c = __ldg(&P.vtx[el.z]);
    lx[0] = a.x; ly[0] = a.y; lx[1] = b.x; ly[1] = b.y; lx[2] = c.x; ly[2] = c.y;
    tin = pair_inside(P, kx, ky, xk, yk, lx, ly);
  }
  // (analytic mode: the identical pair keeps its stored blocks on the clipped path)
  const int cat_kl = (full || tin) && !(P.analytic && k == l) ? 0 : 1;
  if (P.analytic) {
    if (cat_kl == 0) {
      an = true;
      return -1;
    }
    if (l_makes) return -1;
  }
  // every item empty in both visits: nothing to emit
  if (lgeom && !tin && pair_far(P, xk, yk, ck, rk, lx, ly, cl, rl)) return -1;
  bool shared = false;
  if (lroot) {
    const int cat_lk = full_lk || tin ? 0 : 1;
    shared = !rej_lk && cat_lk == cat_kl;
  }
  if (shared && inR[l] >= 0 && l < k) return -1;  // root l produces the record
  const bool emitB = shared && needA[l];
  if (!needAk && !emitB) return -1;
  flags = (needAk ? kEmitA : 0) | (emitB ? kEmitB : 0);
  return cat_kl;
}

// count pass (FILL = false): exact singular counts, an upper bound of the
// non-singular records per root (column C_FULL) and the EPI; fill pass:
// records into the root's upper-bound range of `comb` (k | clipped << 30),
// singular pairs into their lists, and the actual full / clipped counts.
constexpr int kCatClip = 1 << 30;

template <bool FILL>
__global__ void __launch_bounds__(256, 3) k_candidates(Params P, Grid G, const int* __restrict__ roots, int nR,
                             const unsigned char* __restrict__ needA, const int* __restrict__ inR,
                             int* __restrict__ cnt, const long long* __restrict__ off, int2* __restrict__ comb,
                             int2* __restrict__ ls0, int2* __restrict__ ls1, int2* __restrict__ ls2,
                             int stride = 1, double* __restrict__ own_a2 = nullptr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  for (long long i0 = (long long)warp * stride; i0 < nR; i0 += (long long)nwarps * stride) {
    const int i = (int)i0;
    const int k = roots[i];
    const int4 ek = P.elem[k];
    const double2 ck = P.ctr[k];
    const double rk = P.rad[k];
    const bool needAk = needA[k];
    double kx[3], ky[3], xk[7], yk[7];
    if (FILL) {
      load_tri(P, k, kx, ky);
      rule_points(P, kx, ky, xk, yk);
    }
    // candidate cells: those within G.reach of the root's barycentre (the
    // grid pitch is half the reach: ~half the candidates of a 3x3 block of
    // reach-sized cells)
    int iy = (int)floor((ck.y - G.oy) / G.cs);
    iy = min(max(iy, 0), G.ny - 1);
    int ix = (int)floor((ck.x - G.ox) / G.cs);
    ix = min(max(ix, 0), G.nx - 1);
    // surely-full radius: dist <= rho  =>  (dist + r_k) + r_l <= delta for every r_l <= r_max
    const double rho = P.delta - rk - G.rmax - 1e-9 * (P.delta + G.rmax) - 2.0 * G.cs * 1e-9;
    int c[7] = {0, 0, 0, 0, 0, 0, 0};
    long long base[4];
    int2* lists[4] = {comb, ls0, ls1, ls2};
    if (FILL) {
      base[0] = off[(long long)C_FULL * (nR + 1) + i];
      for (int j = 1; j < 4; ++j) base[j] = off[(long long)(C_SID + j - 1) * (nR + 1) + i];
    }
    int nfull = 0, nclip = 0;
    // analytic fill: sum of the category-0 partners' areas A2 (per lane in
    // scan order, then a fixed tree: the same for every batch containing k)
    double own = 0.0;
    for (int yy = max(iy - G.span, 0); yy <= min(iy + G.span, G.ny - 1); ++yy) {
      const double ylo = G.oy + yy * G.cs, yhi = ylo + G.cs;
      const double dy = ck.y < ylo ? ylo - ck.y : (ck.y > yhi ? ck.y - yhi : 0.0);
      if (dy > G.reach) continue;
      const double hw = sqrt(G.reach * G.reach - dy * dy);
      const int x0 = max((int)floor((ck.x - hw - G.ox) / G.cs), 0);
      const int x1 = min((int)floor((ck.x + hw - G.ox) / G.cs), G.nx - 1);
      if (x0 > x1) continue;
      const int c0 = G.start[yy * G.nx + x0];
      const int c1 = G.start[yy * G.nx + x1 + 1];
      // analytic: cells that lie wholly within rho of the barycentre hold
      // only full partners (dist + r_k + r_l <= delta with room to spare):
      // they are counted, and their areas summed, cell by cell -- no
      // candidate test.  The root's own cell is scanned (the pair (k, k)).
      int seg_lo[3] = {c0, c1, c1}, seg_hi[3] = {c1, c1, c1};
      if (P.analytic && rho > 0.0) {
        const double dym = fmax(fabs(ylo - ck.y), fabs(yhi - ck.y));
        if (dym < rho) {
          const double hwd = sqrt(rho * rho - dym * dym);
          const int xa = max((int)ceil((ck.x - hwd - G.ox) / G.cs), x0);
          const int xb = min((int)floor((ck.x + hwd - G.ox) / G.cs) - 1, x1);
          if (xa <= xb) {
            // deep cells [xa, xb], minus the root's own cell
            int ra[2] = {xa, 0}, rb[2] = {xb, -1};
            if (yy == iy && ix >= xa && ix <= xb) {
              rb[0] = ix - 1;
              ra[1] = ix + 1;
              rb[1] = xb;
            }
            int ns = 0, cur = c0;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              if (ra[q] > rb[q]) continue;
              const int da = G.start[yy * G.nx + ra[q]], db = G.start[yy * G.nx + rb[q] + 1];
              seg_lo[ns] = cur;
              seg_hi[ns] = da;
              ++ns;
              cur = db;
              if (!FILL) {
                if (lane == 0) c[C_EPI] += db - da;
              } else {
                for (int cx = ra[q] + lane; cx <= rb[q]; cx += 32) own += G.gcsum[yy * G.nx + cx];
              }
            }
            seg_lo[ns] = cur;
            seg_hi[ns] = c1;
          }
        }
      }
#pragma unroll 1
      for (int sg = 0; sg < 3; ++sg)
      for (int j0 = seg_lo[sg]; j0 < seg_hi[sg]; j0 += 32) {
        const int c1 = seg_hi[sg];
        const int j = j0 + lane;
        int cat = -1, fl = 0;
        bool vis = false, an = false;
        const int l = j < c1 ? G.items[j] : 0;
        int4 el = make_int4(0, 0, 0, 0);
        double2 cl = make_double2(0.0, 0.0);
        double rl = 0.0, a2l = 0.0;
        if (j < c1) {
          el = G.gel[j];
          cl = G.gctr[j];
          rl = G.grad[j];
          if (FILL && P.analytic) a2l = __ldg(&G.gft[j].w);
        }
        if (!FILL) {
          if (j < c1) cat = classify<true>(P, k, ek, ck, rk, kx, ky, xk, yk, needAk, needA, inR, l, el, cl, rl, vis, fl, an);
          c[C_EPI] += vis;
          // C_FULL: all records, C_PART: the possibly clipped ones
          if (cat >= 0) {
            if (cat <= 1) { c[C_FULL]++; c[C_PART] += cat; } else c[cat]++;
          }
        } else {
          if (j < c1) cat = classify<false>(P, k, ek, ck, rk, kx, ky, xk, yk, needAk, needA, inR, l, el, cl, rl, vis, fl, an);
          if (an) own += a2l;
          nfull += cat == 0;
          nclip += cat == 1;
          // lists: 0 = combined (full or clipped), 1..3 = singular families
          const int q0 = cat < 0 ? -1 : (cat <= 1 ? 0 : cat - 1);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const unsigned m = __ballot_sync(0xffffffffu, q0 == q);
            if (q0 == q) {
              // canonical orientation: a pair record is always (smaller,
              // larger) element -- its blocks are then computed identically
              // whichever root (and batch, and GPU) produces it, and the row
              // split cannot change a value.  A root's own visit of a smaller
              // partner becomes the record's side B.
              int2 rec = make_int2(k | (cat == 1 ? kCatClip : 0), l | fl);
              if (q == 0 && l < k && !(P.dbg & 32))  // (NLG_DEBUG & 32: A/B only)
                rec = make_int2(l | (cat == 1 ? kCatClip : 0),
                                k | ((fl & kEmitA) ? kEmitB : 0) | ((fl & kEmitB) ? kEmitA : 0));
              lists[q][base[q] + __popc(m & lt)] = rec;
            }
            base[q] += __popc(m);
          }
        }
      }
    }
    if (!FILL) {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        int v = c[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        c[q] = v;
      }
      if (lane == 0) {
        for (int q = 0; q < 6; ++q) cnt[(long long)q * nR + i] = c[q];
        // does this root own the batch's count of its pairs (EPI home rule)?
        const int4 d = P.dofs[k];
        const long long rmin = (long long)P.nc * min(d.x, min(d.y, d.z));
        cnt[(long long)C_KK * nR + i] = needAk ? ((rmin >= P.row_lo && rmin < P.row_hi) ? 2 : 1) : 0;
      }
    } else {
      for (int o = 16; o; o >>= 1) {
        nfull += __shfl_xor_sync(0xffffffffu, nfull, o);
        nclip += __shfl_xor_sync(0xffffffffu, nclip, o);
      }
      if (P.analytic)
        for (int o = 16; o; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
      if (lane == 0) {
        cnt[(long long)C_FULL * nR + i] = nfull;
        cnt[(long long)C_PART * nR + i] = nclip;
        if (P.analytic) own_a2[i] = own;
      }
    }
  }
}

// per-row cost of a batch attempt that does not fit (batch planning): each
// root's memory (bytes), record and COO-slot counts go to its first in-range row
__global__ void k_root_cost(Params P, const int* __restrict__ roots, int nR, const int* __restrict__ cnt,
                            double rec_bytes, double store_bytes, double sing_bytes, double root_bytes, double rec_slots,
                            double sing_slots, unsigned long long* row_cost, double scale, double epi_bytes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nR) return;
  const int4 d = P.dofs[roots[i]];
  const int da[3] = {d.x, d.y, d.z};
  long long home = -1;
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < P.nc; ++c) {
      const long long r = (long long)P.nc * da[a] + c;
      if (r >= P.row_lo && r < P.row_hi && (home < 0 || r < home)) home = r;
    }
  if (home < 0) home = P.row_lo;
  const long long rec = cnt[(long long)C_FULL * nR + i];
  const long long stored = P.analytic ? cnt[(long long)C_PART * nR + i] : rec;
  const long long sing = (long long)cnt[(long long)C_SID * nR + i] + cnt[(long long)C_SED * nR + i] +
                         cnt[(long long)C_SVX * nR + i];
  unsigned long long* rc = row_cost + 3 * (home - P.row_lo);
  const long long epi = cnt[(long long)C_EPI * nR + i];
  atomicAdd(&rc[0], (unsigned long long)(scale * (rec * rec_bytes + stored * store_bytes + sing * sing_bytes + root_bytes +
                                                  epi * epi_bytes)));
  atomicAdd(&rc[1], (unsigned long long)(scale * rec));
  atomicAdd(&rc[2], (unsigned long long)(scale * (rec * rec_slots + sing * sing_slots + 9 * P.nc * P.nc)));
}


// per dof base: the EPI of every outer root incident to it (shard balancing)
__global__ void k_base_work(Params P, const int* __restrict__ roots, int nR, const int* __restrict__ cnt,
                            unsigned long long* work) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nR) return;
  const int4 d = P.dofs[roots[i]];
  const unsigned long long e = (unsigned long long)cnt[(long long)C_EPI * nR + i];
  atomicAdd(&work[d.x], e);
  atomicAdd(&work[d.y], e);
  atomicAdd(&work[d.z], e);
}

// sum of the visits (EPI) and count of the roots whose home row is in the batch
__global__ void k_epi_home(const int* __restrict__ cnt, int nR, unsigned long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long e = 0, r = 0;
  if (i < nR && cnt[(long long)C_KK * nR + i] == 2) {
    e = (unsigned long long)cnt[(long long)C_EPI * nR + i];
    r = 1;
  }
  for (int o = 16; o; o >>= 1) {
    e += __shfl_xor_sync(0xffffffffu, e, o);
    r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  if (lane_id() == 0 && r) {
    atomicAdd(&out[0], e);
    atomicAdd(&out[1], r);
  }
}

// per-root compaction of the fill's records (contiguous at the start of each
// root's upper-bound range, full and clipped interleaved in candidate order)
// into the full and clipped lists at the roots' exact offsets: one warp per
// root, list order preserved
__global__ void k_split_records(const int2* __restrict__ comb, const long long* __restrict__ ub_off,
                                const long long* __restrict__ foff, const long long* __restrict__ poff,
                                const int* __restrict__ cnt, int nR, int2* lf, int2* lp) {
  const int i = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  if (i >= nR) return;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  const int n = cnt[(long long)C_FULL * nR + i] + cnt[(long long)C_PART * nR + i];
  const int2* src = comb + ub_off[i];
  int2* fd = lf + foff[i];
  int2* pd = lp + poff[i];
  int fp = 0, pp = 0;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    const bool valid = j < n;
    const int2 r = valid ? src[j] : make_int2(0, 0);
    const bool clip = valid && (r.x & kCatClip);
    const unsigned mf = __ballot_sync(0xffffffffu, valid && !clip), mp = __ballot_sync(0xffffffffu, clip);
    if (valid && !clip) fd[fp + __popc(mf & lt)] = r;
    if (clip) pd[pp + __popc(mp & lt)] = r;
    fp += __popc(mf);
    pp += __popc(mp);
  }
}

__global__ void k_rank(const int* __restrict__ roots, int nR, int* inR) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nR) inR[roots[i]] = i;
}

// reverse index of side-B records: key = rank of the partner root (nR = none)
__global__ void k_rev_keys(const int2* __restrict__ rec, long long n, const int* __restrict__ inR, int nR,
                           unsigned* key, int* val) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 r = rec[i];
  key[i] = (r.y & kEmitB) ? (unsigned)inR[r.y & kIdMask] : (unsigned)nR;
  val[i] = (int)i;
}

// position of each record in the reverse order (its side B block goes there)
// and, for the emitted ones, the record's root (the partner of side B)
__global__ void k_rev_pos(const int* __restrict__ rev_item, long long n, const int2* __restrict__ rec, int* revpos,
                          int* partB) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = rev_item[i];
  revpos[r] = (int)i;
  partB[i] = rec[r].x & kIdMask;
}

template <typename KT> __host__ __device__ constexpr KT key_sentinel() { return (KT)~(KT)0; }

// ---------------------------------------------------------------- visits
__device__ __forceinline__ unsigned long long coo_key(const Params& P, long long row, long long col) {
  if (row < P.row_lo || row >= P.row_hi) return kSentinel;
  return (unsigned long long)(row - P.row_lo) * (unsigned long long)P.J + (unsigned long long)col;
}
// COO key store: 32-bit when the batch's keys fit (the radix sort then reads
// half the key bytes), the sentinel truncating to the 32-bit sentinel
__device__ __forceinline__ void put_key(const Params& P, unsigned long long* keys, long long slot,
                                        unsigned long long k) {
  if (P.narrow) reinterpret_cast<unsigned*>(keys)[slot] = (unsigned)k;
  else keys[slot] = k;
}
// reference emits a triplet iff v != 0 (_engine.py:410-424); an absent
// entry is stored as +0.0, a present one that is exactly zero as -0.0
__device__ __forceinline__ double emit_val(double v) { return v != 0.0 ? v : 0.0; }

// inf/nan <=> all exponent bits set; checked with integer ops, reported once
__device__ __forceinline__ bool nonfinite(double v) {
  return ((unsigned long long)__double_as_longlong(v) & 0x7ff0000000000000ull) == 0x7ff0000000000000ull;
}
// errpair[0]: lexicographically smallest (root, partner) -- the reference's
// first failing visit under "brute" traversal (roots ascending, partners
// ascending, _engine.py:483-490); errpair[1]: smallest root whose visit of
// itself failed -- under "bfs" the root's own pair is its first visit
// (_engine.py:545-560), so the host reports (k, k) when k == errpair[1]
__device__ __forceinline__ void report_nonfinite(bool bad, int k, int l, int K, unsigned long long* errpair) {
  if (bad) {
    atomicMin(errpair, (unsigned long long)k * (unsigned long long)K + l);
    if (k == l) atomicMin(errpair + 1, (unsigned long long)k);
  }
}


template <typename T>
__device__ __forceinline__ void warp_add_ll(T v, unsigned long long* dst) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane_id() == 0 && v) atomicAdd(dst, (unsigned long long)v);
}

struct VisitOut {
  double* kkv;              // [record][side][NKK] own blocks of visit A (k, l) / B (l, k), symmetric: I <= J
  double* klv;              // [record][side][I][NVP] neighbour blocks, row-major and padded
  long long a_base;         // side A of list record v -> block a_base + v
  long long b_base;         // side B -> block b_base + revpos[v] (reverse-index order)
  const int* revpos;
  long long nlist;
  unsigned long long* counters;
  unsigned long long* errpair;
  unsigned long long* vmax;  // max |value| written (bits of a nonnegative double), for the merge's fixed point
  unsigned long long* emax;  // [K] per element: max |value| of the emitted sides of its visits (root), as bits
};

// A root's bound for the merge's fixed-point scale: the largest |value| of
// its emitted record sides.  A root's sides are the same whichever batch
// evaluates it, so the scale of each row -- from its incident elements'
// bounds -- and with it every sum does not depend on the row split.
__device__ __forceinline__ void elem_bound(unsigned long long* emax, int e, double m) {
  if (!(m > 0.0 && m <= 1e300)) return;
  const unsigned long long b = (unsigned long long)__double_as_longlong(m);
  // a root's records are processed side by side: read first, so that only
  // a new maximum (rare after the first records) pays for the atomic
  if (b > __ldcg(&emax[e])) atomicMax(&emax[e], b);
}

// max of nonnegative doubles (as bit patterns) over the warp, one atomic
__device__ __forceinline__ void warp_max_abs(double m, unsigned long long* dst) {
  unsigned long long b = (unsigned long long)__double_as_longlong(m == m ? m : 0.0);
  for (int o = 16; o; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  if (lane_id() == 0 && b) atomicMax(dst, b);
}

// per-record-side block layouts: the own block is symmetric (I <= J, packed
// in (I <= J) row-major order, presence = value != 0); the neighbour block is
// row-major (row I on the root, J = b nc + d on the neighbour), rows padded to
// 32 B for nc = 1, so one root row of the block is one sector (merge)
template <int NC> struct Blk {
  static constexpr int N3 = 3 * NC, E = 9 * NC * NC, NKK = N3 * (N3 + 1) / 2;
  static constexpr int NV = N3 * NC, NVP = NC == 1 ? 4 : N3, KLS = N3 * NVP;
  __host__ __device__ static constexpr int sym(int I, int J) { return I * N3 - I * (I - 1) / 2 + (J - I); }
  __host__ __device__ static constexpr int kl(int I, int J) { return I * NVP + J; }
};

// emit one side of a record: own block -> kkv, neighbour block -> klv
template <int NC>
__device__ __forceinline__ void emit_side(const Params& P, const VisitOut& O, long long slot, bool on,
                                          int root, int nb, const double* kk, const double* kl, double& vm) {
  using B = Blk<NC>;
  bool bad = false;
  double sm = 0.0;
#pragma unroll
  for (int e = 0; e < B::E; ++e) {
    const int I = e / B::N3, J = e % B::N3;
    if (I <= J) O.kkv[slot * B::NKK + B::sym(I, J)] = on ? kk[e] : 0.0;
    bad |= nonfinite(kk[e]) | nonfinite(kl[e]);
    O.klv[slot * B::KLS + B::kl(I, J)] = on ? emit_val(kl[e]) : 0.0;
    if (on) sm = fmax(sm, fmax(fabs(kk[e]), fabs(kl[e])));
  }
  report_nonfinite(on && bad, root, nb, P.K, O.errpair);
  vm = fmax(vm, sm);
  if (on) elem_bound(O.emax, root, sm);
}

__device__ __forceinline__ double4 ld_f4(const double4* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Per-element factors of the analytic full pairs (Params::analytic).  For a
// full pair of the constant (f = c) or affine (f(x) = (1 + a x_1) b) kernel
// the visit (r, n) block of _engine._sweep (:46-185, both sweeps over the
// whole triangles) is, with A2 = twice the area and f at the 7 rule points,
//   kk[a,b] = 2 A2_r A2_n sw Phi_r[a,b],   Phi_r[a,b] = sum_p w_p H_pa H_pb f(x_p on r)
//   kl[a,b] = -2 A2_r whs_a (A2_n psi_n[b]), psi_n[b] = sum_q w_q H_qb f(y_q on n)
// (sw = sum w, whs_a = sum_p w_p H_pa): the partner enters only through
// A2_n and A2_n psi_n, so stage R sums those per root / neighbour dof.
// fmax: max |A2|, max |A2 psi_b|, max |Phi_ab| over the elements (bounds of
// the analytic terms for the merge's fixed-point scale)
template <int KID>
__global__ void k_elem_factors(Params P, double4* ft, unsigned long long* fbound) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
  if (e < P.K) {
    double tx[3], ty[3], px[7], py[7];
    load_tri(P, e, tx, ty);
    rule_points(P, tx, ty, px, py);
    double ps[3] = {0.0, 0.0, 0.0}, phi[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) phi[i] = 0.0;
#pragma unroll
    for (int p = 0; p < 7; ++p) {
      const double f = KID == 2 ? P.cst : (1.0 + P.kp0 * px[p]) * P.kp1;
      m3 = fmax(m3, fabs(f));  // (f is affine: its extremes on a triangle are at vertices, rule points 1-3)
#pragma unroll
      for (int a = 0; a < 3; ++a) ps[a] = fma(c_rule.wh[p][a], f, ps[a]);
#pragma unroll
      for (int i = 0; i < 9; ++i) phi[i] = fma(c_rule.whh[p][i], f, phi[i]);
    }
    const double a2 = twice_area(tx, ty);
    ft[e] = make_double4(a2 * ps[0], a2 * ps[1], a2 * ps[2], a2);
    m0 = fabs(a2);
    m1 = fmax(fabs(a2 * ps[0]), fmax(fabs(a2 * ps[1]), fabs(a2 * ps[2])));
#pragma unroll
    for (int i = 0; i < 9; ++i) m2 = fmax(m2, fabs(phi[i]));
  }
  warp_max_abs(m0, &fbound[0]);
  warp_max_abs(m1, &fbound[1]);
  warp_max_abs(m2, &fbound[2]);
  warp_max_abs(m3, &fbound[3]);
}

// Phi_r[a][b] of the root (see k_elem_factors)
template <int KID>
__device__ __forceinline__ double root_phi(const Params& P, int r, int a, int b) {
  double tx[3], ty[3], px[7], py[7];
  load_tri(P, r, tx, ty);
  rule_points(P, tx, ty, px, py);
  double v = 0.0;
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    const double f = KID == 2 ? P.cst : (1.0 + P.kp0 * px[p]) * P.kp1;
    v = fma(c_rule.whh[p][a * 3 + b], f, v);
  }
  return v;
}

// one side of a peridynamic full record from its unique components
// (full_pair_peri): own block c2 K, neighbour block -c2 G (side B: G transposed)
__device__ __forceinline__ void emit_peri(const Params& P, const VisitOut& O, long long slot, bool on, int root,
                                          int nb, double c2, const double (*K)[3], const double (*G)[3][3],
                                          bool transpose, double& vm) {
  using B = Blk<2>;
  bool bad = false;
  double sm = 0.0;
#pragma unroll
  for (int I = 0; I < 6; ++I)
#pragma unroll
    for (int J = 0; J < 6; ++J) {
      const int a = I >> 1, c = I & 1, b = J >> 1, d = J & 1, u = c + d;
      if (I <= J) {
        const double kk = c2 * K[sym3i(a, b)][u];
        O.kkv[slot * B::NKK + B::sym(I, J)] = on ? kk : 0.0;
        bad |= nonfinite(kk);
        if (on) sm = fmax(sm, fabs(kk));
      }
      const double kl = -c2 * (transpose ? G[b][a][u] : G[a][b][u]);
      O.klv[slot * B::KLS + B::kl(I, J)] = on ? emit_val(kl) : 0.0;
      bad |= nonfinite(kl);
      if (on) sm = fmax(sm, fabs(kl));
    }
  report_nonfinite(on && bad, root, nb, P.K, O.errpair);
  vm = fmax(vm, sm);
  if (on) elem_bound(O.emax, root, sm);
}

// one side of a symmetric scalar full record (full_pair_sym1): own block c2 K,
// neighbour block -c2 G (side B: G transposed)
__device__ __forceinline__ void emit_sym1(const Params& P, const VisitOut& O, long long slot, bool on, int root,
                                          int nb, double c2, const double* K, const double (*G)[3], bool transpose,
                                          double& vm) {
  using B = Blk<1>;
  bool bad = false;
  double sm = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (a <= b) {
        const double kk = c2 * K[sym3i(a, b)];
        O.kkv[slot * B::NKK + B::sym(a, b)] = on ? kk : 0.0;
        bad |= nonfinite(kk);
        if (on) sm = fmax(sm, fabs(kk));
      }
      const double kl = -c2 * (transpose ? G[b][a] : G[a][b]);
      O.klv[slot * B::KLS + B::kl(a, b)] = on ? emit_val(kl) : 0.0;
      bad |= nonfinite(kl);
      if (on) sm = fmax(sm, fabs(kl));
    }
  report_nonfinite(on && bad, root, nb, P.K, O.errpair);
  vm = fmax(vm, sm);
  if (on) elem_bound(O.emax, root, sm);
}

// full records, one thread each: the 7x7 point-pair matrix gives both visits
// MODE 0: every record; kid 0 / 1 run two launches, MODE 1 the records of
// the unique-component fast path (non-identical; kid 0: no diagonal skip)
// and MODE 2 the others, so the fast launch does not carry the general
// path's registers
template <int KID, int MODE = 0>
__global__ void __launch_bounds__(128) k_full(Params P, const int2* __restrict__ list, VisitOut O) {
  using T = KTraits<KID>;
  constexpr int E = T::E, NC = T::NC;
  __shared__ PowTab s_tab;
  if (KID == 0) {
    for (int i = threadIdx.x; i < (int)(sizeof(PowTab) / sizeof(double)); i += blockDim.x)
      reinterpret_cast<double*>(&s_tab)[i] = reinterpret_cast<const double*>(&c_powtab)[i];
    __syncthreads();
  }
  long long ev0 = 0, ev2 = 0, out0 = 0, out2 = 0;
  double vm = 0.0;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < O.nlist;
       v += (long long)gridDim.x * blockDim.x) {
    const int2 pr = list[v];
    const int k = pr.x, l = pr.y & kIdMask;
    const bool emitA = pr.y & kEmitA, emitB = pr.y & kEmitB;
    if constexpr (MODE != 0) {  // fast path: non-identical (kid 0: and no diagonal skip, path 1 only)
      bool fast = k != l;
      if (KID == 0 && fast && P.path == 1) {
        const int4 a = __ldg(&P.elem[k]), b = __ldg(&P.elem[l]);
        fast = !(a.x == b.x || a.x == b.y || a.x == b.z || a.y == b.x || a.y == b.y || a.y == b.z || a.z == b.x ||
                 a.z == b.y || a.z == b.z);
      }
      if (fast != (MODE == 1)) continue;
    }
    double kx[3], ky[3], lx[3], ly[3];
    load_tri(P, k, kx, ky);
    const int4 ek = __ldg(&P.elem[k]);
    const int4 el = __ldg(&P.elem[l]);
    const bool touching = (k == l) || ek.x == el.x || ek.x == el.y || ek.x == el.z || ek.y == el.x ||
                          ek.y == el.y || ek.y == el.z || ek.z == el.x || ek.z == el.y || ek.z == el.z;
    const double rs2 = (touching && P.path == 1) ? P.rskip2 : 0.0;
    if constexpr (KID == 0 && MODE != 2) {
      if (k != l && !(rs2 > 0.0)) {  // symmetric scalar kernel: unique components
        double lx[3], ly[3], K[6], K2[6], G[3][3];
        load_tri(P, l, lx, ly);
        long long ne = 0;
        full_pair_sym1(P, kx, ky, lx, ly, K, K2, G, ne, &s_tab);
        const double c2 = 2.0 * twice_area(kx, ky) * twice_area(lx, ly) * lab_scale(P, ek.w, el.w);
        const int mult = (emitA ? 1 : 0) + (emitB ? 1 : 0);
        ev0 += ne * mult;
        out0 += 14 * mult;
        emit_sym1(P, O, O.a_base + v, emitA, k, l, c2, K, G, false, vm);
        emit_sym1(P, O, O.b_base + __ldg(&O.revpos[v]), emitB, l, k, c2, K2, G, true, vm);
        continue;
      }
    }
    if constexpr (KID == 1 && MODE != 2) {
      if (k != l) {  // unique components, emitted on the fly (no 36-entry blocks in registers)
        double lx[3], ly[3], K[6][3], K2[6][3], G[3][3][3];
        load_tri(P, l, lx, ly);
        long long ne = 0;
        full_pair_peri(P, kx, ky, lx, ly, rs2, K, K2, G, ne);
        const double c2 = 2.0 * twice_area(kx, ky) * twice_area(lx, ly) * lab_scale(P, ek.w, el.w);
        const int mult = (emitA ? 1 : 0) + (emitB ? 1 : 0);
        ev0 += ne * mult;
        out0 += 14 * mult;
        emit_peri(P, O, O.a_base + v, emitA, k, l, c2, K, G, false, vm);
        emit_peri(P, O, O.b_base + __ldg(&O.revpos[v]), emitB, l, k, c2, K2, G, true, vm);
        continue;
      }
    }
    if constexpr (MODE == 1) {
      continue;  // (not reached: every MODE 1 record took a fast path)
    } else {
    double kkA[E], klA[E], kkB[E], klB[E];
    if (k == l) {
      // identical pair: both column halves of the reference's B hit k's dofs;
      // keep them apart for the per-triplet presence test (_engine.py:403-424)
      full_identical<KID>(P, kx, ky, rs2, kkA, klA, ev2, &s_tab);
      out2 += 7;
#pragma unroll
      for (int e = 0; e < E; ++e) kkB[e] = klB[e] = 0.0;
    } else {
      load_tri(P, l, lx, ly);
      long long ne = 0;
      full_pair2<KID>(P, kx, ky, lx, ly, rs2, kkA, klA, kkB, klB, ne, &s_tab);
      // flop accounting: the reference integrates the pair once per visit
      const int mult = (emitA ? 1 : 0) + (emitB ? 1 : 0);
      ev0 += ne * mult;
      out0 += 14 * mult;
    }
    if (P.has_lab) {
      const double ls = lab_scale(P, ek.w, el.w);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        kkA[e] *= ls; klA[e] *= ls; kkB[e] *= ls; klB[e] *= ls;
      }
    }
    emit_side<NC>(P, O, O.a_base + v, emitA, k, l, kkA, klA, vm);
    emit_side<NC>(P, O, O.b_base + __ldg(&O.revpos[v]), emitB && k != l, l, k, kkB, klB, vm);
    }
  }
  warp_max_abs(vm, O.vmax);
  warp_add_ll(ev0, &O.counters[K_EVAL_FULL0]);
  warp_add_ll(ev2, &O.counters[K_EVAL_FULL2]);
  warp_add_ll(out0, &O.counters[K_OUT_FULL0]);
  warp_add_ll(out2, &O.counters[K_OUT_FULL2]);
}

// ---------------------------------------------------------------------
// clipped (truncated) records, warp-cooperative.
// A warp takes two records at a time (lanes 0-13 and 16-29); lane = item
// (sweep m, outer point p) with m = 0: outer k / inner l, m = 1: outer l /
// inner k, m = 2: identical pair (reference mode 2).
//  phase 1: each lane clips its item with the reference's exact predicates
//           (nlg_geom.cuh) and queues its kept fan sub-triangles;
//  phase 2: lanes take one queued sub-triangle each and integrate its 7
//           inner points into the sums S0, SyP, SyQ, Syy (_engine.py:113-153);
//           a segmented warp reduction adds them to the item's row in smem;
//  phase 3: each item folds its sums (_engine.py:154-184) into BOTH visits
//           of the record -- the reference's mode-0 fold of one visit and the
//           mode-1 fold of the other use the same sweep -- and a reduce-scatter
//           over the record's 16 lanes produces the two blocks.
// Unit-to-lane mapping and reduction trees are fixed: run-to-run deterministic.
// ---------------------------------------------------------------------
template <int KID> struct ClipCfg {
  static constexpr int NC = KTraits<KID>::NC;
  static constexpr int NC2 = NC * NC;
  static constexpr bool SYM = KTraits<KID>::SYM;
  static constexpr int NKK = 3 * NC * (3 * NC + 1) / 2;  // symmetric own block, unique
  static constexpr int NKL = 9 * NC * NC;
  static constexpr int NSIDE = NKK + NKL;
  static constexpr int NVAL = 2 * NSIDE;                 // sides A and B
  // kernel-matrix components carried: the peridynamic matrix is symmetric (P_01 = P_10)
  static constexpr int NCU = KID == 1 ? 3 : NC2;
  static constexpr int NSUM = NCU * (SYM ? 6 : 9);       // barycentric moments (SumIdx)
};

// SQ: the square ball needs clip scratch rows; the circle balls clip in place
template <int KID, bool SQ>
struct ClipWarp {
  double px[32][kMaxPoly], py[32][kMaxPoly];
  double sx[SQ ? 32 : 1][kMaxPoly], sy[SQ ? 32 : 1][kMaxPoly];  // clip scratch (square ball)
  double xo[32][2];
  double W[32];
  double tri[2][2][8];  // [record slot][side]: o.x o.y e1x e1y e2x e2y idet
  double tv[2][2][6];   // [record slot][side]: the inner triangle's vertices x0 x1 x2 y0 y1 y2
  double rs2[2];
  unsigned char pm[32];
  unsigned char nv[32];  // polygon rows of each item
  int vk[2], vl[2], fl[2];  // per record slot
  int4 ek[2], el[2];        // element records (vertices, label) of the slot's record
};
// warps per k_clipped block: the fractional kernel's expensive points want
// small blocks (6 per SM); the others gain from larger clip / fan queues
template <int KID> __host__ __device__ constexpr int clip_warps() { return KID == 0 || KID == 2 ? 4 : 8; }
constexpr int kClipWarps = 4;  // (trace statistics only)
template <int KID>
struct ClipBlock {  // block-wide work queues
  int n[2];                                 // clip queue length, by chunk parity (reset one chunk ahead)
  static constexpr int NW = clip_warps<KID>();
  int wtot[NW];                             // sub-triangles per warp
  unsigned char item[32 * NW];              // clip queue: (warp << 5) | lane
  unsigned short sub[32 * NW * 7];          // sub-triangle queue: (item << 4) | t, item-major
  double tile[32 * NW][ClipCfg<KID>::NSUM + 1];  // one round's sub-triangle sums (padded rows)
  PowTab tab;                                            // pow_tab tables (fractional kernel)
};

__device__ __forceinline__ int sym3(int a, int b) {  // index of (min, max) in 00 01 02 11 12 22
  const int i = a < b ? a : b, j = a < b ? b : a;
  return i == 0 ? j : (i == 1 ? 2 + j : 5);
}

// An item's sums are barycentric moments of the weighted kernel values over
// its sub-triangles' inner points, in the inner triangle's coordinates
// (xi1, xi2) (hats h = (1 - xi1 - xi2, xi1, xi2)):
//   P moments: M0 = sum tp, M1 = sum tp xi1, M2 = sum tp xi2
//   Q moments: the same of tq, plus M11, M12, M22 = sum tq xi_a xi_b
// (tq = tp for symmetric kernels, which share the first three).  The
// reference's S0, Sy = sum t h_a and Syy = sum tq h_a h_b are linear in
// these (item_folds); 8 FP64 ops per point instead of 13.
template <int KID> struct SumIdx {
  static constexpr int NCU = ClipCfg<KID>::NCU;  // stored components
  static constexpr bool SYM = KTraits<KID>::SYM;
  // stored component of kernel-matrix entry cd (nc = 2 symmetric: 00 01 11)
  __device__ static constexpr int uc(int cd) { return NCU == 3 ? (cd == 3 ? 2 : (cd == 2 ? 1 : cd)) : cd; }
  // matrix entry of stored component i
  __device__ static constexpr int ucd(int i) { return NCU == 3 ? (i == 2 ? 3 : i) : i; }
  __device__ static constexpr int mp(int k, int i) { return k * NCU + i; }  // k: 0 -> M0, 1 -> M1, 2 -> M2
  __device__ static constexpr int mq(int k, int i) {                        // k: 0..2 as mp, 3 M11, 4 M12, 5 M22
    return SYM ? k * NCU + i : (3 + k) * NCU + i;
  }
};

// The two reference folds of one item's sums (_engine.py:154-184), as one
// block each in the layout [kk unique (I <= J) | kl]:
//   F0 (outer-test terms): kk += W oh_a oh_b S0,  kl -= W oh_a SyQ_b
//   F1 (inner-test terms): kk += W Syy_ab,        kl -= W oh_b SyP_a
template <int KID>
__device__ __forceinline__ void item_folds(double W, const double* oh, const double* s, double* F0, double* F1) {
  using C = ClipCfg<KID>;
  using X = SumIdx<KID>;
  constexpr int NC = C::NC, N3 = 3 * NC;
  const double Woh[3] = {W * oh[0], W * oh[1], W * oh[2]};
  // moments -> S0, SyP_a, SyQ_a, Syy_ab (00 01 02 11 12 22)
  double s0[C::NC2], syp[3][C::NC2], syq[3][C::NC2], syy[6][C::NC2];
#pragma unroll
  for (int cd = 0; cd < C::NC2; ++cd) {
    const int u = X::uc(cd);
    const double p0 = s[X::mp(0, u)], p1 = s[X::mp(1, u)], p2 = s[X::mp(2, u)];
    const double q0 = s[X::mq(0, u)], q1 = s[X::mq(1, u)], q2 = s[X::mq(2, u)];
    s0[cd] = p0;
    syp[0][cd] = (p0 - p1) - p2; syp[1][cd] = p1; syp[2][cd] = p2;
    syq[0][cd] = (q0 - q1) - q2; syq[1][cd] = q1; syq[2][cd] = q2;
    const double m11 = s[X::mq(3, u)], m12 = s[X::mq(4, u)], m22 = s[X::mq(5, u)];
    const double s01 = (q1 - m11) - m12, s02 = (q2 - m12) - m22;
    syy[0][cd] = (syq[0][cd] - s01) - s02; syy[1][cd] = s01; syy[2][cd] = s02;
    syy[3][cd] = m11; syy[4][cd] = m12; syy[5][cd] = m22;
  }
  int u = 0;
#pragma unroll
  for (int I = 0; I < N3; ++I)
#pragma unroll
    for (int J = I; J < N3; ++J) {
      const int a = I / NC, c = I % NC, b = J / NC, d = J % NC, cd = c * NC + d;
      F0[u] = (Woh[a] * oh[b]) * s0[cd];
      F1[u] = W * syy[sym3(a, b)][cd];
      ++u;
    }
#pragma unroll
  for (int I = 0; I < N3; ++I)
#pragma unroll
    for (int J = 0; J < N3; ++J) {
      const int a = I / NC, c = I % NC, b = J / NC, d = J % NC, cd = c * NC + d;
      F0[C::NKK + I * N3 + J] = -Woh[a] * syq[b][cd];
      F1[C::NKK + I * N3 + J] = -Woh[b] * syp[a][cd];
    }
}

// The same folds entry by entry (index g of [kk unique | kl]), so the fold
// phase holds the moment-derived terms only, not two NSIDE-value blocks per
// lane (nc = 2: 57 + 57); identical arithmetic to item_folds.
template <int KID>
struct FoldSrc {
  using C = ClipCfg<KID>;
  using X = SumIdx<KID>;
  static constexpr int NC = C::NC, N3 = 3 * NC, NU = C::NCU;
  double W, oh[3], Woh[3];
  double s0[NU], syp[3][NU], syq[3][NU], syy[6][NU];  // by stored component
  __device__ __forceinline__ FoldSrc(double w, const double* o, const double* s) {
    W = w;
#pragma unroll
    for (int a = 0; a < 3; ++a) { oh[a] = o[a]; Woh[a] = w * o[a]; }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const double p0 = s[X::mp(0, u)], p1 = s[X::mp(1, u)], p2 = s[X::mp(2, u)];
      const double q0 = s[X::mq(0, u)], q1 = s[X::mq(1, u)], q2 = s[X::mq(2, u)];
      s0[u] = p0;
      syp[0][u] = (p0 - p1) - p2; syp[1][u] = p1; syp[2][u] = p2;
      syq[0][u] = (q0 - q1) - q2; syq[1][u] = q1; syq[2][u] = q2;
      const double m11 = s[X::mq(3, u)], m12 = s[X::mq(4, u)], m22 = s[X::mq(5, u)];
      const double s01 = (q1 - m11) - m12, s02 = (q2 - m12) - m22;
      syy[0][u] = (syq[0][u] - s01) - s02; syy[1][u] = s01; syy[2][u] = s02;
      syy[3][u] = m11; syy[4][u] = m12; syy[5][u] = m22;
    }
  }
  // row / column of the u-th unique (I <= J) own-block entry, as I * 8 + J
  struct KKTab {
    unsigned char ij[C::NKK];
  };
  __host__ __device__ static constexpr KKTab kk_tab() {
    KKTab t{};
    int u = 0;
    for (int I = 0; I < N3; ++I)
      for (int J = I; J < N3; ++J) t.ij[u++] = (unsigned char)(I * 8 + J);
    return t;
  }
  __device__ __forceinline__ void entry(int g, double& f0, double& f1) const {
    if (g < C::NKK) {
      constexpr KKTab tab = kk_tab();
      const int I = tab.ij[g] >> 3, J = tab.ij[g] & 7;
      const int a = I / NC, c = I % NC, b = J / NC, d = J % NC, u = X::uc(c * NC + d);
      f0 = (Woh[a] * oh[b]) * s0[u];
      f1 = W * syy[sym3(a, b)][u];
    } else {
      const int e = g - C::NKK, I = e / N3, J = e % N3;
      const int a = I / NC, c = I % NC, b = J / NC, d = J % NC, u = X::uc(c * NC + d);
      f0 = -Woh[a] * syq[b][u];
      f1 = -Woh[b] * syp[a][u];
    }
  }
};

// closed-form moments of one fan sub-triangle for the constant / affine
// kernels (phase 2 of k_clipped): the integrands are polynomials of degree
// <= 3 and the 7-point rule (degree 5) integrates them exactly, so these are
// the reference's point sums with other rounding.  (q0, a, b): the
// sub-triangle; z*: the inner barycentrics at q0 and along a, b; x0: the
// outer point's first coordinate.
template <int KID>
__device__ __forceinline__ void closed_moments(const Params& P, double q0x, double ax, double bx, double jac2,
                                               double x0, double z1, double z2, double z1a, double z2a, double z1b,
                                               double z2b, double* sm) {
  using X = SumIdx<KID>;
  const double w = jac2 * c_rule.iws;
  const double f[3] = {z1, z1 + z1a, z1 + z1b}, g[3] = {z2, z2 + z2a, z2 + z2b};
  const double sf = f[0] + f[1] + f[2], sg = g[0] + g[1] + g[2];
  const double ff = f[0] * f[0] + f[1] * f[1] + f[2] * f[2], gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
  const double fg = f[0] * g[0] + f[1] * g[1] + f[2] * g[2];
  if constexpr (KID == 2) {  // means: (sum)/3, (sum f_i g_i + sum f sum g)/12
    const double m0 = w * P.cst;
    sm[X::mp(0, 0)] = m0;
    sm[X::mp(1, 0)] = m0 * sf * (1.0 / 3.0);
    sm[X::mp(2, 0)] = m0 * sg * (1.0 / 3.0);
    sm[X::mq(3, 0)] = m0 * (ff + sf * sf) * (1.0 / 12.0);
    sm[X::mq(4, 0)] = m0 * (fg + sf * sg) * (1.0 / 12.0);
    sm[X::mq(5, 0)] = m0 * (gg + sg * sg) * (1.0 / 12.0);
  } else {
    const double tp = w * (1.0 + P.kp0 * x0) * P.kp1;
    sm[X::mp(0, 0)] = tp;
    sm[X::mp(1, 0)] = tp * sf * (1.0 / 3.0);
    sm[X::mp(2, 0)] = tp * sg * (1.0 / 3.0);
    const double Q[3] = {(1.0 + P.kp0 * q0x) * P.kp1, (1.0 + P.kp0 * (q0x + ax)) * P.kp1,
                         (1.0 + P.kp0 * (q0x + bx)) * P.kp1};
    const double sq = Q[0] + Q[1] + Q[2];
    const double qf = Q[0] * f[0] + Q[1] * f[1] + Q[2] * f[2], qg = Q[0] * g[0] + Q[1] * g[1] + Q[2] * g[2];
    const double qff = Q[0] * f[0] * f[0] + Q[1] * f[1] * f[1] + Q[2] * f[2] * f[2];
    const double qfg = Q[0] * f[0] * g[0] + Q[1] * f[1] * g[1] + Q[2] * f[2] * g[2];
    const double qgg = Q[0] * g[0] * g[0] + Q[1] * g[1] * g[1] + Q[2] * g[2] * g[2];
    // mean(a b c) = (sa sb sc + (ab) sc + (ac) sb + (bc) sa + 2 (abc)) / 60
    sm[X::mq(0, 0)] = w * sq * (1.0 / 3.0);
    sm[X::mq(1, 0)] = w * (qf + sq * sf) * (1.0 / 12.0);
    sm[X::mq(2, 0)] = w * (qg + sq * sg) * (1.0 / 12.0);
    sm[X::mq(3, 0)] = w * (sq * sf * sf + 2.0 * qf * sf + ff * sq + 2.0 * qff) * (1.0 / 60.0);
    sm[X::mq(4, 0)] = w * (sq * sf * sg + qf * sg + qg * sf + fg * sq + 2.0 * qfg) * (1.0 / 60.0);
    sm[X::mq(5, 0)] = w * (sq * sg * sg + 2.0 * qg * sg + gg * sq + 2.0 * qgg) * (1.0 / 60.0);
  }
}

// WL: warp-local clipping (no block queue, no block barriers) -- the
// closed-form path of the constant / affine kernels only
template <int KID, bool SQ, bool WL = false>
__global__ void __launch_bounds__(32 * clip_warps<KID>(), KID == 0 ? 6 : (KID == 1 ? 2 : (KID == 2 ? 5 : 3))) k_clipped(Params P, const int2* __restrict__ list, VisitOut O) {
  using T = KTraits<KID>;
  using C = ClipCfg<KID>;
  using X = SumIdx<KID>;
  constexpr int NC = T::NC, NC2 = T::NC2, N3 = 3 * NC;
  extern __shared__ __align__(16) unsigned char clip_smem[];
  using CW = ClipWarp<KID, SQ>;
  CW* SW = reinterpret_cast<CW*>(clip_smem);
  constexpr int kClipWarps = clip_warps<KID>();
  ClipBlock<KID>& CQ = *reinterpret_cast<ClipBlock<KID>*>(clip_smem + kClipWarps * sizeof(CW));
  CW& S = SW[threadIdx.x >> 5];
  const int lane = lane_id();
  const long long nchunks = (O.nlist + 1) / 2;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned n_eval0 = 0, n_eval1 = 0, n_eval2 = 0, n_out0 = 0, n_out1 = 0, n_out2 = 0;  // per thread: < 2^32
  double vmx = 0.0;  // max |value| written
  const int vs = lane >> 4, r = lane & 15;
  if (threadIdx.x == 0) CQ.n[0] = 0;
  if (KID == 0)
    for (int i = threadIdx.x; i < (int)(sizeof(PowTab) / sizeof(double)); i += blockDim.x)
      reinterpret_cast<double*>(&CQ.tab)[i] = reinterpret_cast<const double*>(&c_powtab)[i];
  __syncthreads();
  int par = 0;
  // software pipeline: the next chunk's records and element records are
  // fetched while the current chunk computes
  int2 pr = make_int2(0, 0);
  {
    const long long v0 = w0 * 2 + vs;
    if (v0 < O.nlist) {
      pr = list[v0];
      pr.x &= kIdMask;
      if (r == 0) {  // element records of the chunk's records, via shared memory
        S.ek[vs] = __ldg(&P.elem[pr.x]);
        S.el[vs] = __ldg(&P.elem[pr.y & kIdMask]);
      }
    }
  }
  __syncwarp();
  // block-uniform trip count: the block's warps run the phases in step (the
  // __syncthreads below keep their instruction footprint to one phase)
  const long long wib = threadIdx.x >> 5;
  for (long long cb = w0 - wib; cb < nchunks; cb += nw) {
    const long long ch = cb + wib;
    // this chunk counts in CQ.n[par]; CQ.n[par ^ 1] was last read before the
    // previous chunk's post-clip barrier and is next bumped after this
    // chunk's pre-clip barrier
    if (threadIdx.x == 0) CQ.n[par ^ 1] = 0;
    // ---------------- phase 1a: classify one item per lane.  Items beyond
    // the ball are empty, items inside it keep the (deduplicated) triangle;
    // the rest go to the block's clip queue, so the branchy clipping code
    // runs on densely packed lanes.
    const long long v = ch * 2 + vs;
    const bool vok = v < O.nlist;
    bool valid = vok && r < 14;
    const int k = pr.x, l = pr.y & kIdMask, flags = pr.y & ~kIdMask;
    const int4 ek = S.ek[vs], el = S.el[vs];
    int m = r >= 7 ? 1 : 0;
    const int p = r % 7;
    if (valid && k == l) {
      if (m == 1) valid = false;
      m = 2;
    }
    // evaluations of this record count once per reference visit it stands for
    const int mult = ((flags & kEmitA) ? 1 : 0) + ((flags & kEmitB) ? 1 : 0);
    const long long vn = (ch + nw) * 2 + vs;
    const bool next_ok = vn < O.nlist;
    int2 prn = make_int2(0, 0);
    if (next_ok) {
      prn = list[vn];
      prn.x &= kIdMask;
    }
    if (r == 0 && vok) {
      S.vk[vs] = k;
      S.vl[vs] = l;
      S.fl[vs] = flags;
    }
    bool need_clip = false;
    int nv = 0;
    if (valid) {
      double ox[3], oy[3], ix[3], iy[3];
      {
        const int4 eo = m == 1 ? el : ek, ei = m == 1 ? ek : el;
        const double2 a0 = __ldg(&P.vtx[eo.x]), a1 = __ldg(&P.vtx[eo.y]), a2 = __ldg(&P.vtx[eo.z]);
        const double2 b0 = __ldg(&P.vtx[ei.x]), b1 = __ldg(&P.vtx[ei.y]), b2 = __ldg(&P.vtx[ei.z]);
        ox[0] = a0.x; oy[0] = a0.y; ox[1] = a1.x; oy[1] = a1.y; ox[2] = a2.x; oy[2] = a2.y;
        ix[0] = b0.x; iy[0] = b0.y; ix[1] = b1.x; iy[1] = b1.y; ix[2] = b2.x; iy[2] = b2.y;
      }
      const double e1x = ox[1] - ox[0], e2x = ox[2] - ox[0], e1y = oy[1] - oy[0], e2y = oy[2] - oy[0];
      const double x0 = __dadd_rn(__dadd_rn(ox[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
      const double x1 = __dadd_rn(__dadd_rn(oy[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
      // exact early-out: the inner triangle lies in disk(c, r); if that disk is
      // farther than the (widened) ball by a margin no rounding can bridge,
      // the reference's clip finds no vertex inside and no root in (0, 1)
      const int inner_el = m == 1 ? k : l;
      const double2 ci = __ldg(&P.ctr[inner_el]);
      const double reach = P.delta * (1.0 + 1e-6) + __ldg(&P.rad[inner_el]);
      const double dcx = ci.x - x0, dcy = ci.y - x1;
      const bool far = (P.dbg & 2) || (P.ball != 2 && dcx * dcx + dcy * dcy > reach * reach);
      if (!far) {
        // every inner vertex inside the widened ball: clip_circle keeps the
        // triangle (_geom_scalar.py:53-66) and no cap is inserted
        bool inside = P.ball != 2;
        if (inside) {
          const double rad = mul(P.delta, 1.0 + kBallTieRel), r2b = mul(rad, rad);
#pragma unroll
          for (int i = 0; i < 3; ++i) inside = inside && __dsub_rn(sumsq(ix[i] - x0, iy[i] - x1), r2b) <= 0.0;
        }
        if (inside) {
          double* qx = S.px[lane];
          double* qy = S.py[lane];
          const double dtol = mul(kDedupRel, P.delta);
          unsigned fdummy = 0;
#pragma unroll
          for (int i = 0; i < 3; ++i) push_dedup(qx, qy, fdummy, nv, ix[i], iy[i], false, dtol, true);
          if (nv >= 2 && fabs(qx[0] - qx[nv - 1]) <= dtol && fabs(qy[0] - qy[nv - 1]) <= dtol) --nv;
        } else {
          need_clip = true;
        }
      }
      if (g_trace_dev) {
        atomicAdd(&O.counters[K_DBG_ITEMS], 1ull);
        if (far) atomicAdd(&O.counters[K_DBG_FAR], 1ull);
        if (!far && !need_clip) atomicAdd(&O.counters[K_DBG_INSIDE], 1ull);
      }
      S.xo[lane][0] = x0;
      S.xo[lane][1] = x1;
      S.W[lane] = c_rule.ow[p] * twice_area(ox, oy);
      if (p == 0) {  // the record's inner triangle of this sweep, for the hat functions
        double* tr = S.tri[vs][m == 1];
        tr[0] = ix[0]; tr[1] = iy[0];
        tr[2] = ix[1] - ix[0]; tr[3] = iy[1] - iy[0];
        tr[4] = ix[2] - ix[0]; tr[5] = iy[2] - iy[0];
        tr[6] = 1.0 / cross2(tr[2], tr[5], tr[3], tr[4]);
        double* tv = S.tv[vs][m == 1];
        tv[0] = ix[0]; tv[1] = ix[1]; tv[2] = ix[2];
        tv[3] = iy[0]; tv[4] = iy[1]; tv[5] = iy[2];
        if (m != 1) {
          const bool touching = k == l || ek.x == el.x || ek.x == el.y || ek.x == el.z || ek.y == el.x ||
                                ek.y == el.y || ek.y == el.z || ek.z == el.x || ek.z == el.y || ek.z == el.z;
          S.rs2[vs] = (touching && P.path == 1) ? P.rskip2 : 0.0;
        }
      }
    }
    S.pm[lane] = (unsigned char)(p | (m << 4) | (valid ? 0 : 0x80));
    S.nv[lane] = (unsigned char)nv;
    if constexpr (WL) {
      // ---------------- phase 1b (warp-local): each lane clips its own item;
      // no block barrier, the warps run independently
      __syncwarp();
      if (need_clip) {
        const double* tv = S.tv[vs][m == 1];
        const Tri Tq{tv[0], tv[1], tv[2], tv[3], tv[4], tv[5]};
        int nvq;
        if constexpr (SQ)
          nvq = truncate_inner(Tq, S.xo[lane][0], S.xo[lane][1], P.delta, P.ball, S.sx[lane], S.sy[lane], S.px[lane],
                               S.py[lane]);
        else
          nvq = truncate_inner_inplace(Tq, S.xo[lane][0], S.xo[lane][1], P.delta, P.ball, S.px[lane], S.py[lane]);
        S.nv[lane] = (unsigned char)nvq;
      }
      __syncwarp();
    } else {
    {
      const unsigned qm = __ballot_sync(0xffffffffu, need_clip);
      int qb = 0;
      if (lane == 0 && qm) qb = atomicAdd(&CQ.n[par], __popc(qm));
      qb = __shfl_sync(0xffffffffu, qb, 0);
      if (need_clip) CQ.item[qb + __popc(qm & ((1u << lane) - 1u))] = (unsigned char)((wib << 5) | lane);
    }
    __syncthreads();
    // ---------------- phase 1b: the block's lanes clip the queued items
    {
      const int nq = CQ.n[par];
#pragma unroll 1
      for (int qi = threadIdx.x; qi < nq; qi += kClipWarps * 32) {
        const int it = CQ.item[qi], j = it & 31;
        CW& R = SW[it >> 5];
        const int mj = (R.pm[j] >> 4) & 3;
        const double* tv = R.tv[j >> 4][mj == 1];
        const Tri Tq{tv[0], tv[1], tv[2], tv[3], tv[4], tv[5]};
        int nvq;
        if constexpr (SQ)
          nvq = truncate_inner(Tq, R.xo[j][0], R.xo[j][1], P.delta, P.ball, S.sx[lane], S.sy[lane], R.px[j], R.py[j]);
        else
          nvq = truncate_inner_inplace(Tq, R.xo[j][0], R.xo[j][1], P.delta, P.ball, R.px[j], R.py[j]);
        R.nv[j] = (unsigned char)nvq;
      }
    }
    __syncthreads();
    }
    par ^= 1;
    double si[C::NSUM];  // the item's sums over its fan sub-triangles
#pragma unroll
    for (int i = 0; i < C::NSUM; ++i) si[i] = 0.0;
    if ((KID == 2 || KID == 3) && P.path == 0) {
      // closed-form moments are cheap: each item's lane sums its own fan
      // sub-triangles in fan order (no block queue and no rounds; the same
      // arithmetic in the same order as the queued path)
      nv = S.nv[lane];
      if (nv >= 3) {
        n_out0 += m == 0 ? mult : 0;
        n_out1 += m == 1 ? mult : 0;
        n_out2 += m == 2;
        const double* qx = S.px[lane];
        const double* qy = S.py[lane];
        const double* tr = S.tri[vs][m == 1];
        const double o0 = tr[0], o1 = tr[1], e1x = tr[2], e1y = tr[3], e2x = tr[4], e2y = tr[5], idet = tr[6];
        const double q0x = qx[0], q0y = qy[0];
        const double v0 = q0x - o0, v1 = q0y - o1;
        const double z1 = (v0 * e2y - v1 * e2x) * idet, z2 = (e1x * v1 - e1y * v0) * idet;
        const double x0 = S.xo[lane][0];
        int ne = 0;
#pragma unroll 1
        for (int t = 1; t < nv - 1; ++t) {
          const double ax = qx[t] - q0x, ay = qy[t] - q0y;
          const double bx = qx[t + 1] - q0x, by = qy[t + 1] - q0y;
          const double jac2 = cross2(ax, by, ay, bx);
          if (!(jac2 > P.drop2)) continue;
          const double z1a = (ax * e2y - ay * e2x) * idet, z2a = (e1x * ay - e1y * ax) * idet;
          const double z1b = (bx * e2y - by * e2x) * idet, z2b = (e1x * by - e1y * bx) * idet;
          double sm[C::NSUM];
          closed_moments<KID>(P, q0x, ax, bx, jac2, x0, z1, z2, z1a, z2a, z1b, z2b, sm);
#pragma unroll
          for (int i = 0; i < C::NSUM; ++i) si[i] += sm[i];
          ne += 7;
        }
        n_eval0 += m == 0 ? ne * mult : 0;
        n_eval1 += m == 1 ? ne * mult : 0;
        n_eval2 += m == 2 ? ne : 0;
      }
    } else {
    // ---------------- phase 1c: fan sub-triangles of each item -> block queue
    unsigned mask = 0;
    nv = S.nv[lane];
    if (nv >= 3) {
      n_out0 += m == 0 ? mult : 0;
      n_out1 += m == 1 ? mult : 0;
      n_out2 += m == 2;
      const double* qx = S.px[lane];
      const double* qy = S.py[lane];
#pragma unroll 1
      for (int t = 1; t < nv - 1; ++t) {
        const double ax = qx[t] - qx[0], ay = qy[t] - qy[0];
        const double bx = qx[t + 1] - qx[0], by = qy[t + 1] - qy[0];
        if (cross2(ax, by, ay, bx) > P.drop2) mask |= 1u << t;
      }
    }
    if (g_trace_dev && nv >= 3) atomicAdd(&O.counters[K_DBG_NONEMPTY], 1ull);
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) CQ.wtot[wib] = incl;
    __syncthreads();
    int total = 0, wofs = 0;
#pragma unroll
    for (int w = 0; w < kClipWarps; ++w) {
      const int c = CQ.wtot[w];
      wofs += w < wib ? c : 0;
      total += c;
    }
    const int qs = wofs + incl - cnt, qe = wofs + incl;  // this item's sub-triangles in the queue
    {
      int pos = qs;
      const int it = ((int)wib << 5) | lane;
      for (unsigned mm = mask; mm; mm &= mm - 1) CQ.sub[pos++] = (unsigned short)((it << 4) | (__ffs(mm) - 1));
    }
    if (g_trace_dev && threadIdx.x == 0) {
      atomicAdd(&O.counters[K_DBG_SUBTRI], (unsigned long long)total);
      atomicAdd(&O.counters[K_DBG_ROUNDS], (unsigned long long)((total + 127) / 128));
      atomicAdd(&O.counters[K_DBG_CHUNKS], 1ull);
    }
    __syncthreads();
    // ---------------- phase 2: the block's lanes take one queued sub-triangle
    // each and integrate its 7 inner points
    constexpr int BT = kClipWarps * 32;
    for (int u0 = 0; u0 < ((P.dbg & 1) ? 0 : total); u0 += BT) {
      const int u = u0 + (int)threadIdx.x;
      double sm[C::NSUM];
#pragma unroll
      for (int i = 0; i < C::NSUM; ++i) sm[i] = 0.0;
      if (u < total) {
        const int ent = CQ.sub[u];
        const int t = ent & 15, it = ent >> 4, j = it & 31;
        const CW& R = SW[it >> 5];
        const int mj = (R.pm[j] >> 4) & 3, vsj = j >> 4;
        const double q0x = R.px[j][0], q0y = R.py[j][0];
        const double ax = R.px[j][t] - q0x, ay = R.py[j][t] - q0y;
        const double bx = R.px[j][t + 1] - q0x, by = R.py[j][t + 1] - q0y;
        const double jac2 = cross2(ax, by, ay, bx);
        const double x0 = R.xo[j][0], x1 = R.xo[j][1];
        const double rs2 = R.rs2[vsj];
        const double* tr = R.tri[vsj][mj == 1];
        const double o0 = tr[0], o1 = tr[1], e1x = tr[2], e1y = tr[3], e2x = tr[4], e2y = tr[5], idet = tr[6];
        // barycentric coordinates of the inner triangle are affine along the
        // sub-triangle: xi(q) = xi(q0) + ip0 dxi(a) + ip1 dxi(b)
        const double v0 = q0x - o0, v1 = q0y - o1;
        const double z1 = (v0 * e2y - v1 * e2x) * idet, z2 = (e1x * v1 - e1y * v0) * idet;
        const double z1a = (ax * e2y - ay * e2x) * idet, z2a = (e1x * ay - e1y * ax) * idet;
        const double z1b = (bx * e2y - by * e2x) * idet, z2b = (e1x * by - e1y * bx) * idet;
        int ne = 0;
        bool closed = false;
        if constexpr (KID == 2 || KID == 3) {
          // constant / affine kernel: the integrands are polynomials of degree
          // <= 3 and the 7-point rule (degree 5) integrates them exactly, so the
          // reference's point sums equal closed-form moments of the
          // sub-triangle (same quantities, other rounding).  Vertex values of
          // the inner barycentrics and of Q(y) = (1 + a y_1) b:
          if (!(rs2 > 0.0)) {
            closed = true;
            ne = 7;
            closed_moments<KID>(P, q0x, ax, bx, jac2, x0, z1, z2, z1a, z2a, z1b, z2b, sm);
          }
        }
#pragma unroll 1
        for (int q = 0; q < (closed ? 0 : 7); ++q) {
          const double i0 = c_rule.ip[q][0], i1 = c_rule.ip[q][1];
          const double y0 = fma(bx, i1, fma(ax, i0, q0x));
          const double y1 = fma(by, i1, fma(ay, i0, q0y));
          const double d0 = x0 - y0, d1 = x1 - y1;
          const double r2 = fma(d0, d0, d1 * d1);
          if (rs2 > 0.0) {  // the diagonal-skip predicate needs the reference's rounding
            const double ey0 = __dadd_rn(__dadd_rn(q0x, mul(ax, i0)), mul(bx, i1));
            const double ey1 = __dadd_rn(__dadd_rn(q0y, mul(ay, i0)), mul(by, i1));
            if (sumsq(x0 - ey0, x1 - ey1) < rs2) continue;
          }
          double pv[NC2], qv[NC2];
          kval<KID, true, true>(P, x0, y0, d0, d1, r2, pv, qv, &CQ.tab);
          ++ne;
          const double wq = c_rule.iw[q] * jac2;
          const double xi1 = fma(i1, z1b, fma(i0, z1a, z1));
          const double xi2 = fma(i1, z2b, fma(i0, z2a, z2));
#pragma unroll
          for (int i = 0; i < C::NCU; ++i) {
            const double tp = wq * pv[X::ucd(i)];
            const double tq = T::SYM ? tp : wq * qv[X::ucd(i)];
            const double g1 = tq * xi1, g2 = tq * xi2;
            if (T::SYM) {
              sm[X::mp(0, i)] += tp;
              sm[X::mp(1, i)] += g1;
              sm[X::mp(2, i)] += g2;
            } else {
              sm[X::mp(0, i)] += tp;
              sm[X::mp(1, i)] = fma(tp, xi1, sm[X::mp(1, i)]);
              sm[X::mp(2, i)] = fma(tp, xi2, sm[X::mp(2, i)]);
              sm[X::mq(0, i)] += tq;
              sm[X::mq(1, i)] += g1;
              sm[X::mq(2, i)] += g2;
            }
            sm[X::mq(3, i)] = fma(g1, xi1, sm[X::mq(3, i)]);
            sm[X::mq(4, i)] = fma(g1, xi2, sm[X::mq(4, i)]);
            sm[X::mq(5, i)] = fma(g2, xi2, sm[X::mq(5, i)]);
          }
        }
        const int mlt = mj == 2 ? 1 : ((R.fl[vsj] & kEmitA) ? 1 : 0) + ((R.fl[vsj] & kEmitB) ? 1 : 0);
        n_eval0 += mj == 0 ? ne * mlt : 0;
        n_eval1 += mj == 1 ? ne * mlt : 0;
        n_eval2 += mj == 2 ? ne : 0;
      }
      // the round's sums go through shared memory; each item's lane adds the
      // rows of its sub-triangles (the queue is item-major) in queue order
#pragma unroll
      for (int i = 0; i < C::NSUM; ++i) CQ.tile[threadIdx.x][i] = sm[i];
      __syncthreads();
      const int p0 = max(qs, u0), p1 = min(qe, u0 + BT);
      for (int pp = p0; pp < p1; ++pp) {
#pragma unroll
        for (int i = 0; i < C::NSUM; ++i) si[i] += CQ.tile[pp - u0][i];
      }
      __syncthreads();
    }
    __syncthreads();
    }
    // ---------------- phase 3: fold into both visits, reduce over the record's lanes
    const int pmy = S.pm[lane];
    const bool ivalid = !(pmy & 0x80);
    const int mi = (pmy >> 4) & 3, pi = pmy & 15;
    const double Wi = ivalid ? S.W[lane] * (P.has_lab ? lab_scale(P, __ldg(&P.elem[S.vk[vs]]).w, __ldg(&P.elem[S.vl[vs]]).w) : 1.0)
                             : 0.0;  // (label factor of the pair: every entry is linear in W)
    if (next_ok && r == 0) {
      S.ek[vs] = __ldg(&P.elem[prn.x]);
      S.el[vs] = __ldg(&P.elem[prn.y & kIdMask]);
    }
    pr = prn;
    const double* ohi = c_rule.oh[pi];
    const int rk = S.vk[vs], rl = S.vl[vs], rf = S.fl[vs];
    // side A (visit (k, l)) gets the fold of the sweep it calls mode 0 / 1,
    // side B (visit (l, k)) the other one; an identical pair (m = 2) gets both on A
    const FoldSrc<KID> fs(Wi, ohi, si);
    const bool m1 = mi == 1, m2 = ivalid && mi == 2;
    constexpr int NBATCH = (C::NVAL + 31) / 32;  // reduce-scatter batches of 32 values
    double smA = 0.0, smB = 0.0;  // the sides' largest |value| (the roots' merge bounds)
#pragma unroll
    for (int bt = 0; bt < NBATCH; ++bt) {
      double vals[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int g = bt * 32 + i;
        double v = 0.0;
        if (g < C::NVAL) {
          double f0, f1;
          fs.entry(g < C::NSIDE ? g : g - C::NSIDE, f0, f1);
          if (g < C::NSIDE) {
            const double a0 = ivalid ? (m1 ? f1 : f0) : 0.0;
            v = m2 ? a0 + f1 : a0;
          } else {
            v = ivalid && !m2 ? (m1 ? f0 : f1) : 0.0;
          }
        }
        vals[i] = v;
      }
      // reduce-scatter over the 16 lanes of the record: lane r keeps [2r, 2r+2)
#pragma unroll
      for (int off = 8, half = 16; off >= 1; off >>= 1, half >>= 1) {
        const bool upper = lane & off;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const double send = upper ? vals[i] : vals[i + half];
          const double keep = upper ? vals[i + half] : vals[i];
          vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int g = bt * 32 + r * 2 + h2;
        if (!vok || g >= C::NVAL) continue;
        const double val = vals[h2];
        const int side = g / C::NSIDE, w = g % C::NSIDE;
        const bool on = side == 0 ? (rf & kEmitA) != 0 : ((rf & kEmitB) != 0 && rk != rl);
        const int root = side == 0 ? rk : rl, nb = side == 0 ? rl : rk;
        const long long slot = side ? O.b_base + __ldg(&O.revpos[v]) : O.a_base + v;
        if (on) {
          report_nonfinite(nonfinite(val), root, nb, P.K, O.errpair);
          vmx = fmax(vmx, fabs(val));
          if (side == 0) smA = fmax(smA, fabs(val));
          else smB = fmax(smB, fabs(val));
        }
        if (w < C::NKK) {
          O.kkv[slot * Blk<NC>::NKK + w] = on ? val : 0.0;  // unique (I <= J) order
        } else {
          const int e = w - C::NKK, I = e / N3, J = e % N3;
          O.klv[slot * Blk<NC>::KLS + Blk<NC>::kl(I, J)] = on ? emit_val(val) : 0.0;
        }
      }
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {  // within the record's 16 lanes
      smA = fmax(smA, __shfl_xor_sync(0xffffffffu, smA, o));
      smB = fmax(smB, __shfl_xor_sync(0xffffffffu, smB, o));
    }
    if (r == 0 && vok) {
      elem_bound(O.emax, rk, smA);
      elem_bound(O.emax, rl, smB);
    }
    __syncwarp();
  }
  warp_max_abs(vmx, O.vmax);
  warp_add_ll((unsigned long long)n_eval0, &O.counters[K_EVAL_M0]);
  warp_add_ll((unsigned long long)n_out0, &O.counters[K_OUT_M0]);
  warp_add_ll((unsigned long long)n_eval1, &O.counters[K_EVAL_M1]);
  warp_add_ll((unsigned long long)n_out1, &O.counters[K_OUT_M1]);
  warp_add_ll((unsigned long long)n_eval2, &O.counters[K_EVAL_M2]);
  warp_add_ll((unsigned long long)n_out2, &O.counters[K_OUT_M2]);
}

// ---------------------------------------------------------------------
// Clipped records of the constant / affine kernels on the standard path
// (closed-form sub-triangle moments): one warp works alone on four records
// per round -- 56 sweep items in 64 slots, two per lane -- with a warp-local
// clip queue, so the ~30 items that need clipping run on ~30 of the 32 lanes
// and no warp ever waits for another (no block barriers).  Same predicates,
// same arithmetic in the same order as k_clipped's closed-form path.
// Slot s: record s >> 4 of the round, item s & 15 (sweep m, outer point p).
// ---------------------------------------------------------------------
template <int KID>
struct CfWarp {
  double px[64][kMaxPoly], py[64][kMaxPoly];
  double xo[64][2];
  double W[64];
  double tri[4][2][7];  // [record][inner side]: o.x o.y e1x e1y e2x e2y idet
  double tv[4][2][6];   // [record][inner side]: the inner triangle's vertices x0 x1 x2 y0 y1 y2
  unsigned char pm[64];
  unsigned char nv[64];
  unsigned char q[64];  // clip queue (slots)
  int vk[4], vl[4], fl[4];
  int4 ek[4], el[4];
};
template <int KID, int NWB, int MINB>
__global__ void __launch_bounds__(32 * NWB, MINB) k_clipped_cf(Params P, const int2* __restrict__ list, VisitOut O) {
  static_assert(KID == 2 || KID == 3, "closed-form path: constant / affine kernels");
  using C = ClipCfg<KID>;
  constexpr int NC = 1, N3 = 3;
  extern __shared__ __align__(16) unsigned char cf_smem[];
  CfWarp<KID>& S = reinterpret_cast<CfWarp<KID>*>(cf_smem)[threadIdx.x >> 5];
  const int lane = lane_id();
  const long long nround = (O.nlist + 3) / 4;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned n_eval0 = 0, n_eval1 = 0, n_eval2 = 0, n_out0 = 0, n_out1 = 0, n_out2 = 0;
  double vmx = 0.0;
  const int r = lane & 15, vs = lane >> 4;
  // software pipeline: lane r < 4 fetches record r of the next round
  int2 pnext = make_int2(0, 0);
  int4 eknext = make_int4(0, 0, 0, 0), elnext = eknext;
  auto fetch = [&](long long rdn) {
    if (lane < 4) {
      const long long v = rdn * 4 + lane;
      if (rdn < nround && v < O.nlist) {
        pnext = list[v];
        eknext = __ldg(&P.elem[pnext.x & kIdMask]);
        elnext = __ldg(&P.elem[pnext.y & kIdMask]);
      }
    }
  };
  fetch(w0);
  for (long long rd = w0; rd < nround; rd += nw) {
    // ---- the round's four records and their element records
    if (lane < 4 && rd * 4 + lane < O.nlist) {
      S.vk[lane] = pnext.x & kIdMask;
      S.vl[lane] = pnext.y & kIdMask;
      S.fl[lane] = pnext.y & ~kIdMask;
      S.ek[lane] = eknext;
      S.el[lane] = elnext;
    }
    __syncwarp();
    fetch(rd + nw);
    // ---- classify both slots of the lane; queue the ones that need a clip
    int qn = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rec = vs + 2 * h, sl = lane + 32 * h;
      const long long v = rd * 4 + rec;
      bool valid = v < O.nlist && r < 14;
      const int k = valid ? S.vk[rec] : 0, l = valid ? S.vl[rec] : 0;
      int m = r >= 7 ? 1 : 0;
      const int p = r % 7;
      if (valid && k == l) {
        if (m == 1) valid = false;
        m = 2;
      }
      bool need_clip = false;
      int nv = 0;
      if (valid) {
        const int4 ek = S.ek[rec], el = S.el[rec];
        double ox[3], oy[3], ix[3], iy[3];
        {
          const int4 eo = m == 1 ? el : ek, ei = m == 1 ? ek : el;
          const double2 a0 = __ldg(&P.vtx[eo.x]), a1 = __ldg(&P.vtx[eo.y]), a2 = __ldg(&P.vtx[eo.z]);
          const double2 b0 = __ldg(&P.vtx[ei.x]), b1 = __ldg(&P.vtx[ei.y]), b2 = __ldg(&P.vtx[ei.z]);
          ox[0] = a0.x; oy[0] = a0.y; ox[1] = a1.x; oy[1] = a1.y; ox[2] = a2.x; oy[2] = a2.y;
          ix[0] = b0.x; iy[0] = b0.y; ix[1] = b1.x; iy[1] = b1.y; ix[2] = b2.x; iy[2] = b2.y;
        }
        const double e1x = ox[1] - ox[0], e2x = ox[2] - ox[0], e1y = oy[1] - oy[0], e2y = oy[2] - oy[0];
        const double x0 = __dadd_rn(__dadd_rn(ox[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
        const double x1 = __dadd_rn(__dadd_rn(oy[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
        const int inner_el = m == 1 ? k : l;
        const double2 ci = __ldg(&P.ctr[inner_el]);
        const double reach = P.delta * (1.0 + 1e-6) + __ldg(&P.rad[inner_el]);
        const double dcx = ci.x - x0, dcy = ci.y - x1;
        const bool far = P.ball != 2 && dcx * dcx + dcy * dcy > reach * reach;
        if (!far) {
          bool inside = P.ball != 2;
          if (inside) {
            const double rad = mul(P.delta, 1.0 + kBallTieRel), r2b = mul(rad, rad);
#pragma unroll
            for (int i = 0; i < 3; ++i) inside = inside && __dsub_rn(sumsq(ix[i] - x0, iy[i] - x1), r2b) <= 0.0;
          }
          if (inside) {
            double* qx = S.px[sl];
            double* qy = S.py[sl];
            const double dtol = mul(kDedupRel, P.delta);
            unsigned fdummy = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) push_dedup(qx, qy, fdummy, nv, ix[i], iy[i], false, dtol, true);
            if (nv >= 2 && fabs(qx[0] - qx[nv - 1]) <= dtol && fabs(qy[0] - qy[nv - 1]) <= dtol) --nv;
          } else {
            need_clip = true;
          }
        }
        S.xo[sl][0] = x0;
        S.xo[sl][1] = x1;
        // (the pair's label factor rides on the weight: every entry is linear in W)
        S.W[sl] = c_rule.ow[p] * twice_area(ox, oy) * lab_scale(P, ek.w, el.w);
        if (p == 0) {  // the record's inner triangle of this sweep, for the hat functions
          double* tr = S.tri[rec][m == 1];
          tr[0] = ix[0]; tr[1] = iy[0];
          tr[2] = ix[1] - ix[0]; tr[3] = iy[1] - iy[0];
          tr[4] = ix[2] - ix[0]; tr[5] = iy[2] - iy[0];
          tr[6] = 1.0 / cross2(tr[2], tr[5], tr[3], tr[4]);
          double* tv = S.tv[rec][m == 1];
          tv[0] = ix[0]; tv[1] = ix[1]; tv[2] = ix[2];
          tv[3] = iy[0]; tv[4] = iy[1]; tv[5] = iy[2];
        }
      }
      S.pm[sl] = (unsigned char)(p | (m << 4) | (valid ? 0 : 0x80));
      S.nv[sl] = (unsigned char)nv;
      const unsigned qm = __ballot_sync(0xffffffffu, need_clip);
      if (need_clip) S.q[qn + __popc(qm & ((1u << lane) - 1u))] = (unsigned char)sl;
      qn += __popc(qm);
    }
    __syncwarp();
    // ---- the queued clips on consecutive lanes
#pragma unroll 1
    for (int qi = lane; qi < ((P.dbg & 64) ? 0 : qn); qi += 32) {  // (NLG_DEBUG & 64 / 128 / 256: timing experiments)
      const int sl = S.q[qi];
      const int mj = (S.pm[sl] >> 4) & 3;
      const double* tv = S.tv[sl >> 4][mj == 1];
      const Tri Tq{tv[0], tv[1], tv[2], tv[3], tv[4], tv[5]};
      S.nv[sl] = (unsigned char)truncate_inner_inplace(Tq, S.xo[sl][0], S.xo[sl][1], P.delta, P.ball, S.px[sl],
                                                       S.py[sl]);
    }
    __syncwarp();
    // ---- per slot: closed-form fan sums, then fold and reduce two records
#pragma unroll 1
    for (int h = 0; h < ((P.dbg & 128) ? 0 : 2); ++h) {
      const int rec = vs + 2 * h, sl = lane + 32 * h;
      const long long v = rd * 4 + rec;
      const bool vok = v < O.nlist;
      const int pmy = S.pm[sl];
      const bool ivalid = !(pmy & 0x80);
      const int mi = (pmy >> 4) & 3, pi = pmy & 15;
      const int rf = vok ? S.fl[rec] : 0, rk = vok ? S.vk[rec] : 0, rl = vok ? S.vl[rec] : 0;
      const int mult = ((rf & kEmitA) ? 1 : 0) + ((rf & kEmitB) ? 1 : 0);
      double si[C::NSUM];
#pragma unroll
      for (int i = 0; i < C::NSUM; ++i) si[i] = 0.0;
      const int nv = S.nv[sl];
      if (ivalid && nv >= 3 && !(P.dbg & 256)) {
        n_out0 += mi == 0 ? mult : 0;
        n_out1 += mi == 1 ? mult : 0;
        n_out2 += mi == 2;
        const double* qx = S.px[sl];
        const double* qy = S.py[sl];
        const double* tr = S.tri[rec][mi == 1];
        const double o0 = tr[0], o1 = tr[1], e1x = tr[2], e1y = tr[3], e2x = tr[4], e2y = tr[5], idet = tr[6];
        const double q0x = qx[0], q0y = qy[0];
        const double v0 = q0x - o0, v1 = q0y - o1;
        const double z1 = (v0 * e2y - v1 * e2x) * idet, z2 = (e1x * v1 - e1y * v0) * idet;
        const double x0 = S.xo[sl][0];
        int ne = 0;
#pragma unroll 1
        for (int t = 1; t < nv - 1; ++t) {
          const double ax = qx[t] - q0x, ay = qy[t] - q0y;
          const double bx = qx[t + 1] - q0x, by = qy[t + 1] - q0y;
          const double jac2 = cross2(ax, by, ay, bx);
          if (!(jac2 > P.drop2)) continue;
          const double z1a = (ax * e2y - ay * e2x) * idet, z2a = (e1x * ay - e1y * ax) * idet;
          const double z1b = (bx * e2y - by * e2x) * idet, z2b = (e1x * by - e1y * bx) * idet;
          double sm[C::NSUM];
          closed_moments<KID>(P, q0x, ax, bx, jac2, x0, z1, z2, z1a, z2a, z1b, z2b, sm);
#pragma unroll
          for (int i = 0; i < C::NSUM; ++i) si[i] += sm[i];
          ne += 7;
        }
        n_eval0 += mi == 0 ? ne * mult : 0;
        n_eval1 += mi == 1 ? ne * mult : 0;
        n_eval2 += mi == 2 ? ne : 0;
      }
      // fold into both visits, reduce-scatter over the record's 16 lanes
      const double Wi = ivalid ? S.W[sl] : 0.0;
      const double* ohi = c_rule.oh[pi];
      const FoldSrc<KID> fs(Wi, ohi, si);
      const bool m1 = mi == 1, m2 = ivalid && mi == 2;
      constexpr int NBATCH = (C::NVAL + 31) / 32;
      double smA = 0.0, smB = 0.0;  // the sides' largest |value| (the roots' merge bounds)
#pragma unroll
      for (int bt = 0; bt < NBATCH; ++bt) {
        double vals[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int g = bt * 32 + i;
          double val = 0.0;
          if (g < C::NVAL) {
            double f0, f1;
            fs.entry(g < C::NSIDE ? g : g - C::NSIDE, f0, f1);
            if (g < C::NSIDE) {
              const double a0 = ivalid ? (m1 ? f1 : f0) : 0.0;
              val = m2 ? a0 + f1 : a0;
            } else {
              val = ivalid && !m2 ? (m1 ? f0 : f1) : 0.0;
            }
          }
          vals[i] = val;
        }
#pragma unroll
        for (int off = 8, half = 16; off >= 1; off >>= 1, half >>= 1) {
          const bool upper = lane & off;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const double send = upper ? vals[i] : vals[i + half];
            const double keep = upper ? vals[i + half] : vals[i];
            vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int g = bt * 32 + r * 2 + h2;
          if (!vok || g >= C::NVAL) continue;
          const double val = vals[h2];
          const int side = g / C::NSIDE, w = g % C::NSIDE;
          const bool on = side == 0 ? (rf & kEmitA) != 0 : ((rf & kEmitB) != 0 && rk != rl);
          const int root = side == 0 ? rk : rl, nb = side == 0 ? rl : rk;
          const long long slot = side ? O.b_base + __ldg(&O.revpos[v]) : O.a_base + v;
          if (on) {
            report_nonfinite(nonfinite(val), root, nb, P.K, O.errpair);
            vmx = fmax(vmx, fabs(val));
            if (side == 0) smA = fmax(smA, fabs(val));
            else smB = fmax(smB, fabs(val));
          }
          if (w < C::NKK) {
            O.kkv[slot * Blk<NC>::NKK + w] = on ? val : 0.0;
          } else {
            const int e = w - C::NKK, I = e / N3, J = e % N3;
            O.klv[slot * Blk<NC>::KLS + Blk<NC>::kl(I, J)] = on ? emit_val(val) : 0.0;
          }
        }
      }
      if (!P.analytic) {  // (analytic rows: a plan bound covers the clipped values)
#pragma unroll
        for (int o = 8; o; o >>= 1) {  // within the record's 16 lanes
          smA = fmax(smA, __shfl_xor_sync(0xffffffffu, smA, o));
          smB = fmax(smB, __shfl_xor_sync(0xffffffffu, smB, o));
        }
        if (r == 0 && vok) {
          elem_bound(O.emax, rk, smA);
          elem_bound(O.emax, rl, smB);
        }
      }
    }
    __syncwarp();
  }
  warp_max_abs(vmx, O.vmax);
  warp_add_ll((unsigned long long)n_eval0, &O.counters[K_EVAL_M0]);
  warp_add_ll((unsigned long long)n_out0, &O.counters[K_OUT_M0]);
  warp_add_ll((unsigned long long)n_eval1, &O.counters[K_EVAL_M1]);
  warp_add_ll((unsigned long long)n_out1, &O.counters[K_OUT_M1]);
  warp_add_ll((unsigned long long)n_eval2, &O.counters[K_EVAL_M2]);
  warp_add_ll((unsigned long long)n_out2, &O.counters[K_OUT_M2]);
}

// k_clipped_cf with a clip queue that runs across rounds.  A round of four
// records queues ~21 items that need a clip, so a clip pass of k_clipped_cf
// runs on ~21 of 32 lanes.  Here the queue is a ring: a round is classified
// one round ahead of its sums, and a clip pass runs when 32 items are queued
// (or when the previous round still waits for some of its own), on full
// lanes.  Clip results live in a ring of kCfCap polygons indexed by queue
// position; items wholly inside the ball keep no polygon (it is the inner
// triangle, read from tv).  The per-round state is double buffered.  Items
// are computed exactly as in k_clipped_cf and folded by the same shuffles:
// the values are the same bits, only the schedule differs.
constexpr int kCfCap = 64;
template <int KID>
struct CfMeta {
  double xo[64][2];
  double tri[4][2][7];  // [record][inner side]: o.x o.y e1x e1y e2x e2y idet
  double tv[4][2][6];   // [record][inner side]: the inner triangle's vertices x0 x1 x2 y0 y1 y2
  double ta[4][2];      // [record][outer side is l]: twice the outer triangle's area
  double ls[4];         // the record's label factor
  unsigned char pm[64];  // p | m << 4 | 0x40 (inside: polygon = tv) | 0x80 (no item)
  unsigned char nv[64];
  unsigned char st[64];  // clipped items: polygon ring index
  int vk[4], vl[4], fl[4];
};
template <int KID>
struct CfRing {
  CfMeta<KID> M[2];
  double px[kCfCap][kMaxPoly], py[kCfCap][kMaxPoly];
  int4 ek[4], el[4];
  unsigned char q[128];  // queued items: slot | round parity << 6
};
template <int KID, int NWB, int MINB, int CU = 2, int SY = 0, int BALL = -1, int AN = -1>
__global__ void __launch_bounds__(32 * NWB, MINB) k_clipped_cfr(Params P, const int2* __restrict__ list, VisitOut O) {
  static_assert(KID == 2 || KID == 3, "closed-form path: constant / affine kernels");
  using C = ClipCfg<KID>;
  constexpr int NC = 1, N3 = 3;
  extern __shared__ __align__(16) unsigned char cf_smem[];
  CfRing<KID>& S = reinterpret_cast<CfRing<KID>*>(cf_smem)[threadIdx.x >> 5];
  const int ball = BALL >= 0 ? BALL : P.ball;  // (BALL: the ball's code alone, a denser instruction stream)
  const bool analytic = AN >= 0 ? AN != 0 : P.analytic != 0;  // (AN: likewise for the per-element bounds)
  const int lane = lane_id();
  const long long nround = (O.nlist + 3) / 4;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned n_eval0 = 0, n_eval1 = 0, n_eval2 = 0, n_out0 = 0, n_out1 = 0, n_out2 = 0;
  double vmx = 0.0;
  const int r = lane & 15, vs = lane >> 4;
  int2 pnext = make_int2(0, 0);
  int4 eknext = make_int4(0, 0, 0, 0), elnext = eknext;
  auto fetch = [&](long long rdn) {
    if (lane < 4) {
      const long long v = rdn * 4 + lane;
      if (rdn < nround && v < O.nlist) {
        pnext = list[v];
        eknext = __ldg(&P.elem[pnext.x & kIdMask]);
        elnext = __ldg(&P.elem[pnext.y & kIdMask]);
      }
    }
  };
  fetch(w0);
  int head = 0, tail = 0;  // clip items processed / queued so far by this warp
  int prev_start = 0, prev_end = 0, par = 0;
  long long prev = -1;
  // every warp of a block runs the block's iteration count (its first warp's
  // rounds + the flush), so that the block can re-align its warps' phases
  // every SY rounds: warps in the same phase share the instruction cache
  const long long wb0 = (blockIdx.x * (long long)blockDim.x) >> 5;
  const long long niter = wb0 < nround ? (nround - wb0 + nw - 1) / nw + 1 : 0;
  long long rd = w0;
  for (long long it = 0; it < niter; ++it, rd += nw) {
    if (SY > 0 && it % SY == 0) __syncthreads();
    if (SY < 0 && it % (-SY) == 0)  // the four warps of a scheduler (warp % 4) only
      asm volatile("bar.sync %0, 128;" ::"r"(1 + ((threadIdx.x >> 5) & 3)) : "memory");
    const bool have = rd < nround;
    const int cur_start = tail;
    if (have) {
      CfMeta<KID>& M = S.M[par];
      if (lane < 4 && rd * 4 + lane < O.nlist) {
        M.vk[lane] = pnext.x & kIdMask;
        M.vl[lane] = pnext.y & kIdMask;
        M.fl[lane] = pnext.y & ~kIdMask;
        S.ek[lane] = eknext;
        S.el[lane] = elnext;
      }
      __syncwarp();
      fetch(rd + nw);
      // ---- classify both slots of the lane; queue the ones that need a clip
#pragma unroll CU
      for (int h = 0; h < 2; ++h) {
        const int rec = vs + 2 * h, sl = lane + 32 * h;
        const long long v = rd * 4 + rec;
        bool valid = v < O.nlist && r < 14;
        const int k = valid ? M.vk[rec] : 0, l = valid ? M.vl[rec] : 0;
        int m = r >= 7 ? 1 : 0;
        const int p = r % 7;
        if (valid && k == l) {
          if (m == 1) valid = false;
          m = 2;
        }
        bool need_clip = false, inside_item = false;
        int nv = 0;
        if (valid) {
          const int4 ek = S.ek[rec], el = S.el[rec];
          double ox[3], oy[3], ix[3], iy[3];
          {
            const int4 eo = m == 1 ? el : ek, ei = m == 1 ? ek : el;
            const double2 a0 = __ldg(&P.vtx[eo.x]), a1 = __ldg(&P.vtx[eo.y]), a2 = __ldg(&P.vtx[eo.z]);
            const double2 b0 = __ldg(&P.vtx[ei.x]), b1 = __ldg(&P.vtx[ei.y]), b2 = __ldg(&P.vtx[ei.z]);
            ox[0] = a0.x; oy[0] = a0.y; ox[1] = a1.x; oy[1] = a1.y; ox[2] = a2.x; oy[2] = a2.y;
            ix[0] = b0.x; iy[0] = b0.y; ix[1] = b1.x; iy[1] = b1.y; ix[2] = b2.x; iy[2] = b2.y;
          }
          const double e1x = ox[1] - ox[0], e2x = ox[2] - ox[0], e1y = oy[1] - oy[0], e2y = oy[2] - oy[0];
          const double x0 = __dadd_rn(__dadd_rn(ox[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
          const double x1 = __dadd_rn(__dadd_rn(oy[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
          const int inner_el = m == 1 ? k : l;
          const double2 ci = __ldg(&P.ctr[inner_el]);
          const double reach = P.delta * (1.0 + 1e-6) + __ldg(&P.rad[inner_el]);
          const double dcx = ci.x - x0, dcy = ci.y - x1;
          const bool far = ball != 2 && dcx * dcx + dcy * dcy > reach * reach;
          if (!far) {
            bool inside = ball != 2;
            if (inside) {
              const double rad = mul(P.delta, 1.0 + kBallTieRel), r2b = mul(rad, rad);
#pragma unroll
              for (int i = 0; i < 3; ++i) inside = inside && __dsub_rn(sumsq(ix[i] - x0, iy[i] - x1), r2b) <= 0.0;
            }
            if (inside) {
              // the deduplicated inner triangle: three rows unless two vertices coincide within dtol
              const double dtol = mul(kDedupRel, P.delta);
              double lx = ix[0], ly = iy[0];
              nv = 1;
#pragma unroll
              for (int i = 1; i < 3; ++i)
                if (fabs(lx - ix[i]) > dtol || fabs(ly - iy[i]) > dtol) {
                  lx = ix[i];
                  ly = iy[i];
                  ++nv;
                }
              if (nv >= 2 && fabs(ix[0] - lx) <= dtol && fabs(iy[0] - ly) <= dtol) --nv;
              inside_item = true;
            } else {
              need_clip = true;
            }
          }
          M.xo[sl][0] = x0;
          M.xo[sl][1] = x1;
          if (p == 0) {  // the record's triangles of this sweep
            M.ta[rec][m == 1] = twice_area(ox, oy);
            if (m != 1) M.ls[rec] = lab_scale(P, ek.w, el.w);
            double* tr = M.tri[rec][m == 1];
            tr[0] = ix[0]; tr[1] = iy[0];
            tr[2] = ix[1] - ix[0]; tr[3] = iy[1] - iy[0];
            tr[4] = ix[2] - ix[0]; tr[5] = iy[2] - iy[0];
            tr[6] = 1.0 / cross2(tr[2], tr[5], tr[3], tr[4]);
            double* tv = M.tv[rec][m == 1];
            tv[0] = ix[0]; tv[1] = ix[1]; tv[2] = ix[2];
            tv[3] = iy[0]; tv[4] = iy[1]; tv[5] = iy[2];
          }
        }
        M.pm[sl] = (unsigned char)(p | (m << 4) | (inside_item ? 0x40 : 0) | (valid ? 0 : 0x80));
        M.nv[sl] = (unsigned char)nv;
        const unsigned qm = __ballot_sync(0xffffffffu, need_clip);
        if (need_clip) S.q[(tail + __popc(qm & ((1u << lane) - 1u))) & 127] = (unsigned char)(sl | (par << 6));
        tail += __popc(qm);
      }
    }
    __syncwarp();
    // ---- clip passes: full lanes, or whatever the previous round still waits for
    {
      const int live0 = prev >= 0 ? prev_start : cur_start;  // oldest polygon still needed
      for (;;) {
        const int n = min(min(32, tail - head), kCfCap - (head - live0));
        const bool forced = prev >= 0 && head < prev_end;
        if (n <= 0 || (n < 32 && !forced)) break;
        if (lane < n) {
          const int qi = head + lane, e = S.q[qi & 127];
          const int sl = e & 63, si = qi & (kCfCap - 1);
          CfMeta<KID>& Mq = S.M[e >> 6];
          const int mj = (Mq.pm[sl] >> 4) & 3;
          const double* tv = Mq.tv[sl >> 4][mj == 1];
          const Tri Tq{tv[0], tv[1], tv[2], tv[3], tv[4], tv[5]};
          Mq.nv[sl] = (unsigned char)truncate_inner_inplace(Tq, Mq.xo[sl][0], Mq.xo[sl][1], P.delta, ball,
                                                            S.px[si], S.py[si]);
          Mq.st[sl] = (unsigned char)si;
        }
        head += n;
      }
    }
    __syncwarp();
    // ---- the previous round: closed-form fan sums per slot, then fold and reduce two records
    if (prev >= 0) {
      const CfMeta<KID>& M = S.M[par ^ 1];
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int rec = vs + 2 * h, sl = lane + 32 * h;
        const long long v = prev * 4 + rec;
        const bool vok = v < O.nlist;
        const int pmy = M.pm[sl];
        const bool ivalid = !(pmy & 0x80);
        const int mi = (pmy >> 4) & 3, pi = pmy & 15;
        const int rf = vok ? M.fl[rec] : 0, rk = vok ? M.vk[rec] : 0, rl = vok ? M.vl[rec] : 0;
        const int mult = ((rf & kEmitA) ? 1 : 0) + ((rf & kEmitB) ? 1 : 0);
        double si[C::NSUM];
#pragma unroll
        for (int i = 0; i < C::NSUM; ++i) si[i] = 0.0;
        const int nv = M.nv[sl];
        if (ivalid && nv >= 3) {
          n_out0 += mi == 0 ? mult : 0;
          n_out1 += mi == 1 ? mult : 0;
          n_out2 += mi == 2;
          const double* tvi = M.tv[rec][mi == 1];
          const int st = M.st[sl];
          const double* qx = (pmy & 0x40) ? tvi : S.px[st];
          const double* qy = (pmy & 0x40) ? tvi + 3 : S.py[st];
          const double* tr = M.tri[rec][mi == 1];
          const double o0 = tr[0], o1 = tr[1], e1x = tr[2], e1y = tr[3], e2x = tr[4], e2y = tr[5], idet = tr[6];
          const double q0x = qx[0], q0y = qy[0];
          const double v0 = q0x - o0, v1 = q0y - o1;
          const double z1 = (v0 * e2y - v1 * e2x) * idet, z2 = (e1x * v1 - e1y * v0) * idet;
          const double x0 = M.xo[sl][0];
          int ne = 0;
#pragma unroll 1
          for (int t = 1; t < nv - 1; ++t) {
            const double ax = qx[t] - q0x, ay = qy[t] - q0y;
            const double bx = qx[t + 1] - q0x, by = qy[t + 1] - q0y;
            const double jac2 = cross2(ax, by, ay, bx);
            if (!(jac2 > P.drop2)) continue;
            const double z1a = (ax * e2y - ay * e2x) * idet, z2a = (e1x * ay - e1y * ax) * idet;
            const double z1b = (bx * e2y - by * e2x) * idet, z2b = (e1x * by - e1y * bx) * idet;
            double sm[C::NSUM];
            closed_moments<KID>(P, q0x, ax, bx, jac2, x0, z1, z2, z1a, z2a, z1b, z2b, sm);
#pragma unroll
            for (int i = 0; i < C::NSUM; ++i) si[i] += sm[i];
            ne += 7;
          }
          n_eval0 += mi == 0 ? ne * mult : 0;
          n_eval1 += mi == 1 ? ne * mult : 0;
          n_eval2 += mi == 2 ? ne : 0;
        }
        // fold into both visits, reduce-scatter over the record's 16 lanes
        // (the pair's label factor rides on the weight: every entry is linear in W)
        const double Wi = ivalid ? mul(mul(c_rule.ow[pi], M.ta[rec][mi == 1]), M.ls[rec]) : 0.0;
        const double* ohi = c_rule.oh[pi];
        const FoldSrc<KID> fs(Wi, ohi, si);
        const bool m1 = mi == 1, m2 = ivalid && mi == 2;
        constexpr int NBATCH = (C::NVAL + 31) / 32;
        double smA = 0.0, smB = 0.0;  // the sides' largest |value| (the roots' merge bounds)
#pragma unroll
        for (int bt = 0; bt < NBATCH; ++bt) {
          double vals[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int g = bt * 32 + i;
            double val = 0.0;
            if (g < C::NVAL) {
              double f0, f1;
              fs.entry(g < C::NSIDE ? g : g - C::NSIDE, f0, f1);
              if (g < C::NSIDE) {
                const double a0 = ivalid ? (m1 ? f1 : f0) : 0.0;
                val = m2 ? a0 + f1 : a0;
              } else {
                val = ivalid && !m2 ? (m1 ? f0 : f1) : 0.0;
              }
            }
            vals[i] = val;
          }
#pragma unroll
          for (int off = 8, half = 16; off >= 1; off >>= 1, half >>= 1) {
            const bool upper = lane & off;
#pragma unroll
            for (int i = 0; i < half; ++i) {
              const double send = upper ? vals[i] : vals[i + half];
              const double keep = upper ? vals[i + half] : vals[i];
              vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int g = bt * 32 + r * 2 + h2;
            if (!vok || g >= C::NVAL) continue;
            const double val = vals[h2];
            const int side = g / C::NSIDE, w = g % C::NSIDE;
            const bool on = side == 0 ? (rf & kEmitA) != 0 : ((rf & kEmitB) != 0 && rk != rl);
            const int root = side == 0 ? rk : rl, nb = side == 0 ? rl : rk;
            const long long slot = side ? O.b_base + __ldg(&O.revpos[v]) : O.a_base + v;
            if (on) {
              report_nonfinite(nonfinite(val), root, nb, P.K, O.errpair);
              vmx = fmax(vmx, fabs(val));
              if (!analytic) {
                if (side == 0) smA = fmax(smA, fabs(val));
                else smB = fmax(smB, fabs(val));
              }
            }
            if (w < C::NKK) {
              O.kkv[slot * Blk<NC>::NKK + w] = on ? val : 0.0;
            } else {
              const int e = w - C::NKK, I = e / N3, J = e % N3;
              O.klv[slot * Blk<NC>::KLS + Blk<NC>::kl(I, J)] = on ? emit_val(val) : 0.0;
            }
          }
        }
        if (!analytic) {  // (analytic rows: a plan bound covers the clipped values)
#pragma unroll
          for (int o = 8; o; o >>= 1) {  // within the record's 16 lanes
            smA = fmax(smA, __shfl_xor_sync(0xffffffffu, smA, o));
            smB = fmax(smB, __shfl_xor_sync(0xffffffffu, smB, o));
          }
          if (r == 0 && vok) {
            elem_bound(O.emax, rk, smA);
            elem_bound(O.emax, rl, smB);
          }
        }
      }
      __syncwarp();
    }
    prev = have ? rd : -1;
    prev_start = cur_start;
    prev_end = tail;
    par ^= 1;
  }
  warp_max_abs(vmx, O.vmax);
  warp_add_ll((unsigned long long)n_eval0, &O.counters[K_EVAL_M0]);
  warp_add_ll((unsigned long long)n_out0, &O.counters[K_OUT_M0]);
  warp_add_ll((unsigned long long)n_eval1, &O.counters[K_EVAL_M1]);
  warp_add_ll((unsigned long long)n_out1, &O.counters[K_OUT_M1]);
  warp_add_ll((unsigned long long)n_eval2, &O.counters[K_EVAL_M2]);
  warp_add_ll((unsigned long long)n_out2, &O.counters[K_OUT_M2]);
}

// ---------------------------------------------------------------------
// local_contribution (assembly.py:327-448): the 4-term block of the ORDERED
// pair (k, l) -- outer points on k, the inner element l retriangulated
// against the ball of each -- as a dense (6 nc) x (6 nc) block over the
// dofs (k's, l's).  One warp per pair, lane p < 7 = outer point p: clip,
// fan, 7 inner points (kernel values, no closed forms), barycentric moments
// and the two folds of the item; the 7 items are summed in order p = 0..6.
// (The touching pairs of the regularizing path go through k_singular.)
template <int KID>
__global__ void k_pair_local(Params P, const int2* __restrict__ pairs, int n, double* __restrict__ out,
                             unsigned long long* errpair) {
  using T = KTraits<KID>;
  using C = ClipCfg<KID>;
  using X = SumIdx<KID>;
  constexpr int NC = T::NC, NC2 = T::NC2, N3 = 3 * NC, NB = 6 * NC;
  __shared__ double sF[7][2 * C::NSIDE];
  const int lane = threadIdx.x;
  for (int pi = blockIdx.x; pi < n; pi += gridDim.x) {
    const int k = pairs[pi].x, l = pairs[pi].y;
    if (lane < 7) {
      const int p = lane;
      double kx[3], ky[3], lx[3], ly[3];
      load_tri(P, k, kx, ky);
      load_tri(P, l, lx, ly);
      const int4 ek = __ldg(&P.elem[k]), el = __ldg(&P.elem[l]);
      const bool touching = k == l || ek.x == el.x || ek.x == el.y || ek.x == el.z || ek.y == el.x ||
                            ek.y == el.y || ek.y == el.z || ek.z == el.x || ek.z == el.y || ek.z == el.z;
      const double rs2 = (touching && P.path == 1) ? P.rskip2 : 0.0;
      const double e1x = kx[1] - kx[0], e2x = kx[2] - kx[0], e1y = ky[1] - ky[0], e2y = ky[2] - ky[0];
      const double x0 = __dadd_rn(__dadd_rn(kx[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
      const double x1 = __dadd_rn(__dadd_rn(ky[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
      double qx[kMaxPoly], qy[kMaxPoly], sx[kMaxPoly], sy[kMaxPoly];
      const int nv = truncate_inner(lx, ly, x0, x1, P.delta, P.ball, sx, sy, qx, qy);
      // the inner element's frame (hat functions)
      const double o0 = lx[0], o1 = ly[0], f1x = lx[1] - lx[0], f1y = ly[1] - ly[0], f2x = lx[2] - lx[0],
                   f2y = ly[2] - ly[0];
      const double idet = 1.0 / cross2(f1x, f2y, f1y, f2x);
      double si[C::NSUM];
#pragma unroll
      for (int i = 0; i < C::NSUM; ++i) si[i] = 0.0;
      for (int t = 1; t < nv - 1; ++t) {
        const double q0x = qx[0], q0y = qy[0];
        const double ax = qx[t] - q0x, ay = qy[t] - q0y, bx = qx[t + 1] - q0x, by = qy[t + 1] - q0y;
        const double jac2 = cross2(ax, by, ay, bx);
        if (!(jac2 > P.drop2)) continue;
        const double v0 = q0x - o0, v1 = q0y - o1;
        const double z1 = (v0 * f2y - v1 * f2x) * idet, z2 = (f1x * v1 - f1y * v0) * idet;
        const double z1a = (ax * f2y - ay * f2x) * idet, z2a = (f1x * ay - f1y * ax) * idet;
        const double z1b = (bx * f2y - by * f2x) * idet, z2b = (f1x * by - f1y * bx) * idet;
        for (int q = 0; q < 7; ++q) {
          const double i0 = c_rule.ip[q][0], i1 = c_rule.ip[q][1];
          const double y0 = fma(bx, i1, fma(ax, i0, q0x)), y1 = fma(by, i1, fma(ay, i0, q0y));
          const double d0 = x0 - y0, d1 = x1 - y1;
          const double r2 = fma(d0, d0, d1 * d1);
          if (rs2 > 0.0) {  // the diagonal-skip predicate in the reference's rounding
            const double ey0 = __dadd_rn(__dadd_rn(q0x, mul(ax, i0)), mul(bx, i1));
            const double ey1 = __dadd_rn(__dadd_rn(q0y, mul(ay, i0)), mul(by, i1));
            if (sumsq(x0 - ey0, x1 - ey1) < rs2) continue;
          }
          double pv[NC2], qv[NC2];
          kval<KID>(P, x0, y0, d0, d1, r2, pv, qv);
          const double wq = c_rule.iw[q] * jac2;
          const double xi1 = fma(i1, z1b, fma(i0, z1a, z1)), xi2 = fma(i1, z2b, fma(i0, z2a, z2));
#pragma unroll
          for (int i = 0; i < C::NCU; ++i) {
            const double tp = wq * pv[X::ucd(i)];
            const double tq = T::SYM ? tp : wq * qv[X::ucd(i)];
            const double g1 = tq * xi1, g2 = tq * xi2;
            si[X::mp(0, i)] += tp;
            if (T::SYM) {
              si[X::mp(1, i)] += g1;
              si[X::mp(2, i)] += g2;
            } else {
              si[X::mp(1, i)] = fma(tp, xi1, si[X::mp(1, i)]);
              si[X::mp(2, i)] = fma(tp, xi2, si[X::mp(2, i)]);
              si[X::mq(0, i)] += tq;
              si[X::mq(1, i)] += g1;
              si[X::mq(2, i)] += g2;
            }
            si[X::mq(3, i)] = fma(g1, xi1, si[X::mq(3, i)]);
            si[X::mq(4, i)] = fma(g1, xi2, si[X::mq(4, i)]);
            si[X::mq(5, i)] = fma(g2, xi2, si[X::mq(5, i)]);
          }
        }
      }
      const double W = c_rule.ow[p] * twice_area(kx, ky);
      item_folds<KID>(W, c_rule.oh[p], si, &sF[p][0], &sF[p][C::NSIDE]);
    }
    __syncwarp();
    // sum the items in order and lay out the dense block: rows / columns are
    // (k's 3 nc dofs, l's 3 nc dofs); F0 -> the k rows, F1 -> the l rows
    double* B = out + (long long)pi * NB * NB;
    const double ls = lab_scale(P, __ldg(&P.elem[k]).w, __ldg(&P.elem[l]).w);
    for (int e = lane; e < NB * NB; e += 32) {
      const int R = e / NB, Cc = e % NB;
      const bool rk = R < N3, ck = Cc < N3;
      const int I = rk ? R : R - N3, J = ck ? Cc : Cc - N3;
      double v = 0.0;
      int g = -1;
      if (rk == ck) {  // own part: the symmetric kk of F0 (k rows) / F1 (l rows)
        const int a = min(I, J), b = max(I, J);
        g = a * N3 - a * (a - 1) / 2 + (b - a);
      } else {
        g = C::NKK + I * N3 + J;
      }
      const int off = rk ? 0 : C::NSIDE;
#pragma unroll 1
      for (int p = 0; p < 7; ++p) v += sF[p][off + g];
      v *= ls;
      B[e] = v;
      report_nonfinite(nonfinite(v), k, l, P.K, errpair);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- per-root reduction
// Merge stage R.  A root's contributions are the blocks of its record sides:
// side A of the records it owns (full list, then clipped list) and side B of
// the records where it is the partner (reverse index), in that fixed order
// (the reference adds them visit by visit into the root's rows).
//  * own block: summed over the sides in a fixed order (thread stride, warp
//    tree, warps in order), E entries at kk_base + rank E;
//  * neighbour blocks: every (side, neighbour dof base w) item carries a
//    column of 3NC x NC values (klv is [J][I]).  A chunk of up to kRootCap
//    items is radix-sorted by w in shared memory (deterministic block sort),
//    equal-w runs are summed in sorted order, and each run becomes the COO
//    entries of the root's in-range rows.  Chunks get their output offset by
//    a decoupled look-back in ticket order (no count pass, no compaction).
// Roots typically have 3-6k items, so one chunk sees every side of its root
// and the reduction is complete per root (cfg2: 251M values -> ~54M entries).
constexpr int kRootThreads = 256, kRootItems = 12, kRootCap = kRootThreads * kRootItems;
// stage-R run entries per record value, for the buffer estimate (cfg2: 0.2);
// a batch that needs more is split
constexpr double kRunFrac = 0.35;
// stage-W CSR entries per record value, for the entry buffer (cfg4 0.012,
// cfg1-3 0.03); a batch that needs more is split
constexpr double kEntFrac = 0.08;

// CSR entries of a batch's rows: a row holds about 0.47 nc x the EPI of a
// root (the partner vertices), so kEntPerEpi leaves headroom; records alone
// under-count in analytic mode, where most visits have none
constexpr double kEntPerEpi = 0.75;
inline long long ent_estimate(const Params& P, long long n_records, long long epi, long long nR) {
  const double E = 9.0 * P.nc * P.nc;
  const double by_rec = kEntFrac * (double)n_records * 2.0 * E;
  const double epi_avg = nR ? (double)epi / (double)nR : 0.0;
  const double by_epi = (double)(P.row_hi - P.row_lo) * (kEntPerEpi * P.nc * epi_avg + 64.0);
  return (long long)std::max(by_rec, by_epi);
}

struct RootIn {
  const int* roots;
  int nR;
  const int* cnt;
  const long long* off;
  long long nF;
  const int2* rec;  // full then clipped records
  // reverse indices (side B by partner root), one per list: per-root ranges
  // and the record's root at each reverse position
  const int* rstartF;
  const int* rstartP;
  const int* partBF;
  const int* partBP;
  // block slots: side A of list record v -> a + v, side B -> b + reverse position
  long long aF, bF, aP, bP;
  int analytic;             // full sides carry no blocks: their terms come from ftab
  const int* inR;           // element -> root rank (-1: not a root of the batch)
  const double* kkv;  // [side][NKK]
  const double* klv;  // [side][3][NVP]
  const int* chunk_first;  // [nR + 1], chunk_first[nR] = number of chunks
  const int* chunk_root;   // [chunks] root rank of each chunk
  const double* own_a2;    // analytic: [nR] sum of the category-0 partners' A2
};
struct RootOut {
  unsigned* ticket;
  unsigned long long* lb;  // [chunks] look-back words: flag << 62 | count
  unsigned long long* keys;
  double* vals;
  long long kk_base;  // root rank i's own block at kk_base + i E
  long long r_base, r_cap;
  int* overflow;
  unsigned long long* total;  // run entries of all chunks (written by the last one)
  unsigned long long* errpair;
};

// A root's record sides in their fixed order: side A of its full records,
// side B of the full records where it is the partner, then the same two for
// the clipped list (the reference adds the visits one by one into the root's
// rows; any fixed order is run-to-run deterministic)
struct RootSides {
  long long f0, fn, fb0, fbn, p0, pn, pb0, pbn;
  __device__ __forceinline__ long long n() const { return fn + fbn + pn + pbn; }
  __device__ __forceinline__ long long nfull() const { return fn + fbn; }
  __device__ __forceinline__ long long slot(const RootIn& I, long long rs) const {
    if (rs < fn) return I.aF + f0 + rs;
    rs -= fn;
    if (rs < fbn) return I.bF + fb0 + rs;
    rs -= fbn;
    if (rs < pn) return I.aP + p0 + rs;
    return I.bP + pb0 + (rs - pn);
  }
  // the other element of that side's pair
  __device__ __forceinline__ int partner(const RootIn& I, long long rs) const {
    if (rs < fn) return __ldg(&I.rec[f0 + rs].y) & kIdMask;
    rs -= fn;
    if (rs < fbn) return __ldg(&I.partBF[fb0 + rs]);
    rs -= fbn;
    if (rs < pn) return __ldg(&I.rec[I.nF + p0 + rs].y) & kIdMask;
    return __ldg(&I.partBP[pb0 + (rs - pn)]);
  }
};

__device__ __forceinline__ RootSides root_sides(const RootIn& I, int i) {
  RootSides R;
  R.f0 = I.off[0 * (long long)(I.nR + 1) + i];
  R.fn = I.cnt[(long long)C_FULL * I.nR + i];
  R.fb0 = I.rstartF[i];
  R.fbn = I.rstartF[i + 1] - R.fb0;
  R.p0 = I.off[1 * (long long)(I.nR + 1) + i];
  R.pn = I.cnt[(long long)C_PART * I.nR + i];
  R.pb0 = I.rstartP[i];
  R.pbn = I.rstartP[i + 1] - R.pb0;
  return R;
}

__global__ void k_root_chunk_map(RootIn I, int* chunk_root) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I.nR) return;
  for (int c = I.chunk_first[i]; c < I.chunk_first[i + 1]; ++c) chunk_root[c] = i;
}

__global__ void k_root_chunks(RootIn I, int* nch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I.nR) return;
  const long long items = 3 * root_sides(I, i).n();
  nch[i] = (int)max(1LL, (items + kRootCap - 1) / kRootCap);
}

template <int NC>
struct RootSmem {
  static constexpr int NV = 3 * NC * NC;  // values of one (side, neighbour dof) item
  using Sort = cub::BlockRadixSort<unsigned, kRootThreads, kRootItems, unsigned>;
  using Scan = cub::BlockScan<int, kRootThreads>;
  union {
    typename Sort::TempStorage sort;
    double red[kRootThreads / 32][9 * NC * NC + 1];
  } u;
  typename Scan::TempStorage scan;
  unsigned last_key[kRootThreads];   // key at each thread's last sorted position
  double cont[kRootThreads][NV + 1]; // each thread's leading partial run (before its first head)
  unsigned cont_pres[kRootThreads];
  unsigned char has_head[kRootThreads];
};

// AN: analytic full sides (nc = 1).  Their own-block term is
// 2 A2_r sw Phi_r * sum A2_n and their neighbour term for row a and dof w is
// -2 A2_r whs_a * sum (A2_n psi_n[b]) (k_elem_factors): one scalar per item,
// kept beside the stored columns (bit 31 of the presence mask) and combined
// at the end of each run.
template <int NC, bool AN>
__global__ void __launch_bounds__(kRootThreads, 3) k_root_reduce(Params P, RootIn I, RootOut O, int key_bits) {
  constexpr int N3 = 3 * NC, E = 9 * NC * NC, NWARP = kRootThreads / 32, NV = N3 * NC, IT = kRootItems;
  constexpr unsigned PT = 1u << 31;  // presence bit of the analytic scalar
  using SM = RootSmem<NC>;
  extern __shared__ __align__(16) unsigned char root_smem[];
  SM& S = *reinterpret_cast<SM*>(root_smem);
  __shared__ int s_chunk;
  __shared__ long long s_base;
  __shared__ unsigned long long s_fl;
  const int t = threadIdx.x, lane = lane_id(), warp = t >> 5;
  if (t == 0) {
    s_chunk = (int)atomicAdd(O.ticket, 1u);
    s_fl = 0;
  }
  __syncthreads();
  const int ch = s_chunk;
  const int nchunks = I.chunk_first[I.nR];
  if (ch >= nchunks) return;  // surplus block of the upper-bound grid
  const int i = I.chunk_root[ch], c = ch - I.chunk_first[i];
  const int k = I.roots[i];
  const RootSides R = root_sides(I, i);
  const long long n_rs = R.n(), nitems = 3 * n_rs, nan_rs = AN ? R.nfull() : 0;
  const int4 dk4 = P.dofs[k];
  const int dka[3] = {dk4.x, dk4.y, dk4.z};
  unsigned inr = 0;  // in-range local rows I = (a, c)
  int nr = 0;
#pragma unroll
  for (int r = 0; r < N3; ++r) {
    const long long row = (long long)NC * dka[r / NC] + r % NC;
    if (row >= P.row_lo && row < P.row_hi) { inr |= 1u << r; ++nr; }
  }
  const double a2r = AN ? __ldg(&P.ftab[k].w) : 0.0;
  // ---- the root's own block (symmetric, packed), by its first chunk
  if (c == 0) {
    constexpr int NKK = Blk<NC>::NKK;
    double acc[NKK + 1];  // [NKK]: sum of the analytic partners' A2
#pragma unroll
    for (int e = 0; e <= NKK; ++e) acc[e] = 0.0;
    unsigned fl = 0;  // presence: some side's value is nonzero
    if (AN) {
      const double4 fr = ld_f4(P.ftab + k);
      const bool rbad = nonfinite(fr.x) | nonfinite(fr.y) | nonfinite(fr.z) | nonfinite(fr.w);
      for (long long rs = t; rs < nan_rs; rs += kRootThreads) {
        const int n = R.partner(I, rs);
        const double4 fn = ld_f4(P.ftab + n);
        acc[NKK] += fn.w;
        fl |= fn.w != 0.0 ? PT : 0u;
        report_nonfinite(rbad | nonfinite(fn.x) | nonfinite(fn.y) | nonfinite(fn.z) | nonfinite(fn.w), k, n, P.K,
                         O.errpair);
      }
    }
#pragma unroll 2
    for (long long rs = nan_rs + t; rs < n_rs; rs += kRootThreads) {
      const double* src = I.kkv + R.slot(I, rs) * NKK;
#pragma unroll
      for (int e = 0; e < NKK; ++e) {
        const double v = __ldg(&src[e]);
        acc[e] += v;
        fl |= (v != 0.0 ? 1u : 0u) << e;
      }
    }
#pragma unroll
    for (int e = 0; e < (AN ? NKK + 1 : NKK); ++e) {
      double v = acc[e];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) S.u.red[warp][e] = v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    if (lane == 0 && fl) atomicOr(&s_fl, (unsigned long long)fl);
    __syncthreads();
    if (t < E) {
      const int rr = t / N3, cc = t % N3;
      const int u = Blk<NC>::sym(min(rr, cc), max(rr, cc));
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) v += S.u.red[w][u];
      bool pres = (s_fl >> u) & 1ull;
      if (AN && (s_fl & PT)) {
        double sa = 0.0, sw = 0.0;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) sa += S.u.red[w][NKK];
#pragma unroll
        for (int p = 0; p < 7; ++p) sw += c_rule.ow[p];
        const double phi = (2.0 * a2r * sw) * (P.kid == 2 ? root_phi<2>(P, k, rr, cc) : root_phi<3>(P, k, rr, cc));
        v = fma(phi, sa, v);
        pres |= phi != 0.0;
      }
      const bool present = I.cnt[(long long)C_KK * I.nR + i] != 0 && pres;
      const long long slot = O.kk_base + (long long)i * E + t;
      put_key(P, O.keys, slot,
              present ? coo_key(P, (long long)NC * dka[rr / NC] + rr % NC, (long long)NC * dka[cc / NC] + cc % NC)
                      : kSentinel);
      O.vals[slot] = present ? (v != 0.0 ? v : -0.0) : 0.0;
    }
    __syncthreads();
  }
  // ---- neighbour items of this chunk: (dof base w, item position) sorted by w
  const long long c0 = (long long)c * kRootCap;
  const int nval = nr ? (int)min((long long)kRootCap, max(0LL, nitems - c0)) : 0;
  unsigned key[IT], col[IT];  // col: the item's position in the chunk (item g = c0 + col: side g / 3, dof g % 3)
  int nseg = 0, hb = 0;
  unsigned heads = 0;
  if (nval) {
    const unsigned PAD = (1u << key_bits) - 1u;
#pragma unroll
    for (int q = 0; q < IT; ++q) {
      const int j = t * IT + q;
      key[q] = PAD;
      col[q] = 0;
      if (j < nval) {
        const long long g = c0 + j, rs = g / 3;
        const int b = (int)(g - 3 * rs);
        const int4 dn = __ldg(&P.dofs[R.partner(I, rs)]);
        key[q] = (unsigned)(b == 0 ? dn.x : (b == 1 ? dn.y : dn.z));
        col[q] = (unsigned)j;
      }
    }
    typename SM::Sort(S.u.sort).Sort(key, col, 0, key_bits);  // blocked: position t IT + q
    S.last_key[t] = key[IT - 1];
    __syncthreads();
    const unsigned prev = t ? S.last_key[t - 1] : ~0u;
    int hc = 0;
#pragma unroll
    for (int q = 0; q < IT; ++q) {
      const int pos = t * IT + q;
      const bool h = pos < nval && key[q] != (q ? key[q - 1] : prev);
      heads |= (h ? 1u : 0u) << q;
      hc += h;
    }
    typename SM::Scan(S.scan).ExclusiveSum(hc, hb, nseg);
    S.has_head[t] = heads != 0;
  }
  // ---- output offset: decoupled look-back over the chunks in ticket order
  const long long count = (long long)nseg * nr * NC;
  if (t == 0) {
    constexpr unsigned long long FA = 1ull << 62, FP = 2ull << 62, VM = (1ull << 62) - 1;
    long long excl = 0;
    if (ch == 0) {
      atomicExch(&O.lb[0], FP | (unsigned long long)count);
    } else {
      atomicExch(&O.lb[ch], FA | (unsigned long long)count);
      for (int j = ch - 1;;) {
        const unsigned long long v = *(volatile unsigned long long*)&O.lb[j];
        const unsigned long long f = v >> 62;
        if (f == 0) continue;
        excl += (long long)(v & VM);
        if (f == 2) break;
        --j;
      }
      atomicExch(&O.lb[ch], FP | (unsigned long long)(excl + count));
    }
    if (ch == nchunks - 1) *O.total = (unsigned long long)(excl + count);
    if (count && excl + count > O.r_cap) atomicExch(O.overflow, 1);
    s_base = excl;
  }
  if (!nval) return;  // block-uniform
  // analytic row factors -2 A2_r whs_a
  double fkl[N3];
#pragma unroll
  for (int r = 0; r < N3; ++r) {
    fkl[r] = 0.0;
    if (AN) {
      double whs = 0.0;
#pragma unroll
      for (int p = 0; p < 7; ++p) whs += c_rule.wh[p][r];
      fkl[r] = -2.0 * a2r * whs;
    }
  }
  // ---- run sums: each thread adds its sorted positions in order; a run that
  // starts in an earlier thread gets this thread's leading piece afterwards
  const int npos = min(IT, max(0, nval - t * IT));
  double acc[NV], acc_t = 0.0;
  unsigned pres = 0;
#pragma unroll
  for (int e = 0; e < NV; ++e) acc[e] = 0.0;
  auto flush = [&](int seg, unsigned w) {  // write run `seg` (complete) of dof base w
    long long pos = O.r_base + s_base + (long long)seg * nr * NC;
#pragma unroll
    for (int r = 0; r < N3; ++r) {
      if (!((inr >> r) & 1u)) continue;
      const long long row = (long long)NC * dka[r / NC] + r % NC - P.row_lo;
#pragma unroll
      for (int d = 0; d < NC; ++d) {
        const int e = d * N3 + r;
        double v = acc[e];
        bool pr = (pres >> e) & 1u;
        if (AN && (pres & PT)) {
          v = fma(fkl[r], acc_t, v);
          pr |= fkl[r] != 0.0;
        }
        put_key(P, O.keys, pos, (unsigned long long)row * (unsigned long long)P.J + (unsigned long long)NC * w + d);
        O.vals[pos] = pr ? (v != 0.0 ? v : -0.0) : 0.0;
        ++pos;
      }
    }
  };
  // the value columns of this thread's stored positions, fetched while the
  // block waits for its output offset
#pragma unroll
  for (int q = 0; q < IT; ++q)
    if (q < npos) {
      const long long g = c0 + col[q], rs = g / 3;
      if (rs >= nan_rs)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(I.klv + R.slot(I, rs) * Blk<NC>::KLS + (g - 3 * rs) * NC));
    }
  __syncthreads();  // s_base, has_head
  const long long base = s_base;
  const bool fits = base + count <= O.r_cap;
  int seg = hb - 1;  // run of the current position (-1: a run begun in an earlier thread)
  unsigned wseg = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    if (q < npos) {
      if ((heads >> q) & 1u) {
        if (seg >= hb) {  // the previous run ended inside this thread
          if (fits) flush(seg, wseg);
        } else {  // leading piece of a run begun earlier
#pragma unroll
          for (int e = 0; e < NV; ++e) S.cont[t][e] = acc[e];
          S.cont[t][NV] = acc_t;
          S.cont_pres[t] = pres;
        }
        ++seg;
        wseg = key[q];
#pragma unroll
        for (int e = 0; e < NV; ++e) acc[e] = 0.0;
        acc_t = 0.0;
        pres = 0;
      }
      const long long g = c0 + col[q], rs = g / 3;
      const int b = (int)(g - 3 * rs);
      if (AN && rs < nan_rs) {
        const double4 fn = ld_f4(P.ftab + R.partner(I, rs));
        const double v = b == 0 ? fn.x : (b == 1 ? fn.y : fn.z);
        acc_t += v;
        pres |= v != 0.0 ? PT : 0u;
      } else {
        const double* src = I.klv + R.slot(I, rs) * Blk<NC>::KLS + b * NC;
#pragma unroll
        for (int e = 0; e < NV; ++e) {  // e = d * N3 + I: row I, column b nc + d
          const double v = __ldg(&src[(e % N3) * Blk<NC>::NVP + e / N3]);
          acc[e] += v;
          pres |= (__double_as_longlong(v) != 0 ? 1u : 0u) << e;
        }
      }
    }
  }
  if (!heads && npos > 0) {  // the whole range continues an earlier run
#pragma unroll
    for (int e = 0; e < NV; ++e) S.cont[t][e] = acc[e];
    S.cont[t][NV] = acc_t;
    S.cont_pres[t] = pres;
  }
  __syncthreads();
  if (heads) {  // the last run begun here may continue into the next threads
    const int ntot = (nval + IT - 1) / IT;
    for (int u = t + 1; u < ntot; ++u) {
      // thread u's leading piece belongs to this run (up to its first head)
      const unsigned uh = S.has_head[u];
#pragma unroll
      for (int e = 0; e < NV; ++e) acc[e] += S.cont[u][e];
      acc_t += S.cont[u][NV];
      pres |= S.cont_pres[u];
      if (uh) break;
    }
    if (fits) flush(seg, wseg);
  }
}

// ---------------------------------------------------------------- row merge
// Merge stage W (replaces stage R + the global sort when every row fits a
// shared-memory table): one CTA per dof base d gathers, for its in-range rows
// NC d + c, every contribution the reference's _merge_triplets
// (assembly.py:137-173) would sum into them -- the own blocks and neighbour
// blocks of the record sides of the batch roots incident to d, the analytic
// full-pair terms and the touching-pair (singular) entries -- into a hash
// table keyed by the column dof base.  Sums are exact 128-bit fixed point
// (value x 2^S, S from a bound of every contribution's magnitude), so their
// result does not depend on the order the threads add them: run-to-run
// deterministic without a sort.  The table is then radix-sorted by column
// in shared memory and each row leaves as one sorted CSR row.  A row whose
// distinct columns outgrow the table is retried with a larger one; beyond
// the largest, the batch falls back to stage R + the global sort.
constexpr unsigned kRowEmpty = 0x7fffffffu;

struct RowIn {
  const int* de_start;
  const int* de_items;
  const int* inR;
  const int* dlist;  // dof bases to process, or nullptr: d_lo + blockIdx.x
  long long d_lo;
  int key_bits;      // bits of the largest dof base + 1 (the empty key sorts last)
  int fill_div;      // tests (NLG_ROW_FILL_DIV): a table overflows at CAP / fill_div columns (0: at 7/8)
  // singular entries sorted by key, and each local row's first position
  const unsigned long long* skey64;
  const unsigned* skey32;
  const double* sval;
  const long long* sstart;
  const unsigned long long* vmax;  // max |stored / singular value| of the batch (stage R)
  const unsigned long long* emax;  // [K] per element: max |value| of its roots' emitted sides
  const unsigned long long* fmax;  // plan bounds of the analytic terms (k_elem_factors)
  Grid G;                          // analytic rows enumerate their category-0 partners
};
struct RowOut {
  int* col;
  double* val;
  long long cap;
  unsigned long long* used;
  long long* roff;  // per local row: first entry in col / val
  int* rcnt;        // per local row: entries
  long long* roff2; // per local row: the second run (columns >= the row's dof base, split rows)
  int* rcnt2;
  int* ovf;         // dof bases whose table overflowed
  unsigned* novf;
  int split;        // 0: all columns; 1 / 2: only column bases < / >= d (rows too wide for one table)
};

// Analytic rows (kid 2 / 3 on the standard path): the category-0 visits of
// the incident roots have no records.  The row's CTA enumerates the grid
// around its dof, and for each candidate element n sums the incident roots'
// row factors over the visits (k, n) of category 0 (exact reference
// predicates): one table add per column of n instead of one per visit.
constexpr int kMaxInc = 8;    // incident roots of a dof per enumeration pass
constexpr int kMaxRowsG = 48; // grid cell rows of one enumeration (grid pitch >= reach / 16)
constexpr int kRimCap = 8192; // queued rim candidates of one enumeration (beyond: handled in place)
struct IncRoot {
  double cx, cy, r;
  double kx[3], ky[3], xk[7], yk[7];
  double fkl;     // -2 A2_k sum_p w_p H_pa: the visit's neighbour-block row factor
  int k;          // element, -1: not a root of the batch
};

struct IncSide {  // an incident root of the row: its record sides, dofs, corner
  RootSides R;
  unsigned dk[3];
  int k, a, rank, on;  // on: its own block is emitted by this batch
};

template <int NC, int CAP, int TH>
struct RowSmem {
  using Sort = cub::BlockRadixSort<unsigned, TH, CAP / TH, unsigned>;
  using Scan = cub::BlockScan<int, TH>;
  unsigned key[CAP];                      // column dof base (bit 31: present, nc = 1)
  unsigned pres[NC == 1 ? 1 : CAP];       // nc = 2: presence bit per (c, d) component
  unsigned acc[CAP][NC * NC][3];
  union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } u;
  IncRoot inc[kMaxInc];
  IncSide isd[kMaxInc];                       // stored sides: the group's incident roots
  long long spre[kMaxInc + 1];                // ... and the prefix of their side counts
  unsigned ownacc[kMaxInc][3][NC * NC][3];    // ... and their own-block sums (96-bit fixed point)
  unsigned ownpres[kMaxInc];
  int gr0[kMaxRowsG], gr1[kMaxRowsG], gpre[kMaxRowsG + 1];  // column ranges of the enumeration
  int er0[2 * kMaxRowsG], epre[2 * kMaxRowsG + 1];          // element ranges of the same cell rows (two per row)
  int ngr;
  unsigned long long bnd;  // the row's bound (incident elements' emitted values)
  double gvx, gvy, grmax, gsum_all;  // the dof's vertex, largest incident radius, sum of all row factors
  int gpres_all;
  int nrim;
  int rimq[kRimCap];                  // candidates near the rim of the group's balls (scan slots)
  int used, ovf;
  long long base[NC];
};

template <int NC, int CAP, int TH, bool AN, bool SPL = false>
__global__ void __launch_bounds__(TH) k_row_asm(Params P, RootIn I, RowIn W, RowOut O) {
  constexpr int NC2 = NC * NC, IT = CAP / TH;
  constexpr int LOG2CAP = CAP == 512 ? 9 : CAP == 1024 ? 10 : CAP == 2048 ? 11 : CAP == 4096 ? 12 : 13;
  static_assert((1 << LOG2CAP) == CAP, "CAP must be a power of two in [512, 8192]");
  using SM = RowSmem<NC, CAP, TH>;
  extern __shared__ __align__(16) unsigned char row_smem[];
  SM& S = *reinterpret_cast<SM*>(row_smem);
  const int t = threadIdx.x;
  const long long d = W.dlist ? (long long)W.dlist[blockIdx.x] : W.d_lo + blockIdx.x;
  for (int i = t; i < CAP; i += TH) {
    S.key[i] = kRowEmpty;
    if (NC > 1) S.pres[i] = 0;
#pragma unroll
    for (int e = 0; e < NC2; ++e) S.acc[i][e][0] = S.acc[i][e][1] = S.acc[i][e][2] = 0;
  }
  if (t == 0) {
    S.used = 0;
    S.ovf = 0;
  }
  // fixed-point scale from a bound of every contribution's magnitude
  double whsmax = 0.0, sw = 0.0;
#pragma unroll
  for (int p = 0; p < 7; ++p) sw += c_rule.ow[p];
  // the row's bound: its incident elements' (every contribution to row d
  // comes from a visit or touching pair of an element containing d)
  if (t < 32) {
    unsigned long long b = 0;
    for (int i = W.de_start[d] + t; i < W.de_start[d + 1]; i += 32) b = max(b, W.emax[W.de_items[i] >> 2]);
    for (int o = 16; o; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (t == 0) S.bnd = b;
  }
  __syncthreads();
  double bound = __longlong_as_double((long long)S.bnd);
  double fa2 = 0.0;
  if (AN) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double wsum = 0.0;
#pragma unroll
      for (int p = 0; p < 7; ++p) wsum += c_rule.wh[p][a];
      whsmax = fmax(whsmax, wsum);
    }
    fa2 = __longlong_as_double((long long)W.fmax[0]);
    const double fg = __longlong_as_double((long long)W.fmax[1]);
    const double fphi = __longlong_as_double((long long)W.fmax[2]);
    // neighbour terms: up to kMaxInc roots' factors per column of a partner
    const double fabsmax = __longlong_as_double((long long)W.fmax[3]);
    // neighbour terms: up to kMaxInc roots' factors x a column's factor H
    // (up to 64 incident elements)
    bound = fmax(bound, 2.0 * fa2 * whsmax * fg * kMaxInc * 64.0);
    bound = fmax(bound, 2.0 * fa2 * sw * fphi * fa2 * 0x1p17);  // own term: A2_r Phi_r x (sum of up to 2^17 A2_n)
    // a clipped record side's entries: sums over the outer points (weights
    // sw A2) of integrals of |f| x hats over part of the inner triangle
    bound = fmax(bound, 8.0 * sw * fa2 * fa2 * fabsmax);
  }
  const bool bok = bound > 0.0 && bound <= 1e300;
  const int be = bok ? ilogb(bound) + 1 : 0;
  const double scale = bok ? ldexp(1.0, kFixBits - be) : 1.0, inv = bok ? ldexp(1.0, be - kFixBits) : 1.0;
  unsigned inr = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long row = NC * d + c;
    if (row >= P.row_lo && row < P.row_hi) inr |= 1u << c;
  }
  __syncthreads();
  // slot of column dof base w (inserted if new); -1 once the table overflowed
  // (nc = 1: a key is inserted with its presence bit -- only present
  // contributions reach the table)
  constexpr unsigned kIns = NC == 1 ? 0x80000000u : 0u;
  auto slot_of = [&](unsigned w) -> int {
    unsigned h = (w * 2654435761u) >> (32 - LOG2CAP);
    for (int probe = 0; probe < CAP; ++probe) {
      const unsigned kk = *(volatile unsigned*)&S.key[h] & 0x7fffffffu;
      if (kk == w) return (int)h;
      if (kk == kRowEmpty) {
        if (*(volatile int*)&S.ovf) return -1;
        const unsigned old = atomicCAS(&S.key[h], kRowEmpty, w | kIns);
        if (old == kRowEmpty) {
          if (atomicAdd(&S.used, 1) >= (W.fill_div ? CAP / W.fill_div : CAP - CAP / 8)) S.ovf = 1;
          return (int)h;
        }
        if ((old & 0x7fffffffu) == w) return (int)h;
      }
      h = (h + 1) & (CAP - 1);
    }
    S.ovf = 1;
    return -1;
  };
  auto mark = [&](int h, int comp) {
    if (NC == 1) {
      // (set at insertion)
    } else {
      if (!((*(volatile unsigned*)&S.pres[h] >> comp) & 1u)) atomicOr(&S.pres[h], 1u << comp);
    }
  };
  auto add_fix = [&](unsigned w, int comp, fix_t f, bool pres) {
    if (!pres) return;
    if (SPL && ((w < (unsigned)d) != (O.split == 1))) return;  // the other half's column
    const int h = slot_of(w);
    if (h < 0) return;
    fix_atomic(S.acc[h][comp], f);
    mark(h, comp);
  };
  auto add = [&](unsigned w, int comp, double v, bool pres) {
    if (!pres || !(v == v) || fabs(v) > 1e300) return;  // absent; nonfinite values are reported elsewhere
    add_fix(w, comp, fix_of(v, scale), true);
  };
  if (inr) {
    // ---- the stored record sides of the batch roots incident to d
    // (analytic mode: the clipped sides only; category-0 visits follow below).
    // The sides of up to kMaxInc incident roots form one flat index space,
    // so every thread of the CTA has work until the last few sides.  Own-block
    // values are summed in fixed point (exact: neither the CTA size nor the
    // order of the sides, which depends on the batch, matters): per warp and
    // root with one reduction, then into the group's accumulators.
    const int e0 = W.de_start[d], e1 = W.de_start[d + 1];
    for (int g0 = e0; g0 < ((P.dbg & 4) ? e0 : e1); g0 += kMaxInc) {  // (NLG_DEBUG & 4: timing experiments)
      const int ng = min(e1 - g0, kMaxInc);
      __syncthreads();
      if (t < ng) {
        IncSide& Q = S.isd[t];
        const int it = __ldg(&W.de_items[g0 + t]);
        const int k = it >> 2;
        const int rank = __ldg(&W.inR[k]);
        Q.k = k;
        Q.a = it & 3;
        Q.rank = rank;
        Q.on = 0;
        RootSides R;
        R.f0 = R.fn = R.fb0 = R.fbn = R.p0 = R.pn = R.pb0 = R.pbn = 0;
        if (rank >= 0) {
          R = root_sides(I, rank);
          const int4 dk4 = __ldg(&P.dofs[k]);
          Q.dk[0] = (unsigned)dk4.x;
          Q.dk[1] = (unsigned)dk4.y;
          Q.dk[2] = (unsigned)dk4.z;
          Q.on = I.cnt[(long long)C_KK * I.nR + rank] != 0;
        }
        Q.R = R;
      }
      for (int i = t; i < kMaxInc * 3 * NC2 * 3; i += TH) (&S.ownacc[0][0][0][0])[i] = 0;
      if (t < kMaxInc) S.ownpres[t] = 0;
      __syncthreads();
      if (t == 0) {
        long long run = 0;
        for (int i = 0; i < ng; ++i) {
          S.spre[i] = run;
          run += S.isd[i].R.n();
        }
        S.spre[ng] = run;
      }
      __syncthreads();
      const long long total = S.spre[ng];
      int i = 0;
      for (long long fb = t & ~31; fb < total; fb += TH) {  // (warp-uniform trip count)
        if (*(volatile int*)&S.ovf) break;  // this table is too small: retried with a larger one
        const long long f = fb + (t & 31);
        const bool valid = f < total;
        fix_t own[3][NC2];
        unsigned opres = 0;  // bit b * NC2 + comp
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int e = 0; e < NC2; ++e) own[b][e] = 0;
        if (valid) {
          while (f >= S.spre[i + 1]) ++i;
          const IncSide& Q = S.isd[i];
          const RootSides R = Q.R;
          const long long rs = f - S.spre[i];
          const int a = Q.a;
          const int n = R.partner(I, rs);
          const int4 dn4 = __ldg(&P.dofs[n]);
          const unsigned dn[3] = {(unsigned)dn4.x, (unsigned)dn4.y, (unsigned)dn4.z};
          const long long slot = R.slot(I, rs);
          const double* kk = I.kkv + slot * Blk<NC>::NKK;
          const double* kl = I.klv + slot * Blk<NC>::KLS;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (!((inr >> c) & 1u)) continue;
            const int Ir = a * NC + c;
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
              for (int dd = 0; dd < NC; ++dd) {
                const int Jc = b * NC + dd;
                const double vo = __ldg(&kk[Blk<NC>::sym(min(Ir, Jc), max(Ir, Jc))]);
                const double vn = __ldg(&kl[Blk<NC>::kl(Ir, Jc)]);
                if (vo != 0.0 && vo == vo && fabs(vo) <= 1e300) {
                  own[b][c * NC + dd] = fix_of(vo, scale);
                  opres |= 1u << (b * NC2 + c * NC + dd);
                }
                add(dn[b], c * NC + dd, vn, __double_as_longlong(vn) != 0);
              }
          }
        }
        // own partials: one warp reduction per root present in the warp
        unsigned rem = __ballot_sync(0xffffffffu, valid);
        while (rem) {
          const int leader = __ffs(rem) - 1;
          const int il = __shfl_sync(0xffffffffu, i, leader);
          const unsigned grp = __ballot_sync(0xffffffffu, valid && i == il);
          if (valid && i == il) {
            const unsigned gp = __reduce_or_sync(grp, opres);
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
              for (int e = 0; e < NC2; ++e) {
                if (!((gp >> (b * NC2 + e)) & 1u)) continue;  // group-uniform
                const fix_t fs = fix_group_sum(grp, own[b][e]);
                if ((t & 31) == leader) fix_atomic(S.ownacc[il][b][e], fs);
              }
            if ((t & 31) == leader && gp) atomicOr(&S.ownpres[il], gp);
          }
          rem &= ~grp;
        }
      }
      __syncthreads();
      // the group's own blocks -> table
      for (int q = t; q < ng * 3 * NC2; q += TH) {
        const int gi = q / (3 * NC2), b = (q / NC2) % 3, e = q % NC2;
        const IncSide& Q = S.isd[gi];
        if (!Q.on || !((S.ownpres[gi] >> (b * NC2 + e)) & 1u)) continue;
        const unsigned* c = S.ownacc[gi][b][e];
        const fix_t f = (fix_t)(((unsigned __int128)c[2] << 64 | (unsigned __int128)c[1] << 32 | c[0]) << 32) >> 32;
        add_fix(Q.dk[b], e, f, true);
      }
      if (AN && t < 3 * ng) {
        // analytic own terms: 2 A2_k sw Phi_k[a][b] x (sum of the category-0
        // partners' A2, summed exactly by the candidate fill pass)
        const IncSide& Q = S.isd[t / 3];
        const int b = t % 3;
        if (Q.on) {
          const double sa_d = __ldg(&I.own_a2[Q.rank]);
          if (sa_d != 0.0) {
            const double fown = (2.0 * __ldg(&P.ftab[Q.k].w) * sw) *
                                (P.kid == 2 ? root_phi<2>(P, Q.k, Q.a, b) : root_phi<3>(P, Q.k, Q.a, b));
            add(Q.dk[b], 0, fown * sa_d, fown != 0.0);
          }
        }
      }
    }
    if constexpr (AN) {
      // ---- category-0 visits of the incident roots, by enumeration
      for (int g0 = e0; g0 < ((P.dbg & 8) ? e0 : e1); g0 += kMaxInc) {
        const int ng = min(e1 - g0, kMaxInc);
        __syncthreads();
        if (t < ng) {
          IncRoot& Rt = S.inc[t];
          const int it = __ldg(&W.de_items[g0 + t]);
          const int k = it >> 2, a = it & 3;
          const int rank = __ldg(&W.inR[k]);
          Rt.k = rank >= 0 && I.cnt[(long long)C_KK * I.nR + rank] != 0 ? k : -1;
          const double2 ck = __ldg(&P.ctr[k]);
          Rt.cx = ck.x;
          Rt.cy = ck.y;
          Rt.r = __ldg(&P.rad[k]);
          load_tri(P, k, Rt.kx, Rt.ky);
          tri_points(Rt.kx, Rt.ky, Rt.xk, Rt.yk);
          double wsum = 0.0;
#pragma unroll
          for (int p = 0; p < 7; ++p) wsum += c_rule.wh[p][a];
          Rt.fkl = -2.0 * __ldg(&P.ftab[k].w) * wsum;
        }
        __syncthreads();
        if (t == 0) {
          // the vertex of d (corner a of the first incident element): every
          // incident root's barycentre lies within its radius of it
          {
            const int it = __ldg(&W.de_items[g0]);
            const int4 e4 = __ldg(&P.elem[it >> 2]);
            const int a0 = it & 3;
            const double2 v = __ldg(&P.vtx[a0 == 0 ? e4.x : (a0 == 1 ? e4.y : e4.z)]);
            S.gvx = v.x;
            S.gvy = v.y;
            double rm = 0.0, gs = 0.0;
            int gp = 0;
            for (int i = 0; i < ng; ++i) {
              if (S.inc[i].k < 0) continue;
              rm = fmax(rm, S.inc[i].r);
              gs += S.inc[i].fkl;
              gp |= S.inc[i].fkl != 0.0;
            }
            S.grmax = rm;
            S.gsum_all = gs;
            S.gpres_all = gp;
          }
          S.nrim = 0;
        }
        __syncthreads();
        {
          // cell rows within the reach of any contribution,
          // |x_c - v| <= delta (1 + 1e-9) + r_max(group) + 2 r_max: thread y
          // takes row y -- its column range and (phase B) its element ranges.
          // Cells wholly inside the radius where every corner of every
          // element is a deep column (and clear of the near zone around v)
          // hold nothing for phase B: they split the row's elements in two.
          const double cx = S.gvx, cy = S.gvy, R = P.delta * (1.0 + 1e-9) + S.grmax + 2.0 * W.G.rmax;
          int iy = (int)floor((cy - W.G.oy) / W.G.cs);
          iy = min(max(iy, 0), W.G.ny - 1);
          const int span = (int)ceil(R / W.G.cs);
          const int y0 = max(iy - span, 0), nrow = min(min(iy + span, W.G.ny - 1) - y0 + 1, kMaxRowsG);
          if (t < nrow) {
            const int yy = y0 + t;
            int c0 = 0, c1 = 0, ea0 = 0, ea1 = 0, eb0 = 0, eb1 = 0;
            const double ylo = W.G.oy + yy * W.G.cs, yhi = ylo + W.G.cs;
            const double dy = cy < ylo ? ylo - cy : (cy > yhi ? cy - yhi : 0.0);
            if (dy <= R) {
              const double hw = sqrt(R * R - dy * dy);
              const int x0 = max((int)floor((cx - hw - W.G.ox) / W.G.cs), 0);
              const int x1 = min((int)floor((cx + hw - W.G.ox) / W.G.cs), W.G.nx - 1);
              if (x0 <= x1) {
                c0 = W.G.cstart[yy * W.G.nx + x0];
                c1 = W.G.cstart[yy * W.G.nx + x1 + 1];
                ea0 = W.G.start[yy * W.G.nx + x0];
                ea1 = eb0 = eb1 = W.G.start[yy * W.G.nx + x1 + 1];
                const double mrg = W.G.rmax * (1.0 + 1e-9) + 1e-9 * P.delta;
                const double rin = P.delta - 2.0 * S.grmax - 2.0 * W.G.rmax - 1e-12 * (P.delta + 4.0 * W.G.rmax) - mrg;
                const double rn = 2.0 * W.G.rmax * (1.0 + 1e-9) + mrg;
                const double dym = fmax(fabs(ylo - cy), fabs(yhi - cy));
                if (rin > 0.0 && dym < rin && dy > rn) {
                  const double hwd = sqrt(rin * rin - dym * dym);
                  const int xa = max((int)ceil((cx - hwd - W.G.ox) / W.G.cs), x0);
                  const int xb = min((int)floor((cx + hwd - W.G.ox) / W.G.cs) - 1, x1);
                  if (xa <= xb) {
                    ea1 = W.G.start[yy * W.G.nx + xa];
                    eb0 = W.G.start[yy * W.G.nx + xb + 1];
                  }
                }
              }
            }
            S.gr0[t] = c0;
            S.gr1[t] = c1;
            S.er0[2 * t] = ea0;
            S.er0[2 * t + 1] = eb0;
            S.epre[2 * t] = ea1 - ea0;      // (counts; prefixed below)
            S.epre[2 * t + 1] = eb1 - eb0;
          }
          __syncthreads();
          if (t == 0) {
            int tot = 0, etot = 0;
            for (int r = 0; r < nrow; ++r) {
              S.gpre[r] = tot;
              tot += S.gr1[r] - S.gr0[r];
            }
            S.gpre[nrow] = tot;
            for (int r = 0; r < 2 * nrow; ++r) {
              const int c = S.epre[r];
              S.epre[r] = etot;
              etot += c;
            }
            S.epre[2 * nrow] = etot;
            S.ngr = nrow;
          }
        }
        __syncthreads();
        const int ngr = S.ngr, tot = S.gpre[ngr];
        const double tc2 = (P.delta * (1.0 + 1e-9)) * (P.delta * (1.0 + 1e-9));  // beyond: neither full nor all-inside
        const double gvx = S.gvx, gvy = S.gvy, grm = S.grmax, gsum_all = S.gsum_all;
        const bool gpres_all = S.gpres_all != 0;
        const double geta = 1e-12 * (P.delta + 4.0 * W.G.rmax);
        // element level: every visit (k, n) of the group full when
        // |v - c_n| + 2 r_max(group) + r_n <= delta - margin (|c_k - v| <= r_k);
        // none full or all-inside when |v - c_n| > delta (1 + 1e-9) + r_max(group)
        const double eout = P.delta * (1.0 + 1e-9) + grm, eout2 = eout * eout;
        // column level (|c_n - x_c| <= r_n for each element n at column c):
        // every element of the column deep, and none of them in the group
        // (those contain v, so lie within 2 r_max of it)
        const double cin = P.delta - 2.0 * grm - 2.0 * W.G.rmax - geta, cin2 = cin > 0.0 ? cin * cin : -1.0;
        const double cnear = 2.0 * W.G.rmax * (1.0 + 1e-9), cnear2 = cnear * cnear;
        // G(n) = sum of the row factors of the group's category-0 visits (k, n)
        auto elem_g = [&](int n, int4 el, double2 cl, double rl, double dv2, double& gs) -> bool {
          const double gin = P.delta - 2.0 * grm - rl - geta;
          bool deep = gin > 0.0 && dv2 < gin * gin;
          for (int i = 0; i < ng && deep; ++i) deep = S.inc[i].k != n;
          if (deep) {
            gs = gsum_all;
            return gpres_all;
          }
          double g = 0.0;
          bool pres = false;
#pragma unroll 1
          for (int i = 0; i < ng; ++i) {
            const IncRoot& Rt = S.inc[i];
            if (Rt.k < 0 || Rt.k == n) continue;
            VisitDist D(sumsq(Rt.cx - cl.x, Rt.cy - cl.y));
            if (D.d2 > tc2) continue;
            bool cat0 = D.within(Rt.r, rl, P.delta);
            if (!cat0 && P.ball != 2) cat0 = pair_all_in_el(P, Rt.kx, Rt.ky, Rt.xk, Rt.yk, el);
            if (cat0) {
              g += Rt.fkl;
              pres |= Rt.fkl != 0.0;
            }
          }
          gs = g;
          return pres;
        };
        // a column is "deep" when every element at it is a full partner of
        // every group root, and none of them is in the group: one term
        // gsum_all x H.  The same expression decides it for a column of phase A
        // and for an element's corner in phase B (same vertex coordinates).
        auto col_deep = [&](double dc2) -> bool { return dc2 < cin2 && dc2 > cnear2; };
        // an element with a corner at a column that is not deep: G(n) once,
        // then one term per such corner
        auto rim_elem = [&](int j) {
          const int4 el = W.G.gel[j];
          const double2 cl = W.G.gctr[j];
          const double rl = W.G.grad[j];
          double gs = 0.0;
          if (!elem_g(__ldg(&W.G.items[j]), el, cl, rl, sumsq(gvx - cl.x, gvy - cl.y), gs)) return;
          const double4 f = ld_f4(W.G.gft + j);
          const int4 dn = __ldg(&W.G.gdof[j]);
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double2 v = __ldg(&P.vtx[b == 0 ? el.x : (b == 1 ? el.y : el.z)]);
            if (col_deep(sumsq(gvx - v.x, gvy - v.y))) continue;
            const double fb = b == 0 ? f.x : (b == 1 ? f.y : f.z);
            add((unsigned)(b == 0 ? dn.x : (b == 1 ? dn.y : dn.z)), 0, gs * fb, fb != 0.0);
          }
        };
        // phase A: every deep column (all its elements full partners of every
        // group root): gsum_all x H
        for (int q = t, r = 0; q < tot; q += TH) {  // (r: the cell row of q, kept across iterations)
          if (*(volatile int*)&S.ovf) break;
          while (q >= S.gpre[r + 1]) ++r;
          const int jv = S.gr0[r] + (q - S.gpre[r]);
          const double4 cp = ld_f4(W.G.cpos + jv);
          if (col_deep(sumsq(gvx - cp.x, gvy - cp.y)))
            add((unsigned)__ldg(&W.G.cid[jv]), 0, gsum_all * cp.z, gpres_all && cp.w != 0.0);
        }
        // phase B: the elements with a corner at another column, queued so
        // their pair tests run densely.  An element whose corners (within r_n
        // of its barycentre) all lie strictly between the two radii has only
        // deep columns; one beyond eout has no category-0 visit.
        const int etot = S.epre[2 * ngr];
        for (int q = t, r = 0; q < etot; q += TH) {
          if (*(volatile int*)&S.ovf) break;
          while (q >= S.epre[r + 1]) ++r;
          const int j = S.er0[r] + (q - S.epre[r]);
          const double2 cl = W.G.gctr[j];
          const double rl = W.G.grad[j] * (1.0 + 1e-9) + 1e-9 * P.delta;
          const double dv2 = sumsq(gvx - cl.x, gvy - cl.y);
          if (dv2 > eout2) continue;
          const double hi = cin - rl, lo = cnear + rl;
          if (hi > 0.0 && dv2 < hi * hi && dv2 > lo * lo) continue;
          const int slot = atomicAdd(&S.nrim, 1);
          if (slot < kRimCap) S.rimq[slot] = j;
          else rim_elem(j);  // (queue full: in place)
        }
        __syncthreads();
        const int nrim = min(S.nrim, kRimCap);
        for (int q = t; q < nrim; q += TH) {
          if (*(volatile int*)&S.ovf) break;
          rim_elem(S.rimq[q]);
        }
      }
    }
    // ---- touching-pair (singular) entries of the rows
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (!((inr >> c) & 1u)) continue;
      const long long lr = NC * d + c - P.row_lo;
      const long long s0 = W.sstart[lr], s1 = W.sstart[lr + 1];
      for (long long i = s0 + t; i < s1; i += TH) {
        const unsigned long long key = W.skey64 ? W.skey64[i] : (unsigned long long)W.skey32[i];
        const long long col = (long long)(key % (unsigned long long)P.J);
        const double v = W.sval[i];
        add((unsigned)(col / NC), c * NC + (int)(col % NC), v, __double_as_longlong(v) != 0);
      }
    }
  }
  __syncthreads();
  if (S.ovf) {
    if (t == 0) O.ovf[atomicAdd(O.novf, 1u)] = (int)d;
    return;
  }
  if (P.dbg & 16) return;  // (timing experiments)
  // ---- sort the table by column and write each row
  unsigned key[IT], sl[IT];
  const unsigned PAD = (1u << W.key_bits) - 1u;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const int i = t * IT + q;
    const unsigned kk = S.key[i] & 0x7fffffffu;
    key[q] = kk == kRowEmpty ? PAD : kk;
    sl[q] = (unsigned)i;
  }
  __syncthreads();
  typename SM::Sort(S.u.sort).Sort(key, sl, 0, W.key_bits);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    if (!((inr >> c) & 1u)) continue;  // block-uniform
    int cntq = 0;
#pragma unroll
    for (int q = 0; q < IT; ++q) {
      if (key[q] == PAD) continue;
      const unsigned pm = NC == 1 ? (S.key[sl[q]] >> 31) : (S.pres[sl[q]] >> (c * NC)) & ((1u << NC) - 1u);
      cntq += __popc(pm);
    }
    int pre = 0, tot = 0;
    typename SM::Scan(S.u.scan).ExclusiveSum(cntq, pre, tot);
    if (t == 0) {
      const long long b0 = (long long)atomicAdd(O.used, (unsigned long long)tot);
      S.base[c] = b0;
      const long long lr = NC * d + c - P.row_lo;
      if (O.split == 2) {
        O.roff2[lr] = b0;
        O.rcnt2[lr] = tot;
      } else {
        O.roff[lr] = b0;
        O.rcnt[lr] = tot;
      }
    }
    __syncthreads();
    long long pos = S.base[c] + pre;
    if (S.base[c] + tot <= O.cap) {
#pragma unroll
      for (int q = 0; q < IT; ++q) {
        if (key[q] == PAD) continue;
        const int h = (int)sl[q];
        const unsigned pm = NC == 1 ? (S.key[h] >> 31) : (S.pres[h] >> (c * NC)) & ((1u << NC) - 1u);
#pragma unroll
        for (int dd = 0; dd < NC; ++dd) {
          if (!((pm >> dd) & 1u)) continue;
          O.col[pos] = (int)(NC * key[q] + dd);
          O.val[pos] = fix_val3(S.acc[h][c * NC + dd], inv);
          ++pos;
        }
      }
    }
    __syncthreads();
  }
}

__global__ void k_add_int(int* a, const int* __restrict__ b, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] += b[i];
}
__global__ void k_sub_int(int* a, const int* __restrict__ b, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] -= b[i];
}

// CSR of the batch from the per-row entry runs: one warp per row
__global__ void k_row_gather(const long long* __restrict__ roff, const int* __restrict__ rcnt,
                             const long long* __restrict__ roff2, const int* __restrict__ rcnt2,
                             const long long* __restrict__ indptr, long long nrows, const int* __restrict__ col,
                             const double* __restrict__ val, int* indices, double* data) {
  const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  const long long src = roff[r], dst = indptr[r];
  const int n = rcnt[r];
  for (int i = lane_id(); i < n; i += 32) {
    indices[dst + i] = col[src + i];
    data[dst + i] = val[src + i];
  }
  // split rows: the columns >= the row's dof base follow (both runs sorted)
  const long long src2 = roff2[r];
  const int n2 = rcnt2[r];
  for (int i = lane_id(); i < n2; i += 32) {
    indices[dst + n + i] = col[src2 + i];
    data[dst + n + i] = val[src2 + i];
  }
}

// first sorted singular entry of each local row (keys row_local * J + col)
template <typename KT>
__global__ void k_row_starts(const KT* __restrict__ key, long long n, long long nrows, long long J, long long* start) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r > nrows) return;
  const unsigned long long want = (unsigned long long)r * (unsigned long long)J;
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    const KT k = key[mid];
    const bool less = k != key_sentinel<KT>() && (unsigned long long)k < want;
    if (less) lo = mid + 1; else hi = mid;
  }
  start[r] = lo;
}

// ---------------------------------------------------------------- singular pairs
constexpr int kSingThreads = 32;  // threads per touching pair (points strided over them)

struct SingRule {
  const double* __restrict__ xs;
  const double* __restrict__ ys;
  const double* __restrict__ w;
  const double* __restrict__ hx;
  const double* __restrict__ hy;
  int n;
};

template <int U, int NC, bool SYM>
struct SingAcc {
  static constexpr int UN = U * NC;
  static constexpr int N = SYM ? UN * (UN + 1) / 2 : UN * UN;
  __device__ static constexpr int idx(int i, int j) {
    return SYM ? (i <= j ? i * UN - i * (i - 1) / 2 + (j - i) : j * UN - j * (j - 1) / 2 + (i - j))
               : i * UN + j;
  }
};

// FAM 0 identical (U = 3), 1 edge (U = 4, DG 6), 2 vertex (U = 5, DG 6);
// frames and union tables follow _engine._visit_pair :230-308.
template <int KID, int FAM, int U>
__global__ void __launch_bounds__(kSingThreads) k_singular(Params P, const int2* __restrict__ list,
                                                  long long n, SingRule R,
                                                  unsigned long long* keys, double* vals,
                                                  long long cbase, unsigned long long* counters,
                                                  unsigned long long* errpair, unsigned long long* vmax,
                                                  unsigned long long* emax) {
  using T = KTraits<KID>;
  constexpr int NC = T::NC, UN = U * NC;
  using A = SingAcc<U, NC, T::SYM>;
  constexpr int SLOTS = 36 * NC * NC;
  __shared__ double sTA[3][2], sTB[3][2], sScale;
  __shared__ double sPm[kSingThreads / 32];  // the pair's largest |entry| (the elements' merge bounds)
  __shared__ int sMk[6], sMl[6], sUb[6];
  __shared__ double red[kSingThreads / 32][A::N];
  long long npts = 0;
  double vm = 0.0;
  for (long long pi = blockIdx.x; pi < n; pi += gridDim.x) {
    const int k = list[pi].x, l = list[pi].y;
    if (threadIdx.x == 0) {
      const int4 ek = P.elem[k], el = P.elem[l];
      const int4 dk = P.dofs[k], dl = P.dofs[l];
      const int ea[3] = {ek.x, ek.y, ek.z}, eb[3] = {el.x, el.y, el.z};
      const int da[3] = {dk.x, dk.y, dk.z}, db[3] = {dl.x, dl.y, dl.z};
      int permk[3] = {0, 1, 2}, perml[3] = {0, 1, 2};
      int a0 = -1, a1 = -1, b0 = -1, b1 = -1, ns = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          if (ea[a] == eb[b]) {
            if (ns == 0) { a0 = a; b0 = b; } else if (ns == 1) { a1 = a; b1 = b; }
            ++ns;
          }
      if (FAM == 0) {
        for (int m = 0; m < 3; ++m) { sMk[m] = m; sMl[m] = m; sUb[m] = da[m]; }
      } else if (FAM == 1) {
        if (ea[a0] > ea[a1]) { int t = a0; a0 = a1; a1 = t; t = b0; b0 = b1; b1 = t; }
        permk[0] = a0; permk[1] = a1; permk[2] = 3 - a0 - a1;
        perml[0] = b0; perml[1] = b1; perml[2] = 3 - b0 - b1;
        const int mk[4] = {0, 1, 2, -1}, ml[4] = {0, 1, -1, 2};
        for (int m = 0; m < 4; ++m) { sMk[m] = mk[m]; sMl[m] = ml[m]; }
        sUb[0] = da[permk[0]]; sUb[1] = da[permk[1]]; sUb[2] = da[permk[2]]; sUb[3] = db[perml[2]];
      } else {
        permk[0] = a0; permk[1] = (a0 + 1) % 3; permk[2] = (a0 + 2) % 3;
        perml[0] = b0; perml[1] = (b0 + 1) % 3; perml[2] = (b0 + 2) % 3;
        const int mk[5] = {0, 1, 2, -1, -1}, ml[5] = {0, -1, -1, 1, 2};
        for (int m = 0; m < 5; ++m) { sMk[m] = mk[m]; sMl[m] = ml[m]; }
        sUb[0] = da[permk[0]]; sUb[1] = da[permk[1]]; sUb[2] = da[permk[2]];
        sUb[3] = db[perml[1]]; sUb[4] = db[perml[2]];
      }
      if (FAM != 0 && U == 6) {  // DG union: all six local hats
        for (int m = 0; m < 3; ++m) {
          sMk[m] = m; sMk[3 + m] = -1; sMl[m] = -1; sMl[3 + m] = m;
          sUb[m] = da[permk[m]]; sUb[3 + m] = db[perml[m]];
        }
      }
      for (int m = 0; m < 3; ++m) {
        const double2 va = P.vtx[ea[permk[m]]], vb = P.vtx[eb[perml[m]]];
        sTA[m][0] = va.x; sTA[m][1] = va.y;
        sTB[m][0] = vb.x; sTB[m][1] = vb.y;
      }
      const double ck = cross2(sTA[1][0] - sTA[0][0], sTA[2][1] - sTA[0][1], sTA[1][1] - sTA[0][1], sTA[2][0] - sTA[0][0]);
      const double cl = cross2(sTB[1][0] - sTB[0][0], sTB[2][1] - sTB[0][1], sTB[1][1] - sTB[0][1], sTB[2][0] - sTB[0][0]);
      double sc = fabs(ck) * fabs(cl);
      if (k != l) sc *= 2.0;
      sScale = sc * lab_scale(P, __ldg(&P.elem[k]).w, __ldg(&P.elem[l]).w);
    }
    __syncthreads();
    double acc[A::N];
#pragma unroll
    for (int i = 0; i < A::N; ++i) acc[i] = 0.0;
    const double t0x = sTA[0][0], t0y = sTA[0][1], u0x = sTB[0][0], u0y = sTB[0][1];
    const double e1kx = sTA[1][0] - t0x, e1ky = sTA[1][1] - t0y, e2kx = sTA[2][0] - t0x, e2ky = sTA[2][1] - t0y;
    const double e1lx = sTB[1][0] - u0x, e1ly = sTB[1][1] - u0y, e2lx = sTB[2][0] - u0x, e2ly = sTB[2][1] - u0y;
    int mk[U], ml[U];
#pragma unroll
    for (int m = 0; m < U; ++m) { mk[m] = sMk[m]; ml[m] = sMl[m]; }
    // identical pair, symmetric kernel: each sub-rule's mirrored half (x <-> y,
    // quadrature.py:197-207) repeats its first half exactly (d -> -d, tm -> -tm),
    // so only the first halves are evaluated and the weights doubled
    constexpr bool HALF = FAM == 0 && T::SYM;
    const int m4 = R.n / 6;  // points per half sector (identical family: 6 blocks)
    const int npts_eval = HALF ? R.n / 2 : R.n;
    // (HALF: point ii0 of the evaluated halves is i = (ii0 / m4) 2 m4 + ii0 % m4,
    // the quotient and remainder tracked incrementally instead of divided)
    int hq = HALF ? (int)threadIdx.x / m4 : 0, hr = HALF ? (int)threadIdx.x % m4 : 0;
    for (int ii0 = threadIdx.x; ii0 < npts_eval; ii0 += blockDim.x) {
      const int i = HALF ? hq * 2 * m4 + hr : ii0;
      if (HALF) {
        hr += blockDim.x;
        while (hr >= m4) { hr -= m4; ++hq; }
      }
      const double xs0 = __ldg(&R.xs[2 * i]), xs1 = __ldg(&R.xs[2 * i + 1]);
      const double ys0 = __ldg(&R.ys[2 * i]), ys1 = __ldg(&R.ys[2 * i + 1]);
      const double x0 = __dadd_rn(__dadd_rn(t0x, mul(e1kx, xs0)), mul(e2kx, xs1));
      const double x1 = __dadd_rn(__dadd_rn(t0y, mul(e1ky, xs0)), mul(e2ky, xs1));
      const double y0 = __dadd_rn(__dadd_rn(u0x, mul(e1lx, ys0)), mul(e2lx, ys1));
      const double y1 = __dadd_rn(__dadd_rn(u0y, mul(e1ly, ys0)), mul(e2ly, ys1));
      const double d0 = x0 - y0, d1 = x1 - y1;
      const double r2 = sumsq(d0, d1);
      if (r2 <= 0.0) continue;
      double pv[NC * NC], qv[NC * NC];
      kval<KID>(P, x0, y0, d0, d1, r2, pv, qv);
      npts += HALF ? 2 : 1;
      // hat values at the rule points, (1 - p0) - p1, p0, p1 as quadrature._hats
      // (quadrature.py:129-135) computes them: no table reads
      const double hxa[3] = {__dsub_rn(__dsub_rn(1.0, xs0), xs1), xs0, xs1};
      const double hya[3] = {__dsub_rn(__dsub_rn(1.0, ys0), ys1), ys0, ys1};
      double phx[U], phy[U], tm[U];
#pragma unroll
      for (int m = 0; m < U; ++m) {
        phx[m] = mk[m] >= 0 ? (mk[m] == 0 ? hxa[0] : (mk[m] == 1 ? hxa[1] : hxa[2])) : 0.0;
        phy[m] = ml[m] >= 0 ? (ml[m] == 0 ? hya[0] : (ml[m] == 1 ? hya[1] : hya[2])) : 0.0;
        tm[m] = phx[m] - phy[m];
      }
      const double wi = HALF ? 2.0 * __ldg(&R.w[i]) : __ldg(&R.w[i]);
      if (T::SYM) {
        // Bu[(m,c),(m',d)] += w tm_m tm_m' P_cd  as  g[m][cd] = w P_cd tm_m, then g tm_m'
        double g[U][NC * NC];
#pragma unroll
        for (int m = 0; m < U; ++m)
#pragma unroll
          for (int cd = 0; cd < NC * NC; ++cd) g[m][cd] = (wi * pv[cd]) * tm[m];
#pragma unroll
        for (int m = 0; m < U; ++m)
#pragma unroll
          for (int mp = m; mp < U; ++mp)
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
              for (int d = 0; d < NC; ++d) {
                const int ii = m * NC + c, jj = mp * NC + d;
                if (m == mp && jj < ii) continue;
                acc[A::idx(ii, jj)] = fma(g[m][c * NC + d], tm[mp], acc[A::idx(ii, jj)]);
              }
      } else {
#pragma unroll
        for (int m = 0; m < U; ++m)
#pragma unroll
          for (int mp = 0; mp < U; ++mp)
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
              for (int d = 0; d < NC; ++d) {
                const int ii = m * NC + c, jj = mp * NC + d;
                acc[A::idx(ii, jj)] += (wi * tm[m]) * (pv[c * NC + d] * phx[mp] - qv[c * NC + d] * phy[mp]);
              }
      }
    }
    // deterministic block reduction
#pragma unroll
    for (int i = 0; i < A::N; ++i) {
      double v = acc[i];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane_id() == 0) red[threadIdx.x >> 5][i] = v;
    }
    __syncthreads();
    double pm = 0.0;
    for (int s = threadIdx.x; s < SLOTS; s += blockDim.x) {
      const long long slot = cbase + pi * SLOTS + s;
      const int ii = s / (6 * NC), jj = s % (6 * NC);
      if (ii >= UN || jj >= UN) {
        put_key(P, keys, slot, kSentinel);
        vals[slot] = 0.0;
        continue;
      }
      const int ai = A::idx(ii, jj);
      double v = red[0][ai];
#pragma unroll
      for (int w = 1; w < kSingThreads / 32; ++w) v += red[w][ai];
      v *= sScale;
      report_nonfinite(nonfinite(v), k, l, P.K, errpair);
      vm = fmax(vm, fabs(v));
      pm = fmax(pm, fabs(v));
      const int m = ii / NC, c = ii % NC, mp = jj / NC, d = jj % NC;
      put_key(P, keys, slot, coo_key(P, (long long)NC * sUb[m] + c, (long long)NC * sUb[mp] + d));
      vals[slot] = emit_val(v);
    }
    for (int o = 16; o; o >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, o));
    if (lane_id() == 0) sPm[threadIdx.x >> 5] = pm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < kSingThreads / 32; ++w) m = fmax(m, sPm[w]);
      elem_bound(emax, k, m);  // every row of the pair's block is a row of k or of l
      if (l != k) elem_bound(emax, l, m);
    }
    __syncthreads();
  }
  warp_add_ll(npts, &counters[K_SPTS3 + (U - 3)]);
  warp_max_abs(vm, vmax);
}

// ---------------------------------------------------------------- merge

// 64-bit COO keys -> 32-bit when (rows x J) fits (fewer bytes per radix pass)
__global__ void k_narrow_keys(const unsigned long long* __restrict__ in, long long n, unsigned* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = in[i];
  out[i] = k == kSentinel ? 0xffffffffu : (unsigned)k;
}

template <typename KT>
__global__ void k_seg_heads(const KT* __restrict__ key, long long n, int* head) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const KT k = key[i];
  head[i] = k != key_sentinel<KT>() && (i == 0 || key[i - 1] != k);
}

template <typename KT>
__global__ void k_seg_starts(const KT* __restrict__ key, long long n, const int* __restrict__ head,
                             const long long* __restrict__ sid, long long* start) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (head[i]) start[sid[i]] = i;
  const bool valid = key[i] != key_sentinel<KT>();
  if (valid && (i + 1 == n || key[i + 1] == key_sentinel<KT>())) start[sid[i] + head[i]] = i + 1;
}

// one thread per (row, col): left-to-right sum in COO position order
template <typename KT>
__global__ void k_seg_sum(const KT* __restrict__ key, const double* __restrict__ val,
                          const long long* __restrict__ start, long long nseg, long long J, int* present,
                          int* segrow, int* col, double* sum) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const long long a = start[s], b = start[s + 1];
  double acc = 0.0;
  bool pres = false;
  for (long long i = a; i < b; ++i) {
    const double v = val[i];
    acc += v;
    pres |= __double_as_longlong(v) != 0;
  }
  const unsigned long long kk = (unsigned long long)key[a];
  present[s] = pres;
  col[s] = (int)(kk % (unsigned long long)J);
  segrow[s] = (int)(kk / (unsigned long long)J);
  sum[s] = acc;
}

// CSR row pointers from the row-sorted segments: indptr[r] = output position
// of the first segment whose row is >= r (no per-row atomics)
__global__ void k_seg_indptr(const int* __restrict__ segrow, const long long* __restrict__ pos,
                             const int* __restrict__ present, long long nseg, long long nrows, long long* indptr) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int r = segrow[s];
  const int rp = s ? segrow[s - 1] : -1;
  for (int rr = rp + 1; rr <= r; ++rr) indptr[rr] = pos[s];
  if (s == nseg - 1) {
    const long long end = pos[s] + present[s];
    for (long long rr = r + 1; rr <= nrows; ++rr) indptr[rr] = end;
  }
}

__global__ void k_seg_scatter(const int* __restrict__ present, const long long* __restrict__ pos,
                              const int* __restrict__ col, const double* __restrict__ sum,
                              long long nseg, int* indices, double* data) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= nseg || !present[s]) return;
  indices[pos[s]] = col[s];
  data[pos[s]] = sum[s];
}

__global__ void k_add_offset(long long* p, long long n, long long off) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] += off;
}

// ---------------------------------------------------------------- load vector
__global__ void k_load_points(Params P, const int* __restrict__ act, int nact, double* pts) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)nact * 7) return;
  const int m = (int)(t / 7), p = (int)(t % 7);
  double tx[3], ty[3];
  load_tri(P, act[m], tx, ty);
  const double e1x = tx[1] - tx[0], e1y = ty[1] - ty[0], e2x = tx[2] - tx[0], e2y = ty[2] - ty[0];
  // coords[:, 0] + e1 * op0 + e2 * op1 (assembly.py:468-469)
  pts[2 * t] = __dadd_rn(__dadd_rn(tx[0], mul(e1x, c_rule.op[p][0])), mul(e2x, c_rule.op[p][1]));
  pts[2 * t + 1] = __dadd_rn(__dadd_rn(ty[0], mul(e1y, c_rule.op[p][0])), mul(e2y, c_rule.op[p][1]));
}

// per active element: contrib[a][c] = 2A sum_p ow_p oh_pa f(x_p)_c
__global__ void k_load_contrib(Params P, const int* __restrict__ act, int nact,
                               const double* __restrict__ fx, int fconst, double* contrib) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nact) return;
  double tx[3], ty[3];
  load_tri(P, act[m], tx, ty);
  const double twoA = twice_area(tx, ty);
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < P.nc; ++c) {
      double s = 0.0;
      for (int p = 0; p < 7; ++p) {
        const double f = fconst ? fx[c] : fx[((long long)m * 7 + p) * P.nc + c];
        s += (c_rule.ow[p] * c_rule.oh[p][a]) * f;
      }
      contrib[((long long)m * 3 + a) * P.nc + c] = s * twoA;
    }
}

// b[nc*dof + c]: sum over the (element, local hat) incidences of the dof in
// element order (the np.add.at scatter order, assembly.py:477-480)
__global__ void k_load_gather(const int* __restrict__ inc_start, const int* __restrict__ inc_item,
                              const double* __restrict__ contrib, int nbase, int nc, double* b) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nbase) return;
  for (int c = 0; c < nc; ++c) {
    double s = 0.0;
    for (int j = inc_start[v]; j < inc_start[v + 1]; ++j) s += contrib[(long long)inc_item[j] * nc + c];
    b[(long long)nc * v + c] = s;
  }
}

__global__ void k_load_inc(Params P, const int* __restrict__ act, int nact, unsigned* key, int* item) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)nact * 3) return;
  const int m = (int)(t / 3), a = (int)(t % 3);
  const int4 d = P.dofs[act[m]];
  key[t] = (unsigned)(a == 0 ? d.x : a == 1 ? d.y : d.z);
  item[t] = (int)t;  // m * 3 + a, element-major
}

// ---------------------------------------------------------------- mass matrix
// assemble_mass (assembly.py:484-506): per active element the exact P1
// block area * (1 + delta_ab) / 12 on every component, as COO for merge_csr.
// area = signed_areas (mesh.py:36-42) in the reference's operation order.
__global__ void k_mass(Params P, const int* __restrict__ act, int nact, unsigned long long* keys, double* vals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nact) return;
  const int k = act[t];
  const int4 e = P.elem[k], d = P.dofs[k];
  const double2 p0 = P.vtx[e.x], p1 = P.vtx[e.y], p2 = P.vtx[e.z];
  const double area =
      mul(0.5, __dsub_rn(mul(p1.x - p0.x, p2.y - p0.y), mul(p1.y - p0.y, p2.x - p0.x)));
  const int da[3] = {d.x, d.y, d.z};
  const int NC = P.nc;
  const long long base = (long long)t * 9 * NC;
  for (int c = 0; c < NC; ++c)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        const long long row = (long long)NC * da[a] + c, col = (long long)NC * da[b] + c;
        const long long slot = base + c * 9 + a * 3 + b;
        keys[slot] = (unsigned long long)row * (unsigned long long)P.J + (unsigned long long)col;
        vals[slot] = mul(area, (a == b ? 2.0 : 1.0) / 12.0);
      }
}

__global__ void k_active(Params P, int* flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < P.K) flag[k] = (P.elem[k].w & 15) != 0;
}

// ---------------------------------------------------------------- fp64 peak
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_iota(int* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

inline unsigned grid_for(long long n, int bs) {
  long long g = (n + bs - 1) / bs;
  return (unsigned)std::max(1LL, std::min(g, 2147483647LL));
}

}  // namespace

// ===================================================================== plan
struct nlg_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // host outputs: batch CSR pieces copied to pinned staging while later batches run
  Params P{};
  // owned device arrays
  double2* vtx = nullptr;
  int4* elem = nullptr;
  int4* dofs = nullptr;
  double2* ctr = nullptr;
  double* rad = nullptr;
  double4* ftab = nullptr;  // analytic full-pair factors (k_elem_factors)
  unsigned long long* fmax = nullptr;  // [4] bounds of the analytic terms (max |A2|, |A2 psi|, |Phi|, |f|)
  int* de_start = nullptr;  // dof base -> its (element, local vertex) pairs: [J / nc + 1]
  int* de_items = nullptr;  // element * 4 + local vertex, by dof base
  double* sing_tab[3][5] = {};
  int sing_n[3] = {0, 0, 0};
  bool prepped = false;
  Grid G{};
  int* grid_start = nullptr;
  int* grid_items = nullptr;
  int4* grid_el = nullptr;
  double2* grid_ctr = nullptr;
  double* grid_rad = nullptr;
  double4* grid_ft = nullptr;
  int4* grid_dof = nullptr;
  double* grid_csum = nullptr;
  int* col_start = nullptr;   // analytic: column grid
  int* col_id = nullptr;
  double4* col_pos = nullptr;
  // load vector support
  int* act = nullptr;
  int nact = -1;
  int nbase = 0;
  int row_cap = 0;  // stage-W table size the last batches needed (start there)
  bool use_rows = true;  // merge stage W (NLG_MERGE=sort: stage R + global sort)
  size_t arena_used = 0;  // virtual bump offset into the device arena during a call
  std::vector<long long> last_batches;  // row ranges (lo, hi) of the last nlg_assemble's batches
};

namespace {

// Process-wide per-device scratch arena, reused by every plan and call on the
// device (grown once to the cumulative peak a call needed), so steady-state
// assemblies never reach the allocator; plus a pinned host staging buffer for
// host-resident outputs.  A per-device mutex serialises calls that share them.
struct DeviceScratch {
  std::mutex mu;
  char* arena = nullptr;
  size_t cap = 0, peak = 0;
  char* pinned = nullptr;
  size_t pinned_cap = 0;
  long long pin_nnz = 0;  // staging layout: data[pin_nnz] | indices[pin_nnz] | indptr (grows with the outputs seen)
  unsigned long long pin_sig = 0;  // problem / row range the hint was measured on (caller-provided arenas)
  // small device -> host readbacks (counts, totals) go through mapped pinned
  // memory written by a kernel, not through the copy engine: a 4-byte
  // cudaMemcpy would queue behind the bulk D2H of the previous batch's CSR
  // (same engine) and stall the host for the whole copy
  char* rb_host = nullptr;
  char* rb_dev = nullptr;
  size_t rb_used = 0;
  struct RbPending { void* dst; size_t off, n; };
  std::vector<RbPending> rb_pending;
};
DeviceScratch g_scratch[64];
constexpr size_t kRbCap = 1 << 20;

thread_local nlg_plan* g_arena_plan = nullptr;  // plan whose device arena backs DevBuf

struct DevBuf {  // scratch: bump-allocated from the plan's arena, else stream-ordered
  void* p = nullptr;
  cudaStream_t s = nullptr;
  bool arena = false;
  cudaError_t alloc(size_t n, cudaStream_t st) {
    s = st;
    n = (std::max<size_t>(n, 16) + 255) & ~(size_t)255;
    if (nlg_plan* pl = g_arena_plan) {
      // arena_used is a virtual bump offset advanced for every scratch
      // allocation, so arena_peak is the true cumulative peak even when the
      // arena is absent or too small (the next call grows it once)
      DeviceScratch& ds = g_scratch[pl->device];
      const size_t off = pl->arena_used, peak0 = ds.peak;
      pl->arena_used += n;
      ds.peak = std::max(ds.peak, pl->arena_used);
      if (ds.arena && off + n <= ds.cap) {
        p = ds.arena + off;
        arena = true;
        return cudaSuccess;
      }
      const cudaError_t e = cudaMallocAsync(&p, n, st);
      if (e != cudaSuccess) {  // a buffer that did not fit is not part of the peak to grow to
        pl->arena_used = off;
        ds.peak = peak0;
        p = nullptr;
      }
      return e;
    }
    return cudaMallocAsync(&p, n, st);
  }
  // stream-ordered, never from the arena (buffers that outlive the batches:
  // the arena may be handed back before the outputs are allocated)
  cudaError_t alloc_pool(size_t n, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(&p, (std::max<size_t>(n, 16) + 255) & ~(size_t)255, st);
  }
  ~DevBuf() {
    if (p && !arena) cudaFreeAsync(p, s);
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// arena allocations made inside a scope are released when it ends (LIFO)
struct ArenaScope {
  nlg_plan* pl;
  size_t mark;
  explicit ArenaScope(nlg_plan* p) : pl(p), mark(p ? p->arena_used : 0) {}
  ~ArenaScope() {
    if (pl) pl->arena_used = mark;
  }
};

nlg_status prep(nlg_plan* pl) {
  if (pl->prepped) return NLG_OK;
  ArenaScope arena_scope(g_arena_plan);
  Params& P = pl->P;
  cudaStream_t st = pl->stream;
  const int K = P.K;
  DevBuf ext;
  CK(ext.alloc(5 * sizeof(unsigned long long), st));
  unsigned long long init[5] = {~0ull, ~0ull, 0ull, 0ull, 0ull};
  CK(cudaMemcpyAsync(ext.p, init, sizeof init, cudaMemcpyHostToDevice, st));
  k_bounds<<<grid_for(K, 256), 256, 0, st>>>(P, pl->ctr, pl->rad, ext.as<unsigned long long>());
  LAUNCHED();
  CK(cudaMemsetAsync(pl->fmax, 0, 4 * sizeof(unsigned long long), st));
  if (P.analytic && K) {
    if (P.kid == 2) k_elem_factors<2><<<grid_for(K, 256), 256, 0, st>>>(P, pl->ftab, pl->fmax);
    else k_elem_factors<3><<<grid_for(K, 256), 256, 0, st>>>(P, pl->ftab, pl->fmax);
    LAUNCHED();
  }
  {
    // dof base -> (element, local vertex) incidence, for the row merge
    const long long nb = P.J / P.nc, n3 = 3LL * K;
    DevBuf dk, dk2, dv;
    CK(dk.alloc(sizeof(unsigned) * std::max(n3, 1LL), st));
    CK(dk2.alloc(sizeof(unsigned) * std::max(n3, 1LL), st));
    CK(dv.alloc(sizeof(int) * std::max(n3, 1LL), st));
    if (pl->de_items) cudaFreeAsync(pl->de_items, st);
    if (pl->de_start) cudaFreeAsync(pl->de_start, st);
    CK(cudaMallocAsync(&pl->de_items, sizeof(int) * std::max(n3, 1LL), st));
    CK(cudaMallocAsync(&pl->de_start, sizeof(int) * (nb + 1), st));
    if (n3) {
      k_dof_keys<<<grid_for(n3, 256), 256, 0, st>>>(P, dk.as<unsigned>(), dv.as<int>());
      LAUNCHED();
      int bits = 1;
      while ((1ll << bits) <= nb) ++bits;
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk.as<unsigned>(), dk2.as<unsigned>(), dv.as<int>(),
                                         pl->de_items, (int)n3, 0, bits, st));
      DevBuf tmp;
      CK(tmp.alloc(tb, st));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk.as<unsigned>(), dk2.as<unsigned>(), dv.as<int>(),
                                         pl->de_items, (int)n3, 0, bits, st));
      g_launches += 1 + (bits + 7) / 8;
    }
    k_cell_ranges<<<grid_for(nb + 1, 256), 256, 0, st>>>(dk2.as<unsigned>(), (int)n3, (int)nb, pl->de_start);
    LAUNCHED();
  }
  unsigned long long h[5];
  CK(cudaMemcpyAsync(h, ext.p, sizeof h, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double ox = ord2d(h[0]), oy = ord2d(h[1]), mx = ord2d(h[2]), my = ord2d(h[3]), rmax = ord2d(h[4]);
  if (h[2] == 0ull) { ox = oy = mx = my = 0.0; rmax = 0.0; }  // no active element
  const double reach = (P.prer + 2.0 * rmax) * (1.0 + 1e-9) + 1e-300;
  // pitch: reach / 8 (the scanned cell rows hug the disk, and the cells wholly inside the analytic
  // kernels' surely-full radius cover most of it; reach / 2 scanned ~2.4x the disk's area);
  // NLG_GRID_DIV: A/B (the row merge holds <= kMaxRowsG cell rows)
  static const int grid_div = getenv("NLG_GRID_DIV") ? std::min(16, std::max(1, atoi(getenv("NLG_GRID_DIV")))) : 8;
  double cs = reach / grid_div;
  // keep the cell count bounded (tiny horizons on huge meshes)
  const double ext_x = mx - ox, ext_y = my - oy;
  while ((ext_x / cs + 1.0) * (ext_y / cs + 1.0) > 6.0e7) cs *= 2.0;
  Grid G;
  G.ox = ox; G.oy = oy; G.cs = cs;
  G.reach = reach;
  G.rmax = rmax;
  G.span = (int)ceil(reach / cs);
  G.nx = (int)floor(ext_x / cs) + 1;
  G.ny = (int)floor(ext_y / cs) + 1;
  const int ncell = G.nx * G.ny;
  DevBuf key, val, key2;
  CK(key.alloc(sizeof(unsigned) * K, st));
  CK(val.alloc(sizeof(int) * K, st));
  CK(key2.alloc(sizeof(unsigned) * K, st));
  if (pl->grid_items) cudaFreeAsync(pl->grid_items, st);
  if (pl->grid_start) cudaFreeAsync(pl->grid_start, st);
  CK(cudaMallocAsync(&pl->grid_items, sizeof(int) * std::max(K, 1), st));
  CK(cudaMallocAsync(&pl->grid_start, sizeof(int) * (ncell + 1), st));
  k_cell<<<grid_for(K, 256), 256, 0, st>>>(P, G, key.as<unsigned>(), val.as<int>());
  LAUNCHED();
  int bits = 1;
  while ((1ll << bits) <= ncell) ++bits;
  size_t tmpb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, key.as<unsigned>(), key2.as<unsigned>(), val.as<int>(),
                                     pl->grid_items, K, 0, bits, st));
  DevBuf tmp;
  CK(tmp.alloc(tmpb, st));
  CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmpb, key.as<unsigned>(), key2.as<unsigned>(), val.as<int>(),
                                     pl->grid_items, K, 0, bits, st));
  g_launches += 4;
  k_cell_ranges<<<grid_for(ncell + 1, 256), 256, 0, st>>>(key2.as<unsigned>(), K, ncell, pl->grid_start);
  LAUNCHED();
  G.start = pl->grid_start;
  G.items = pl->grid_items;
  if (pl->grid_el) cudaFreeAsync(pl->grid_el, st);
  if (pl->grid_ctr) cudaFreeAsync(pl->grid_ctr, st);
  if (pl->grid_rad) cudaFreeAsync(pl->grid_rad, st);
  CK(cudaMallocAsync(&pl->grid_el, sizeof(int4) * std::max(K, 1), st));
  CK(cudaMallocAsync(&pl->grid_ctr, sizeof(double2) * std::max(K, 1), st));
  CK(cudaMallocAsync(&pl->grid_rad, sizeof(double) * std::max(K, 1), st));
  if (K) {
    if (P.analytic && !pl->grid_ft) {
      CK(cudaMallocAsync(&pl->grid_ft, sizeof(double4) * K, st));
      CK(cudaMallocAsync(&pl->grid_dof, sizeof(int4) * K, st));
    }
    k_grid_gather<<<grid_for(K, 256), 256, 0, st>>>(P, pl->grid_items, K, pl->grid_el, pl->grid_ctr, pl->grid_rad,
                                                     P.analytic ? pl->grid_ft : nullptr, pl->grid_dof);
    LAUNCHED();
  }
  G.gel = pl->grid_el;
  G.gctr = pl->grid_ctr;
  G.grad = pl->grid_rad;
  G.gft = P.analytic ? pl->grid_ft : nullptr;
  G.gdof = P.analytic ? pl->grid_dof : nullptr;
  G.gcsum = nullptr;
  if (P.analytic && K) {
    if (pl->grid_csum) cudaFreeAsync(pl->grid_csum, st);
    CK(cudaMallocAsync(&pl->grid_csum, sizeof(double) * ncell, st));
    k_cell_sums<<<grid_for(ncell, 256), 256, 0, st>>>(pl->grid_start, ncell, pl->grid_ft, pl->grid_csum);
    LAUNCHED();
    G.gcsum = pl->grid_csum;
  }
  G.cstart = nullptr;
  G.cid = nullptr;
  G.cpos = nullptr;
  if (P.analytic) {
    const int nb = (int)(P.J / P.nc);
    DevBuf ck, ck2, cv, cp;
    CK(ck.alloc(sizeof(unsigned) * std::max(nb, 1), st));
    CK(ck2.alloc(sizeof(unsigned) * std::max(nb, 1), st));
    CK(cv.alloc(sizeof(int) * std::max(nb, 1), st));
    CK(cp.alloc(sizeof(double4) * std::max(nb, 1), st));
    if (!pl->col_start) {
      CK(cudaMallocAsync(&pl->col_start, sizeof(int) * (ncell + 1), st));
      CK(cudaMallocAsync(&pl->col_id, sizeof(int) * std::max(nb, 1), st));
      CK(cudaMallocAsync(&pl->col_pos, sizeof(double4) * std::max(nb, 1), st));
    }
    if (nb) {
      k_col_keys<<<grid_for(nb, 256), 256, 0, st>>>(P, G, pl->de_start, pl->de_items, nb, ck.as<unsigned>(),
                                                    cv.as<int>(), cp.as<double4>());
      LAUNCHED();
      size_t tb2 = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, ck.as<unsigned>(), ck2.as<unsigned>(), cv.as<int>(), pl->col_id,
                                         nb, 0, bits, st));
      DevBuf tmp2;
      CK(tmp2.alloc(tb2, st));
      CK(cub::DeviceRadixSort::SortPairs(tmp2.p, tb2, ck.as<unsigned>(), ck2.as<unsigned>(), cv.as<int>(), pl->col_id,
                                         nb, 0, bits, st));
      g_launches += 4;
      k_col_gather<<<grid_for(nb, 256), 256, 0, st>>>(pl->col_id, nb, cp.as<double4>(), pl->col_pos);
      LAUNCHED();
    }
    k_cell_ranges<<<grid_for(ncell + 1, 256), 256, 0, st>>>(ck2.as<unsigned>(), nb, ncell, pl->col_start);
    LAUNCHED();
    G.cstart = pl->col_start;
    G.cid = pl->col_id;
    G.cpos = pl->col_pos;
  }
  pl->G = G;
  pl->prepped = true;
  return NLG_OK;
}

__global__ void k_readback(unsigned* __restrict__ dst, const unsigned* __restrict__ src, int nwords) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// Queue a small device -> host read on stream s; the value lands in `dst`
// at the next rb_sync(s).  (Larger or unaligned reads use the copy engine.)
cudaError_t rb_read(void* dst, const void* src, size_t n, cudaStream_t s) {
  if (!g_arena_plan) return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s);
  DeviceScratch& ds = g_scratch[g_arena_plan->device];
  if (!ds.rb_host) {
    if (cudaHostAlloc((void**)&ds.rb_host, kRbCap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&ds.rb_dev, ds.rb_host, 0) != cudaSuccess) {
      cudaGetLastError();
      if (ds.rb_host) cudaFreeHost(ds.rb_host);
      ds.rb_host = ds.rb_dev = nullptr;
    }
  }
  if (!ds.rb_host || (n & 3) || ((uintptr_t)src & 3) || ds.rb_used + n > kRbCap)
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s);
  if (!n) return cudaSuccess;
  const int nw = (int)(n / 4);
  k_readback<<<std::min(64, (nw + 255) / 256), 256, 0, s>>>((unsigned*)(ds.rb_dev + ds.rb_used), (const unsigned*)src, nw);
  g_launches += 1;
  ds.rb_pending.push_back({dst, ds.rb_used, n});
  ds.rb_used += (n + 15) & ~(size_t)15;
  return cudaGetLastError();
}
cudaError_t rb_sync(cudaStream_t s) {
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess || !g_arena_plan) return e;
  DeviceScratch& ds = g_scratch[g_arena_plan->device];
  for (const auto& q : ds.rb_pending) memcpy(q.dst, ds.rb_host + q.off, q.n);
  ds.rb_pending.clear();
  ds.rb_used = 0;
  return cudaSuccess;
}

struct Csr {  // one batch's rows
  long long row_lo, row_hi, nnz;
  long long* indptr;
  int* indices;
  double* data;
  long long staged = -1;  // host outputs: entry offset of its copy in the pinned staging (-1: not staged)
};

struct Counters {
  unsigned long long c[K_NCOUNTERS];
};

// algorithmic FP64 flops of the reference for the counted work;
// part: 0 full-pair kernel, 1 clipped-pair kernel, 2 singular kernel
long long alg_flops(const Params& P, const unsigned long long* c, int part) {
  const long long nc = P.nc, nc2 = nc * nc;
  const bool ns = !P.sym;
  const long long kf = P.kid == 0 ? 2 : P.kid == 1 ? 9 : P.kid == 3 ? 4 : 0;
  const long long a0 = ns ? 9 * nc2 : 8 * nc2, a1 = ns ? 35 * nc2 : 34 * nc2, a2 = 35 * nc2;
  const long long f0 = 9 * nc * (3 + 4 * nc) + 9, f1 = 9 * nc * (1 + 4 * nc) + 9, f2 = 9 * nc * (4 + 8 * nc) + 9;
  long long fl = 0;
  if (part == 0) {
    // K_EVAL_FULL0 counts each 7x7 point pair once; the reference evaluates
    // it in mode 0 and again in mode 1
    fl += (long long)c[K_EVAL_FULL0] * ((26 + kf + a0) + (26 + kf + a1));
    fl += (long long)c[K_OUT_FULL0] / 2 * (f0 + f1);
    fl += (long long)c[K_EVAL_FULL2] * (26 + kf + a2) + (long long)c[K_OUT_FULL2] * f2;
  } else if (part == 1) {
    fl += (long long)c[K_EVAL_M0] * (26 + kf + a0) + (long long)c[K_OUT_M0] * f0;
    fl += (long long)c[K_EVAL_M1] * (26 + kf + a1) + (long long)c[K_OUT_M1] * f1;
    fl += (long long)c[K_EVAL_M2] * (26 + kf + a2) + (long long)c[K_OUT_M2] * f2;
  } else {
    for (int u = 3; u <= 6; ++u)
      fl += (long long)c[K_SPTS3 + u - 3] * (16 + 5 + kf + u + u * u * (2 + 2 * nc2));
  }
  return fl;
}

template <int KID>
nlg_status run_visits(nlg_plan* pl, const Params& P, const int2* lf, const int2* lp, VisitOut OF, VisitOut O,
                      cudaEvent_t ev_mid) {
  const long long nF = OF.nlist, nP = O.nlist;
  if (nF) {  // (analytic full pairs: none to integrate)
    // grid-stride: the pow tables are staged into shared memory once per block
    if constexpr (KID == 0) {
      const unsigned gf = (unsigned)std::min<long long>(grid_for(nF, 128), 148LL * 32);
      k_full<KID, 1><<<gf, 128, 0, pl->stream>>>(P, lf, OF);
      k_full<KID, 2><<<gf, 128, 0, pl->stream>>>(P, lf, OF);
      g_launches += 1;
    } else {
      k_full<KID><<<grid_for(nF, 128), 128, 0, pl->stream>>>(P, lf, OF);
    }
    LAUNCHED();
  }
  CK(cudaEventRecord(ev_mid, pl->stream));
  if (nP) {
    const long long chunks = (nP + 1) / 2;
    constexpr int NWB = clip_warps<KID>();
    const unsigned g = (unsigned)std::min<long long>((chunks + NWB - 1) / NWB, 148LL * 256 / NWB);
    // warp-local clipping for the closed-form kernels (NLG_CLIP_WL=0: block queue)
    const bool wl_env = !(getenv("NLG_CLIP_WL") && atoi(getenv("NLG_CLIP_WL")) == 0);  // (read per launch: tests switch it)
    const bool wl = (KID == 2 || KID == 3) && P.path == 0 && wl_env;
    if (P.ball == 2) {
      const int smem = NWB * (int)sizeof(ClipWarp<KID, true>) + (int)sizeof(ClipBlock<KID>);
      CK(cudaFuncSetAttribute(k_clipped<KID, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_clipped<KID, true><<<g, 32 * NWB, smem, pl->stream>>>(P, lp, O);
    } else if (wl) {
      if constexpr (KID == 2 || KID == 3) {
        // four records per warp round, warp-local clip queue.  Default:
        // k_clipped_cfr (ring queue), one 16-warp block per SM, classify loop
        // rolled, the four warps of a scheduler re-aligned every 2 rounds
        // (config 5, ms: 375, 367 instantiated per ball; without the barrier
        // 376-394, every 3 / 4 / 8 rounds 366 / 366 / 369, block barrier every
        // 4 rounds 380, 8-warp blocks 396, classify unrolled 393-412).
        // NLG_CLIP_WL picks the A/B variants: 3 k_clipped_cf (no ring, 439),
        // 5 ring 8 x 2 unrolled, 9 no barrier, 11 block barrier every 4 rounds,
        // 18 the ball read at run time, 23 approxcaps without the analytic instantiation.
        const int var = getenv("NLG_CLIP_WL") ? atoi(getenv("NLG_CLIP_WL")) : 14;
        const long long rounds = (nP + 3) / 4;
        if (var >= 5) {
          auto launch_r = [&](auto kern, int nwb) -> cudaError_t {
            const int smem = nwb * (int)sizeof(CfRing<KID>);
            // (blocks for 512 warps per SM: fewer, longer-lived blocks measured slower, 385 -> 397 at 16)
            static const int gmul = getenv("NLG_CF_GRID") ? atoi(getenv("NLG_CF_GRID")) : 512;
            const unsigned gcf = (unsigned)std::min<long long>((rounds + nwb - 1) / nwb, 148LL * gmul / nwb);
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            kern<<<gcf, 32 * nwb, smem, pl->stream>>>(P, lp, O);
            return cudaGetLastError();
          };
          switch (var) {
            case 5: CK(launch_r(k_clipped_cfr<KID, 8, 2, 2>, 8)); break;
            case 9: CK(launch_r(k_clipped_cfr<KID, 16, 1, 1>, 16)); break;
            case 11: CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, 4>, 16)); break;
            case 18: CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, -2>, 16)); break;
            case 23: CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, -2, 1>, 16)); break;
            default:
              if (P.ball == 0) CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, -2, 0>, 16));
              else if (P.analytic) CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, -2, 1, 1>, 16));
              else CK(launch_r(k_clipped_cfr<KID, 16, 1, 1, -2, 1>, 16));
              break;
          }
        } else {
          const int smem = 8 * (int)sizeof(CfWarp<KID>);
          const unsigned gcf = (unsigned)std::min<long long>((rounds + 7) / 8, 148LL * 64);
          CK(cudaFuncSetAttribute(k_clipped_cf<KID, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          k_clipped_cf<KID, 8, 2><<<gcf, 256, smem, pl->stream>>>(P, lp, O);
          CK(cudaGetLastError());
        }
      }
    } else {
      const int smem = NWB * (int)sizeof(ClipWarp<KID, false>) + (int)sizeof(ClipBlock<KID>);
      CK(cudaFuncSetAttribute(k_clipped<KID, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_clipped<KID, false><<<g, 32 * NWB, smem, pl->stream>>>(P, lp, O);
    }
    LAUNCHED();
  }
  return NLG_OK;
}

template <int KID>
nlg_status run_singular(nlg_plan* pl, const Params& P, int2* const* ls, const long long* nS,
                        unsigned long long* keys, double* vals, long long cbase,
                        unsigned long long* counters, unsigned long long* errpair, unsigned long long* vmax,
                        unsigned long long* emax) {
  constexpr int NC = KTraits<KID>::NC;
  const long long slots = 36LL * NC * NC;
  for (int f = 0; f < 3; ++f) {
    if (!nS[f]) continue;
    SingRule R{pl->sing_tab[f][0], pl->sing_tab[f][1], pl->sing_tab[f][2], pl->sing_tab[f][3],
               pl->sing_tab[f][4], pl->sing_n[f]};
    const unsigned g = (unsigned)std::min<long long>(nS[f], 1 << 20);
    if (f == 0)
      k_singular<KID, 0, 3><<<g, kSingThreads, 0, pl->stream>>>(P, ls[0], nS[0], R, keys, vals, cbase, counters, errpair, vmax, emax);
    else if (P.is_dg)
      (f == 1 ? k_singular<KID, 1, 6> : k_singular<KID, 2, 6>)<<<g, kSingThreads, 0, pl->stream>>>(
          P, ls[f], nS[f], R, keys, vals, cbase, counters, errpair, vmax, emax);
    else if (f == 1)
      k_singular<KID, 1, 4><<<g, kSingThreads, 0, pl->stream>>>(P, ls[1], nS[1], R, keys, vals, cbase, counters, errpair, vmax, emax);
    else
      k_singular<KID, 2, 5><<<g, kSingThreads, 0, pl->stream>>>(P, ls[2], nS[2], R, keys, vals, cbase, counters, errpair, vmax, emax);
    LAUNCHED();
    cbase += nS[f] * slots;
  }
  return NLG_OK;
}

// Stable radix sort of the COO (row, col) keys, then one thread per run
// sums its values in COO position order -> CSR rows of this batch.
template <typename KT>
nlg_status merge_csr(cudaStream_t s, const Params& P, unsigned long long* keys64, double* vals, long long coo,
                     long long nrows, Csr& piece, long long& nnz, long long* coo_kept, bool keys_narrow = false) {
  int bits = 1;
  {
    const unsigned long long maxkey = (unsigned long long)nrows * (unsigned long long)P.J;
    while (bits < 64 && (1ull << bits) <= maxkey) ++bits;
  }
  DevBuf k1, k2, v2;
  KT* keys;
  if (sizeof(KT) == 4 && keys_narrow) {
    keys = reinterpret_cast<KT*>(keys64);  // written as 32-bit keys (put_key)
  } else if (sizeof(KT) == 4) {
    CK(k1.alloc(sizeof(KT) * std::max(coo, 1LL), s));
    if (coo) {
      k_narrow_keys<<<grid_for(coo, 256), 256, 0, s>>>(keys64, coo, k1.as<unsigned>());
      LAUNCHED();
    }
    keys = k1.as<KT>();
  } else {
    keys = (KT*)keys64;
  }
  CK(k2.alloc(sizeof(KT) * std::max(coo, 1LL), s));
  CK(v2.alloc(sizeof(double) * std::max(coo, 1LL), s));
  cub::DoubleBuffer<KT> dk(keys, k2.as<KT>());
  cub::DoubleBuffer<double> dv(vals, v2.as<double>());
  {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)coo, 0, bits, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)coo, 0, bits, s));
    g_launches += (bits + 7) / 8 + 1;
  }
  if (coo_kept) *coo_kept = coo;
  // the sentinel's low `bits` bits are all ones, above every valid key
  const KT* sk = dk.Current();
  const double* sv = dv.Current();
  DevBuf head, sid, start, present, segrow, col, sum, pos;
  CK(head.alloc(sizeof(int) * std::max(coo, 1LL), s));
  CK(sid.alloc(sizeof(long long) * (coo + 1), s));
  if (coo) {
    k_seg_heads<KT><<<grid_for(coo, 256), 256, 0, s>>>(sk, coo, head.as<int>());
    LAUNCHED();
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, tb, head.as<int>(), sid.as<long long>(), cub::Sum(), 0LL, (int)coo, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, head.as<int>(), sid.as<long long>(), cub::Sum(), 0LL, (int)coo, s));
    g_launches += 1;
  }
  long long nseg = 0;
  if (coo) {
    long long lsid;
    int lhead;
    CK(rb_read(&lsid, sid.as<long long>() + coo - 1, sizeof lsid, s));
    CK(rb_read(&lhead, head.as<int>() + coo - 1, sizeof lhead, s));
    CK(rb_sync(s));
    TRACE("sync 1775");
    nseg = lsid + lhead;
  }
  CK(start.alloc(sizeof(long long) * (nseg + 1), s));
  CK(present.alloc(sizeof(int) * std::max(nseg, 1LL), s));
  CK(col.alloc(sizeof(int) * std::max(nseg, 1LL), s));
  CK(sum.alloc(sizeof(double) * std::max(nseg, 1LL), s));
  CK(pos.alloc(sizeof(long long) * (nseg + 1), s));
  CK(segrow.alloc(sizeof(int) * std::max(nseg, 1LL), s));
  CK(cudaMallocAsync(&piece.indptr, sizeof(long long) * (nrows + 1), s));
  nnz = 0;
  if (nseg) {
    k_seg_starts<KT><<<grid_for(coo, 256), 256, 0, s>>>(sk, coo, head.as<int>(), sid.as<long long>(),
                                                        start.as<long long>());
    LAUNCHED();
    k_seg_sum<KT><<<grid_for(nseg, 256), 256, 0, s>>>(sk, sv, start.as<long long>(), nseg, P.J, present.as<int>(),
                                                      segrow.as<int>(), col.as<int>(), sum.as<double>());
    LAUNCHED();
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, tb, present.as<int>(), pos.as<long long>(), cub::Sum(), 0LL, (int)nseg, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, present.as<int>(), pos.as<long long>(), cub::Sum(), 0LL, (int)nseg, s));
    long long lpos;
    int lpres;
    CK(rb_read(&lpos, pos.as<long long>() + nseg - 1, sizeof lpos, s));
    CK(rb_read(&lpres, present.as<int>() + nseg - 1, sizeof lpres, s));
    CK(rb_sync(s));
    TRACE("sync 1803");
    nnz = lpos + lpres;
    CK(cudaMallocAsync(&piece.indices, sizeof(int) * std::max(nnz, 1LL), s));
    CK(cudaMallocAsync(&piece.data, sizeof(double) * std::max(nnz, 1LL), s));
    k_seg_scatter<<<grid_for(nseg, 256), 256, 0, s>>>(present.as<int>(), pos.as<long long>(), col.as<int>(),
                                                      sum.as<double>(), nseg, piece.indices, piece.data);
    LAUNCHED();
    k_seg_indptr<<<grid_for(nseg, 256), 256, 0, s>>>(segrow.as<int>(), pos.as<long long>(), present.as<int>(), nseg,
                                                     nrows, piece.indptr);
    LAUNCHED();
    g_launches += 1;
  } else {
    CK(cudaMallocAsync(&piece.indices, sizeof(int), s));
    CK(cudaMallocAsync(&piece.data, sizeof(double), s));
    CK(cudaMemsetAsync(piece.indptr, 0, sizeof(long long) * (nrows + 1), s));
  }
  piece.nnz = nnz;
  return NLG_OK;
}

// ---- merge stage W (k_row_asm) for one batch
template <int NC, int CAP, bool AN, bool SPL = false>
cudaError_t launch_rows(const Params& P, const RootIn& I, const RowIn& W, const RowOut& O, long long nblk,
                        cudaStream_t s) {
  constexpr int TH = CAP >= 4096 ? 1024 : (CAP >= 2048 || NC == 2 ? 512 : 128);
  const int smem = (int)sizeof(RowSmem<NC, CAP, TH>);
  cudaError_t e =
      cudaFuncSetAttribute(k_row_asm<NC, CAP, TH, AN, SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (nblk) k_row_asm<NC, CAP, TH, AN, SPL><<<(unsigned)nblk, TH, smem, s>>>(P, I, W, O);
  g_launches += 1;
  return cudaGetLastError();
}

// the column-half passes of rows wider than the largest table
cudaError_t launch_rows_split(const Params& P, const RootIn& I, const RowIn& W, const RowOut& O, long long nblk,
                              cudaStream_t s) {
  if (P.nc == 2) return launch_rows<2, 2048, false, true>(P, I, W, O, nblk, s);
  if (P.analytic) return launch_rows<1, 8192, true, true>(P, I, W, O, nblk, s);
  return launch_rows<1, 8192, false, true>(P, I, W, O, nblk, s);
}

cudaError_t launch_rows_cap(const Params& P, const RootIn& I, const RowIn& W, const RowOut& O, long long nblk,
                            int cap, cudaStream_t s) {
  if (P.nc == 2) {
    switch (cap) {
      case 512: return launch_rows<2, 512, false>(P, I, W, O, nblk, s);
      case 1024: return launch_rows<2, 1024, false>(P, I, W, O, nblk, s);
      default: return launch_rows<2, 2048, false>(P, I, W, O, nblk, s);
    }
  }
  if (P.analytic) {
    switch (cap) {
      case 1024: return launch_rows<1, 1024, true>(P, I, W, O, nblk, s);
      case 2048: return launch_rows<1, 2048, true>(P, I, W, O, nblk, s);
      case 4096: return launch_rows<1, 4096, true>(P, I, W, O, nblk, s);
      default: return launch_rows<1, 8192, true>(P, I, W, O, nblk, s);
    }
  }
  switch (cap) {
    case 1024: return launch_rows<1, 1024, false>(P, I, W, O, nblk, s);
    case 2048: return launch_rows<1, 2048, false>(P, I, W, O, nblk, s);
    case 4096: return launch_rows<1, 4096, false>(P, I, W, O, nblk, s);
    default: return launch_rows<1, 8192, false>(P, I, W, O, nblk, s);
  }
}

// Rows [row_lo, row_hi) of the batch through stage W into `piece`.  *fallback:
// some row outgrew the largest table (use stage R + sort); *need_split: the
// entry estimate was too small.
nlg_status merge_rows(nlg_plan* pl, const Params& P, const RootIn& RI, void* skeys, double* svals, long long nsing,
                      const unsigned long long* d_vmax, const unsigned long long* d_emax, long long ent_cap,
                      double cols_est, Csr& piece, long long& nnz,
                      bool* fallback, bool* need_split, long long* retries) {
  cudaStream_t s = pl->stream;
  const int NC = P.nc;
  const long long nrows = P.row_hi - P.row_lo;
  *fallback = *need_split = false;
  // singular entries sorted by (row, col); each row's first position
  DevBuf k2, v2, sstart;
  CK(sstart.alloc(sizeof(long long) * (nrows + 1), s));
  const void* sk = skeys;
  const double* sv = svals;
  int bits = 1;
  {
    const unsigned long long maxkey = (unsigned long long)nrows * (unsigned long long)P.J;
    while (bits < 64 && (1ull << bits) <= maxkey) ++bits;
  }
  if (nsing) {
    CK(k2.alloc((P.narrow ? 4 : 8) * nsing, s));
    CK(v2.alloc(sizeof(double) * nsing, s));
    size_t tb = 0;
    if (P.narrow) {
      cub::DoubleBuffer<unsigned> dk((unsigned*)skeys, k2.as<unsigned>());
      cub::DoubleBuffer<double> dv(svals, v2.as<double>());
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)nsing, 0, bits, s));
      DevBuf tmp;
      CK(tmp.alloc(tb, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)nsing, 0, bits, s));
      sk = dk.Current();
      sv = dv.Current();
    } else {
      cub::DoubleBuffer<unsigned long long> dk((unsigned long long*)skeys, k2.as<unsigned long long>());
      cub::DoubleBuffer<double> dv(svals, v2.as<double>());
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)nsing, 0, bits, s));
      DevBuf tmp;
      CK(tmp.alloc(tb, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)nsing, 0, bits, s));
      sk = dk.Current();
      sv = dv.Current();
    }
    g_launches += (bits + 7) / 8 + 1;
  }
  if (P.narrow)
    k_row_starts<unsigned><<<grid_for(nrows + 1, 256), 256, 0, s>>>((const unsigned*)sk, nsing, nrows, P.J,
                                                                    sstart.as<long long>());
  else
    k_row_starts<unsigned long long><<<grid_for(nrows + 1, 256), 256, 0, s>>>((const unsigned long long*)sk, nsing,
                                                                              nrows, P.J, sstart.as<long long>());
  LAUNCHED();
  const long long d_lo = P.row_lo / NC, d_hi = (P.row_hi - 1) / NC + 1, nd = std::max(0LL, d_hi - d_lo);
  DevBuf col, val, roff, rcnt, roff2, rcnt2, ovf0, ovf1, st;
  CK(col.alloc(sizeof(int) * std::max(ent_cap, 1LL), s));
  CK(val.alloc(sizeof(double) * std::max(ent_cap, 1LL), s));
  CK(roff.alloc(sizeof(long long) * std::max(nrows, 1LL), s));
  CK(rcnt.alloc(sizeof(int) * (nrows + 1), s));
  CK(roff2.alloc(sizeof(long long) * std::max(nrows, 1LL), s));
  CK(rcnt2.alloc(sizeof(int) * (nrows + 1), s));
  CK(cudaMemsetAsync(rcnt2.p, 0, sizeof(int) * (nrows + 1), s));
  CK(ovf0.alloc(sizeof(int) * std::max(nd, 1LL), s));
  CK(ovf1.alloc(sizeof(int) * std::max(nd, 1LL), s));
  CK(st.alloc(4 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(rcnt.p, 0, sizeof(int) * (nrows + 1), s));
  CK(cudaMemsetAsync(st.p, 0, 4 * sizeof(unsigned long long), s));
  RowIn W;
  W.de_start = pl->de_start;
  W.de_items = pl->de_items;
  W.inR = RI.inR;
  W.dlist = nullptr;
  W.d_lo = d_lo;
  W.key_bits = 1;
  while ((1LL << W.key_bits) - 1 < (long long)P.J / NC) ++W.key_bits;
  W.fill_div = getenv("NLG_ROW_FILL_DIV") ? atoi(getenv("NLG_ROW_FILL_DIV")) : 0;
  W.skey64 = P.narrow ? nullptr : (const unsigned long long*)sk;
  W.skey32 = P.narrow ? (const unsigned*)sk : nullptr;
  W.sval = sv;
  W.sstart = sstart.as<long long>();
  W.vmax = d_vmax;
  W.emax = d_emax;
  W.fmax = pl->fmax;
  W.G = pl->G;
  RowOut O;
  O.col = col.as<int>();
  O.val = val.as<double>();
  O.cap = ent_cap;
  O.used = st.as<unsigned long long>();
  O.novf = (unsigned*)(st.as<unsigned long long>() + 1);
  O.roff = roff.as<long long>();
  O.rcnt = rcnt.as<int>();
  O.roff2 = roff2.as<long long>();
  O.rcnt2 = rcnt2.as<int>();
  O.split = 0;
  const int cap_max = NC == 1 ? 8192 : 2048;
  // first table: the plan's last need, or the column estimate at <= 3/4 load
  int cap = NC == 1 ? 1024 : 512;
  while (cap < cap_max && (cap < pl->row_cap || 0.75 * cap < cols_est)) cap *= 2;
  long long nblk = nd;
  int* lists[2] = {ovf0.as<int>(), ovf1.as<int>()};
  unsigned long long used = 0;
  for (int pass = 0;; ++pass) {
    O.ovf = lists[pass & 1];
    CK(launch_rows_cap(P, RI, W, O, nblk, cap, s));
    unsigned long long hst[2] = {0, 0};  // entries used, overflowed dofs
    CK(rb_read(hst, st.p, sizeof hst, s));
    CK(rb_sync(s));
    TRACE("row pass");
    const unsigned hov = (unsigned)hst[1];
    used = hst[0];
    if (!hov) break;
    *retries += hov;
    if (4LL * hov > nblk) pl->row_cap = std::min(cap * 2, cap_max);  // most rows need more: start there next time
    if (cap >= cap_max) {
      // rows too wide for the largest table: their columns below / from the
      // row's own dof base in two passes (two sorted runs per row); a half
      // that still overflows sends the batch to stage R + sort
      W.dlist = lists[pass & 1];
      for (int half = 1; half <= 2; ++half) {
        O.split = half;
        O.ovf = lists[(pass + 1) & 1];
        CK(cudaMemsetAsync(O.novf, 0, sizeof(unsigned), s));
        CK(launch_rows_split(P, RI, W, O, hov, s));
        unsigned long long h2[2] = {0, 0};
        CK(rb_read(h2, st.p, sizeof h2, s));
        CK(rb_sync(s));
        used = h2[0];
        if (h2[1]) { *fallback = true; return NLG_OK; }
      }
      break;
    }
    cap *= 2;
    W.dlist = lists[pass & 1];
    nblk = hov;
    CK(cudaMemsetAsync(O.novf, 0, sizeof(unsigned), s));
  }
  if ((long long)used > ent_cap) { *need_split = true; return NLG_OK; }
  CK(cudaMallocAsync(&piece.indptr, sizeof(long long) * (nrows + 1), s));
  if (O.split) {  // split rows: both runs count
    k_add_int<<<grid_for(nrows + 1, 256), 256, 0, s>>>(rcnt.as<int>(), rcnt2.as<int>(), nrows + 1);
    LAUNCHED();
  }
  {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, tb, rcnt.as<int>(), piece.indptr, cub::Sum(), 0LL, (int)(nrows + 1), s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, rcnt.as<int>(), piece.indptr, cub::Sum(), 0LL, (int)(nrows + 1), s));
    g_launches += 1;
  }
  if (O.split) {  // the gather needs the first run's own length back
    k_sub_int<<<grid_for(nrows + 1, 256), 256, 0, s>>>(rcnt.as<int>(), rcnt2.as<int>(), nrows + 1);
    LAUNCHED();
  }
  nnz = (long long)used;
  CK(cudaMallocAsync(&piece.indices, sizeof(int) * std::max(nnz, 1LL), s));
  CK(cudaMallocAsync(&piece.data, sizeof(double) * std::max(nnz, 1LL), s));
  if (nrows) {
    k_row_gather<<<grid_for(nrows * 32, 256), 256, 0, s>>>(roff.as<long long>(), rcnt.as<int>(), roff2.as<long long>(),
                                                           rcnt2.as<int>(), piece.indptr, nrows, col.as<int>(),
                                                           val.as<double>(), piece.indices, piece.data);
    LAUNCHED();
  }
  piece.nnz = nnz;
  return NLG_OK;
}

struct Timing {
  double prep = 0, cand = 0, full = 0, part = 0, sing = 0, merge = 0, stage_r = 0;
};

// one row batch: returns NLG_OK and appends to `out`, or asks for a split
nlg_status run_batch(nlg_plan* pl, long long row_lo, long long row_hi, long long budget, bool allow_sample,
                     std::vector<Csr>& out, nlg_stats* st, Counters& ctr, Timing& tm,
                     unsigned long long* d_counters, unsigned long long* d_err, bool* need_split,
                     std::vector<long long>* cuts, bool no_analytic, bool* analytic_fallback) {
  *need_split = false;
  *analytic_fallback = false;
  cuts->clear();
  ArenaScope arena_scope(pl);
  Params P = pl->P;
  if (no_analytic) P.analytic = 0;  // (a retried batch: every pair integrated per record)
  P.row_lo = row_lo;
  P.row_hi = row_hi;
  P.narrow = (unsigned long long)(row_hi - row_lo) * (unsigned long long)P.J < 0xffffffffull;
  cudaStream_t s = pl->stream;
  const int K = P.K;
  cudaEvent_t ev[8];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { for (int i = 0; i < 8; ++i) cudaEventDestroy(e[i]); }
  } evg{ev};
  CK(cudaEventRecord(ev[0], s));
  // ---- root selection
  DevBuf needA, vmark, rflag, roots, nroots;
  CK(needA.alloc(K, s));
  CK(rflag.alloc(sizeof(int) * K, s));
  CK(roots.alloc(sizeof(int) * K, s));
  CK(nroots.alloc(sizeof(int), s));
  k_mark_a<<<grid_for(K, 256), 256, 0, s>>>(P, needA.as<unsigned char>());
  LAUNCHED();
  if (P.path == 2) {
    CK(vmark.alloc(P.V, s));
    CK(cudaMemsetAsync(vmark.p, 0, P.V, s));
    k_mark_vertices<<<grid_for(K, 256), 256, 0, s>>>(P, needA.as<unsigned char>(), vmark.as<unsigned char>());
    LAUNCHED();
  }
  k_mark_roots<<<grid_for(K, 256), 256, 0, s>>>(P, needA.as<unsigned char>(), vmark.as<unsigned char>(),
                                                 rflag.as<int>());
  LAUNCHED();
  {
    DevBuf idx;
    CK(idx.alloc(sizeof(int) * K, s));
    k_iota<<<grid_for(K, 256), 256, 0, s>>>(idx.as<int>(), K);
    LAUNCHED();
    size_t tb = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, tb, idx.as<int>(), rflag.as<int>(), roots.as<int>(),
                                  nroots.as<int>(), K, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceSelect::Flagged(tmp.p, tb, idx.as<int>(), rflag.as<int>(), roots.as<int>(),
                                  nroots.as<int>(), K, s));
    g_launches += 1;
  }
  int nR = 0;
  CK(rb_read(&nR, nroots.p, sizeof(int), s));
  CK(rb_sync(s));
  TRACE("sync 1881");
  DevBuf inR;  // element -> rank in the batch's root list, -1 if not a root
  CK(inR.alloc(sizeof(int) * K, s));
  CK(cudaMemsetAsync(inR.p, 0xff, sizeof(int) * K, s));
  if (nR) {
    k_rank<<<grid_for(nR, 256), 256, 0, s>>>(roots.as<int>(), nR, inR.as<int>());
    LAUNCHED();
  }
  // ---- candidate counts
  DevBuf cnt, off;
  CK(cnt.alloc(sizeof(int) * (size_t)kCnt * std::max(nR, 1), s));
  CK(off.alloc(sizeof(long long) * 6 * (size_t)(nR + 1), s));
  const int cand_blocks = (int)std::min<long long>((nR * 32LL + 255) / 256, 148 * 16);
  // a first attempt over very many roots counts a 1/16 sample of them: if
  // the extrapolation does not fit, the cuts are planned from it; if it
  // does, the exact count follows
  int stride = allow_sample && nR > (1 << 18) ? 16 : 1;
count_pass:
  if (stride > 1) CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (size_t)kCnt * nR, s));
  if (nR) {
    k_candidates<false><<<std::max(cand_blocks, 1), 256, 0, s>>>(
        P, pl->G, roots.as<int>(), nR, needA.as<unsigned char>(), inR.as<int>(), cnt.as<int>(), nullptr,
        nullptr, nullptr, nullptr, nullptr, stride);
    LAUNCHED();
  }
  {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, tb, cnt.as<int>(), off.as<long long>(), cub::Sum(), 0LL, nR + 1, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    for (int q = 0; q < 6; ++q) {
      // off[q] = exclusive scan of cnt[q] over nR+1 entries (last = total);
      // the (nR+1)-th input reads the next column's first entry, so scan nR
      // entries and write the total separately
      CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, cnt.as<int>() + (size_t)q * nR,
                                        off.as<long long>() + (size_t)q * (nR + 1), cub::Sum(), 0LL, nR, s));
      g_launches += 1;
    }
  }
  // totals: off[q][nR-1] + cnt[q][nR-1]
  long long tot[6] = {0, 0, 0, 0, 0, 0};
  if (nR) {
    long long lastoff[6];
    int lastcnt[6];
    for (int q = 0; q < 6; ++q) {
      CK(rb_read(&lastoff[q], off.as<long long>() + (size_t)q * (nR + 1) + nR - 1, sizeof(long long), s));
      CK(rb_read(&lastcnt[q], cnt.as<int>() + (size_t)q * nR + nR - 1, sizeof(int), s));
    }
    CK(rb_sync(s));
    TRACE("sync 1925");
    for (int q = 0; q < 6; ++q) {
      tot[q] = lastoff[q] + lastcnt[q];
      CK(cudaMemcpyAsync(off.as<long long>() + (size_t)q * (nR + 1) + nR, &tot[q], sizeof(long long),
                         cudaMemcpyHostToDevice, s));
    }
    // (the totals are stored before they are scaled: a sampled count only plans)
    for (int q = 0; q < 6; ++q) tot[q] *= stride;
  }
  const long long nUB = tot[C_FULL];  // upper bound of full + clipped records
  // records with stored blocks: all, or (analytic full pairs) the clipped ones
  const long long nStUB = P.analytic ? tot[C_PART] : nUB;
  const long long nS[3] = {tot[C_SID], tot[C_SED], tot[C_SVX]};
  const int NC = P.nc;
  const long long E = 9LL * NC * NC;
  {
    // kkv + klv per record side, the reduced COO (own blocks, singular slots,
    // stage-R runs at kRunFrac of the record values) with its sort buffers,
    // lists and indices
    // (stage W needs no run buffer: its COO is the singular slots, its
    // output the CSR entries at kEntFrac of the record values)
    const bool rows_plan = pl->use_rows;
    const long long coo_ub = (long long)nR * E + (nS[0] + nS[1] + nS[2]) * 36LL * NC * NC +
                             (rows_plan ? 0LL : (long long)(kRunFrac * (double)(nUB * 2 * E))) + 1;
    const long long ent_ub = rows_plan ? ent_estimate(P, nUB, tot[C_EPI], nR) : 0LL;
    const long long side_bytes = 8LL * (3 * NC * (3 * NC + 1) / 2 + (NC == 1 ? 12 : 36));  // kkv + klv
    // (ent_ub is ~1.5x the CSR entries: it covers the merge's entry buffer and
    // most of the batch's piece)
    const long long bytes = nStUB * 2 * side_bytes + coo_ub * (16 + 16) + ent_ub * 12 +
                            (2 * nUB + nS[0] + nS[1] + nS[2]) * 8 + nUB * 24;
    if (g_trace)
      fprintf(stderr, "[nlg] plan rows [%lld, %lld) stride %d: est %.1f GB (stored %.1f, entries %.1f) of budget %.1f GB\n",
              row_lo, row_hi, stride, 1e-9 * bytes, 1e-9 * nStUB * 2 * side_bytes, 1e-9 * ent_ub * 12, 1e-9 * budget);
    // 32-bit sizes: records (reverse-index sort) and COO entries must fit
    const bool too_big = (budget > 0 && bytes > budget) || coo_ub >= (1LL << 31) || nUB >= (1LL << 31);
    if (stride > 1 && !too_big) {  // the sample says it fits: count exactly
      stride = 1;
      goto count_pass;
    }
    if (too_big && row_hi - row_lo <= P.nc) {
      if (coo_ub < (1LL << 31) && nUB < (1LL << 31)) goto fits;  // one vertex's rows: try anyway
      set_err("a single row needs %lld COO slots", coo_ub);
      return NLG_ERR_CUDA;
    }
    if (too_big) {
      // plan the row cuts from this attempt's counts: per-row cost of the
      // roots (at their first in-range row), greedy cuts at 70% of each limit
      *need_split = true;
      const long long nrows = row_hi - row_lo;
      DevBuf rcost;
      CK(rcost.alloc(sizeof(unsigned long long) * 3 * nrows, s));
      CK(cudaMemsetAsync(rcost.p, 0, sizeof(unsigned long long) * 3 * nrows, s));
      const double store_bytes = 16.0 * (3 * NC * (3 * NC + 1) / 2 + (NC == 1 ? 12 : 36));
      const double rec_bytes = (rows_plan ? kEntFrac * 2 * E * 12 : kRunFrac * 2 * E * 32) + 40;
      const double sing_bytes = 36.0 * NC * NC * 32 + 8, root_bytes = E * 32.0 + 64;
      if (nR)
        k_root_cost<<<grid_for(nR, 256), 256, 0, s>>>(P, roots.as<int>(), nR, cnt.as<int>(), rec_bytes, store_bytes, sing_bytes,
                                                      root_bytes, rows_plan ? 0.0 : kRunFrac * 2 * E, 36.0 * NC * NC,
                                                      rcost.as<unsigned long long>(), (double)stride,
                                                      rows_plan ? kEntPerEpi * 0.5 * NC * 12.0 : 0.0);
      LAUNCHED();
      std::vector<unsigned long long> hcost((size_t)3 * nrows);
      CK(rb_read(hcost.data(), rcost.p, sizeof(unsigned long long) * 3 * nrows, s));
      CK(rb_sync(s));
      // cut fraction of each limit (the halo roots a batch adds are not in
      // the per-row costs).  Taller batches integrate fewer pairs twice -- a
      // config-4 shard takes 2,393 ms at 0.55 (6 batches), 2,283 at 0.7 (5),
      // 2,210 at 0.75 (4) -- but at 0.7 the eight shards of config 4 run one
      // after the other ran out of memory at the fourth (pieces + outputs)
      static const double pf = getenv("NLG_PLAN_FRAC") ? atof(getenv("NLG_PLAN_FRAC")) : 0.55;
      const double lim[3] = {budget > 0 ? pf * (double)budget : 1e300, pf * (double)(1LL << 31),
                             pf * (double)(1LL << 31)};
      double acc[3] = {0, 0, 0};
      for (long long r = 0; r < nrows; ++r) {
        const long long row = row_lo + r;
        bool over = false;
        for (int q = 0; q < 3; ++q) over |= acc[q] + (double)hcost[3 * r + q] > lim[q];
        if (over && row % P.nc == 0 && row > row_lo && (cuts->empty() || cuts->back() < row)) {
          cuts->push_back(row);
          acc[0] = acc[1] = acc[2] = 0;
        }
        for (int q = 0; q < 3; ++q) acc[q] += (double)hcost[3 * r + q];
      }
      return NLG_OK;
    }
  }
fits:
  // EPI of the roots whose home is this batch (read with the batch's last
  // synchronisation, counted only if the batch completes)
  DevBuf epib;
  CK(epib.alloc(2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(epib.p, 0, 2 * sizeof(unsigned long long), s));
  if (nR) {
    k_epi_home<<<grid_for(nR, 256), 256, 0, s>>>(cnt.as<int>(), nR, epib.as<unsigned long long>());
    LAUNCHED();
  }
  // ---- fill: records into per-root upper-bound ranges, then per-root compaction
  DevBuf comb, lists, own_a2;
  CK(own_a2.alloc(sizeof(double) * (size_t)std::max(nR, 1), s));  // analytic: per-root partner areas
  CK(comb.alloc(sizeof(int2) * (size_t)std::max(1LL, nUB), s));
  CK(lists.alloc(sizeof(int2) * (size_t)std::max(1LL, nUB + nS[0] + nS[1] + nS[2]), s));
  int2* lsing = lists.as<int2>() + nUB;
  int2* ls[3] = {lsing, lsing + nS[0], lsing + nS[0] + nS[1]};
  if (nR) {
    k_candidates<true><<<std::max(cand_blocks, 1), 256, 0, s>>>(
        P, pl->G, roots.as<int>(), nR, needA.as<unsigned char>(), inR.as<int>(), cnt.as<int>(),
        off.as<long long>(), comb.as<int2>(), ls[0], ls[1], ls[2], 1, own_a2.as<double>());
    LAUNCHED();
  }
  // actual per-root full / clipped counts -> list offsets (columns 4, 5 of
  // off; column 0 still holds the fill's upper-bound offsets), their totals
  long long nF = 0, nPt = 0;
  long long* offF = off.as<long long>() + 4 * (size_t)(nR + 1);
  long long* offP = off.as<long long>() + 5 * (size_t)(nR + 1);
  if (nR) {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, tb, cnt.as<int>(), off.as<long long>(), cub::Sum(), 0LL, nR, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, cnt.as<int>() + (size_t)C_FULL * nR, offF, cub::Sum(), 0LL, nR, s));
    CK(cub::DeviceScan::ExclusiveScan(tmp.p, tb, cnt.as<int>() + (size_t)C_PART * nR, offP, cub::Sum(), 0LL, nR, s));
    g_launches += 2;
    long long lo[2];
    int lc[2];
    CK(rb_read(&lo[0], offF + nR - 1, sizeof(long long), s));
    CK(rb_read(&lo[1], offP + nR - 1, sizeof(long long), s));
    CK(rb_read(&lc[0], cnt.as<int>() + (size_t)C_FULL * nR + nR - 1, sizeof(int), s));
    CK(rb_read(&lc[1], cnt.as<int>() + (size_t)C_PART * nR + nR - 1, sizeof(int), s));
    CK(rb_sync(s));
    TRACE("sync list totals");
    nF = lo[0] + lc[0];
    nPt = lo[1] + lc[1];
  }
  int2* lf = lists.as<int2>();
  int2* lp = lf + nF;
  if (nR) {
    k_split_records<<<grid_for((long long)nR * 32, 256), 256, 0, s>>>(comb.as<int2>(), off.as<long long>(), offF, offP,
                                                                      cnt.as<int>(), nR, lf, lp);
    LAUNCHED();
    // the roots' exact offsets where RootSides reads them (columns 0, 1)
    CK(cudaMemcpyAsync(off.as<long long>(), offF, sizeof(long long) * nR, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(off.as<long long>() + (size_t)(nR + 1), offP, sizeof(long long) * nR,
                       cudaMemcpyDeviceToDevice, s));
  }
  const long long nvis = nF + nPt;
  const long long nst = P.analytic ? nPt : nvis;  // records with stored blocks
  const long long coo = (long long)nR * E + nst * 2 * E + (nS[0] + nS[1] + nS[2]) * 36LL * NC * NC;
  // reverse index of side-B records by partner root, one per list (stable:
  // list order): per-root ranges, each record's reverse position (its side-B
  // block goes there) and the record's root at each position
  DevBuf rstartF, rstartP, revposF, revposP, partBF, partBP;
  auto reverse_index = [&](const int2* list, long long n, DevBuf& rstart, DevBuf& revpos, DevBuf& partB) -> nlg_status {
    DevBuf rkey, rkey2, ritem0, ritem;
    CK(rkey.alloc(sizeof(unsigned) * std::max(n, 1LL), s));
    CK(rkey2.alloc(sizeof(unsigned) * std::max(n, 1LL), s));
    CK(ritem0.alloc(sizeof(int) * std::max(n, 1LL), s));
    CK(ritem.alloc(sizeof(int) * std::max(n, 1LL), s));
    CK(rstart.alloc(sizeof(int) * (nR + 1), s));
    CK(revpos.alloc(sizeof(int) * std::max(n, 1LL), s));
    CK(partB.alloc(sizeof(int) * std::max(n, 1LL), s));
    if (n) {
      k_rev_keys<<<grid_for(n, 256), 256, 0, s>>>(list, n, inR.as<int>(), nR, rkey.as<unsigned>(), ritem0.as<int>());
      LAUNCHED();
      int rbits = 1;
      while ((1ll << rbits) <= nR) ++rbits;
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, rkey.as<unsigned>(), rkey2.as<unsigned>(), ritem0.as<int>(),
                                         ritem.as<int>(), (int)n, 0, rbits, s));
      DevBuf tmp;
      CK(tmp.alloc(tb, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, rkey.as<unsigned>(), rkey2.as<unsigned>(), ritem0.as<int>(),
                                         ritem.as<int>(), (int)n, 0, rbits, s));
      g_launches += 1 + (rbits + 7) / 8;
    }
    k_cell_ranges<<<grid_for(nR + 1, 256), 256, 0, s>>>(rkey2.as<unsigned>(), (int)n, nR, rstart.as<int>());
    LAUNCHED();
    if (n) {
      k_rev_pos<<<grid_for(n, 256), 256, 0, s>>>(ritem.as<int>(), n, list, revpos.as<int>(), partB.as<int>());
      LAUNCHED();
    }
    return NLG_OK;
  };
  // (the sort scratch of each index is released at the end of the batch)
  if (nlg_status r = reverse_index(lf, nF, rstartF, revposF, partBF)) return r;
  if (nlg_status r = reverse_index(lp, nPt, rstartP, revposP, partBP)) return r;
  CK(cudaEventRecord(ev[1], s));
  // ---- integrate
  const long long nsing_slots = (nS[0] + nS[1] + nS[2]) * 36LL * NC * NC;
  const long long r_base = (long long)nR * E + nsing_slots;
  const long long r_cap = (long long)(kRunFrac * (double)(nvis * 2 * E)) + 1;
  const bool rows_mode = pl->use_rows;
  DevBuf keys, vals, kkv, klv, vmaxb;
  // stage W needs the singular slots only; stage R also its run buffer
  CK(keys.alloc(sizeof(unsigned long long) * (r_base + (rows_mode ? 0 : r_cap)), s));
  CK(vals.alloc(sizeof(double) * (r_base + (rows_mode ? 0 : r_cap)), s));
  CK(vmaxb.alloc(sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(vmaxb.p, 0, sizeof(unsigned long long), s));
  DevBuf emaxb;  // per-element bounds of the emitted values (the merge's per-row fixed-point scale)
  CK(emaxb.alloc(sizeof(unsigned long long) * std::max(K, 1), s));
  CK(cudaMemsetAsync(emaxb.p, 0, sizeof(unsigned long long) * std::max(K, 1), s));
  unsigned long long* d_vmax = vmaxb.as<unsigned long long>();
  const long long nkk = 3LL * NC * (3 * NC + 1) / 2, kls = NC == 1 ? 12 : 36;  // Blk<NC>::NKK, KLS
  CK(kkv.alloc(sizeof(double) * 2 * nkk * std::max(nst, 1LL), s));
  CK(klv.alloc(sizeof(double) * 2 * kls * std::max(nst, 1LL), s));
  // block slots: [full A | full B | clipped A | clipped B], the full ones
  // only when they are stored
  const long long aF = 0, bF = nF, aP = P.analytic ? 0 : 2 * nF, bP = aP + nPt;
  VisitOut O;
  O.kkv = kkv.as<double>();
  O.klv = klv.as<double>();
  O.counters = d_counters;
  O.errpair = d_err;
  O.vmax = d_vmax;
  O.emax = emaxb.as<unsigned long long>();
  VisitOut OF = O, OP = O;
  OF.a_base = aF; OF.b_base = bF; OF.revpos = revposF.as<int>(); OF.nlist = P.analytic ? 0 : nF;
  OP.a_base = aP; OP.b_base = bP; OP.revpos = revposP.as<int>(); OP.nlist = nPt;
  nlg_status rc = NLG_OK;
  switch (P.kid) {
    case 0: rc = run_visits<0>(pl, P, lf, lp, OF, OP, ev[2]); break;
    case 1: rc = run_visits<1>(pl, P, lf, lp, OF, OP, ev[2]); break;
    case 2: rc = run_visits<2>(pl, P, lf, lp, OF, OP, ev[2]); break;
    default: rc = run_visits<3>(pl, P, lf, lp, OF, OP, ev[2]); break;
  }
  if (rc) return rc;
  CK(cudaEventRecord(ev[3], s));
  unsigned long long* ckeys = keys.as<unsigned long long>();
  double* cvals = vals.as<double>();
  const long long sbase = (long long)nR * E;
  switch (P.kid) {
    case 0: rc = run_singular<0>(pl, P, ls, nS, ckeys, cvals, sbase, d_counters, d_err, d_vmax, emaxb.as<unsigned long long>()); break;
    case 1: rc = run_singular<1>(pl, P, ls, nS, ckeys, cvals, sbase, d_counters, d_err, d_vmax, emaxb.as<unsigned long long>()); break;
    case 2: rc = run_singular<2>(pl, P, ls, nS, ckeys, cvals, sbase, d_counters, d_err, d_vmax, emaxb.as<unsigned long long>()); break;
    default: rc = run_singular<3>(pl, P, ls, nS, ckeys, cvals, sbase, d_counters, d_err, d_vmax, emaxb.as<unsigned long long>()); break;
  }
  if (rc) return rc;
  CK(cudaEventRecord(ev[4], s));
  // ---- merge stage R: per-root reduction of the record blocks
  RootIn RI;
  RI.roots = roots.as<int>();
  RI.nR = nR;
  RI.cnt = cnt.as<int>();
  RI.off = off.as<long long>();
  RI.nF = nF;
  RI.rec = lf;
  RI.rstartF = rstartF.as<int>();
  RI.rstartP = rstartP.as<int>();
  RI.partBF = partBF.as<int>();
  RI.partBP = partBP.as<int>();
  RI.aF = aF; RI.bF = bF; RI.aP = aP; RI.bP = bP;
  RI.analytic = P.analytic;
  RI.inR = inR.as<int>();
  RI.kkv = O.kkv;
  RI.own_a2 = own_a2.as<double>();
  RI.klv = O.klv;
  const long long nrows = row_hi - row_lo;
  Csr piece{row_lo, row_hi, 0, nullptr, nullptr, nullptr};
  long long nnz = 0;
  bool merged = false;
  if (rows_mode) {
    // ---- merge stage W: per-row fixed-point tables -> CSR rows
    bool fb = false, ns = false;
    const long long ent_cap = ent_estimate(P, nvis, tot[C_EPI], nR) + nR * E + nsing_slots + 1024;
    void* sk = P.narrow ? (void*)(reinterpret_cast<unsigned*>(keys.p) + sbase)
                        : (void*)(keys.as<unsigned long long>() + sbase);
    // distinct columns of a row ~ half the visits of a root (the partner vertices)
    const double cols_est = nR ? 0.55 * (double)tot[C_EPI] / (double)nR : 0.0;
    long long retries = 0;
    rc = merge_rows(pl, P, RI, sk, vals.as<double>() + sbase, nsing_slots, d_vmax, emaxb.as<unsigned long long>(),
                    ent_cap, cols_est, piece, nnz,
                    &fb, &ns, &retries);
    st->n_row_retries += retries;
    st->n_merge_fallbacks += fb ? 1 : 0;
    if (rc) return rc;
    if (ns) {
      if (row_hi - row_lo > 1) { *need_split = true; return NLG_OK; }
      set_err("a single row exceeds the entry buffer");
      return NLG_ERR_CUDA;
    }
    merged = !fb;
    if (fb && r_base + r_cap >= (1LL << 31) && row_hi - row_lo > P.nc) {  // stage R's 32-bit sorts
      *need_split = true;
      return NLG_OK;
    }
    if (fb && P.analytic) {
      // stage R needs every visit's record: the batch runs again without the
      // analytic enumeration (full pairs integrated per record)
      *analytic_fallback = true;
      return NLG_OK;
    }
    if (fb) {  // stage R + sort: the COO with its run buffer (singular slots carried over)
      TRACE("stage W fallback");
      DevBuf k2, v2;
      if (k2.alloc(sizeof(unsigned long long) * (r_base + r_cap), s) != cudaSuccess ||
          v2.alloc(sizeof(double) * (r_base + r_cap), s) != cudaSuccess) {
        // the batch was planned for stage W; its stage-R buffer does not fit: split
        cudaGetLastError();
        if (row_hi - row_lo > P.nc) { *need_split = true; return NLG_OK; }
        set_err("stage-R fallback buffer for one row does not fit");
        return NLG_ERR_CUDA;
      }
      CK(cudaMemcpyAsync(k2.p, keys.p, (P.narrow ? 4 : 8) * r_base, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(v2.p, vals.p, sizeof(double) * r_base, cudaMemcpyDeviceToDevice, s));
      std::swap(keys.p, k2.p);
      std::swap(vals.p, v2.p);
      std::swap(keys.arena, k2.arena);
      std::swap(vals.arena, v2.arena);
      ckeys = keys.as<unsigned long long>();
      cvals = vals.as<double>();
    }
  }
  long long r_total = 0;
  if (nR && !merged) {
    DevBuf nch, cfirst, rstate;
    CK(nch.alloc(sizeof(int) * (nR + 1), s));
    CK(cfirst.alloc(sizeof(int) * (nR + 1), s));
    // chunk upper bound: one per root plus the items beyond
    const long long max_chunks = nR + (3 * 2 * nvis + kRootCap - 1) / kRootCap + 1;
    CK(rstate.alloc(sizeof(unsigned long long) * (max_chunks + 4), s));
    CK(cudaMemsetAsync(rstate.p, 0, sizeof(unsigned long long) * (max_chunks + 4), s));
    CK(cudaMemsetAsync(nch.as<int>() + nR, 0, sizeof(int), s));
    k_root_chunks<<<grid_for(nR, 256), 256, 0, s>>>(RI, nch.as<int>());
    LAUNCHED();
    {
      size_t tb = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, nch.as<int>(), cfirst.as<int>(), nR + 1, s));
      DevBuf tmp;
      CK(tmp.alloc(tb, s));
      CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, nch.as<int>(), cfirst.as<int>(), nR + 1, s));
      g_launches += 1;
    }
    RI.chunk_first = cfirst.as<int>();
    DevBuf croot;
    CK(croot.alloc(sizeof(int) * max_chunks, s));
    k_root_chunk_map<<<grid_for(nR, 256), 256, 0, s>>>(RI, croot.as<int>());
    LAUNCHED();
    RI.chunk_root = croot.as<int>();
    unsigned long long* st64 = rstate.as<unsigned long long>();
    RootOut RO;
    RO.lb = st64 + 4;
    RO.ticket = (unsigned*)st64;  // st64[0]: ticket, st64[1]: overflow, st64[2]: total
    RO.overflow = (int*)(st64 + 1);
    RO.total = st64 + 2;
    RO.keys = ckeys;
    RO.vals = cvals;
    RO.kk_base = 0;
    RO.r_base = r_base;
    RO.r_cap = r_cap;
    RO.errpair = d_err;
    int key_bits = 1;
    while ((1LL << key_bits) - 1 < (long long)P.J / NC) ++key_bits;
    if (key_bits > 31) { set_err("dof count too large for the run sort"); return NLG_ERR_CONFIG; }
    if (NC == 1) {
      const int smem = (int)sizeof(RootSmem<1>);
      auto kern = P.analytic ? k_root_reduce<1, true> : k_root_reduce<1, false>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<(unsigned)max_chunks, kRootThreads, smem, s>>>(P, RI, RO, key_bits);
    } else {
      const int smem = (int)sizeof(RootSmem<2>);
      CK(cudaFuncSetAttribute(k_root_reduce<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_root_reduce<2, false><<<(unsigned)max_chunks, kRootThreads, smem, s>>>(P, RI, RO, key_bits);
    }
    LAUNCHED();
    unsigned long long hst[3];
    CK(rb_read(hst, st64, sizeof hst, s));
    CK(rb_sync(s));
    TRACE("stage R done");
    if (hst[1] & 0xffffffffull) {  // the runs exceed the estimate: split the rows
      if (row_hi - row_lo > 1) { *need_split = true; return NLG_OK; }
      set_err("a single row exceeds the run buffer");
      return NLG_ERR_CUDA;
    }
    r_total = (long long)hst[2];
  }
  CK(cudaEventRecord(ev[6], s));
  if (!merged) {
    const long long coo_red = r_base + r_total;
    // ---- sort (row, col) keys (stable: equal keys keep COO position order), sum runs
    long long kept = 0;
    rc = P.narrow ? merge_csr<unsigned>(s, P, ckeys, cvals, coo_red, nrows, piece, nnz, &kept, true)
                  : merge_csr<unsigned long long>(s, P, ckeys, cvals, coo_red, nrows, piece, nnz, &kept);
    st->coo_reduced += kept;
    if (rc) return rc;
    piece.nnz = nnz;
  } else {
    st->coo_reduced += nnz;
  }
  out.push_back(piece);
  CK(cudaEventRecord(ev[5], s));
  unsigned long long hepi[2] = {0, 0};
  CK(rb_read(hepi, epib.p, sizeof hepi, s));
  CK(rb_sync(s));
  TRACE("sync 2089");
  st->epi += (long long)hepi[0];
  st->n_roots += (long long)hepi[1];
  float ms;
  CK(cudaEventElapsedTime(&ms, ev[0], ev[1])); tm.cand += ms;
  CK(cudaEventElapsedTime(&ms, ev[1], ev[2])); tm.full += ms;
  CK(cudaEventElapsedTime(&ms, ev[2], ev[3])); tm.part += ms;
  CK(cudaEventElapsedTime(&ms, ev[3], ev[4])); tm.sing += ms;
  CK(cudaEventElapsedTime(&ms, ev[4], ev[5])); tm.merge += ms;
  CK(cudaEventElapsedTime(&ms, ev[4], ev[6])); tm.stage_r += ms;
  st->n_full += nF;
  st->n_partial += nPt;
  st->n_singular += nS[0] + nS[1] + nS[2];
  st->coo_entries += coo;
  st->n_batches += 1;
  (void)ctr;
  return NLG_OK;
}

// Host outputs: a page-locked block laid out as [data | indices | indptr]
// with room for `nnz_cap` entries; a batch's piece is copied there on the
// plan's copy stream as soon as the batch is merged, while the next batch
// computes.  The block is either the caller's (nlg_assemble_pinned: the CSR
// is left there, no host copy at all) or the library's staging (nlg_assemble
// with out_on_host: a threaded copy into the caller's pageable buffers ends
// the call).
struct HostArena {  // nlg_assemble_pinned: where the caller's block comes from, and the result
  nlg_alloc_fn alloc = nullptr;
  void* user = nullptr;
  nlg_host_csr* out = nullptr;
};
struct Stager {
  nlg_plan* pl = nullptr;
  DeviceScratch* ds = nullptr;
  char* base = nullptr;
  long long nnz_cap = 0, used = 0, nrows = 0;
  bool on = false;
  std::vector<cudaEvent_t> tev;  // NLG_TRACE: copy start / end events per piece
  std::vector<long long> tnnz;
  double* dat() const { return (double*)base; }
  int* idx() const { return (int*)(base + off_idx(nnz_cap)); }
  long long* ptr() const { return (long long*)(base + off_ptr(nnz_cap)); }
  static size_t off_idx(long long nnz) { return 8 * (size_t)nnz; }
  static size_t off_ptr(long long nnz) { return (12 * (size_t)nnz + 15) & ~(size_t)15; }
  static size_t bytes(long long nnz, long long nrows) { return off_ptr(nnz) + 8 * (nrows + 1); }
  // the library's own staging, grown to hold nnz entries
  static char* own(DeviceScratch* d, long long nnz, long long nrows) {
    if (d->pinned_cap < bytes(nnz, nrows)) {
      if (d->pinned) cudaFreeHost(d->pinned);
      d->pinned = nullptr;
      d->pinned_cap = 0;
      if (cudaHostAlloc((void**)&d->pinned, bytes(nnz, nrows), cudaHostAllocPortable) == cudaSuccess)
        d->pinned_cap = bytes(nnz, nrows);
      else
        cudaGetLastError();
    }
    return d->pinned;
  }
  void begin(nlg_plan* p, DeviceScratch* d, long long nrows_, const HostArena* ha, unsigned long long sig) {
    pl = p;
    ds = d;
    nrows = nrows_;
    base = nullptr;
    nnz_cap = 0;
    used = 0;
    on = false;
    // the size hint is the largest output seen so far (of this problem and
    // row range, for a caller's block); without one, everything is copied at the end
    if (!p->cstream || !d->pin_nnz || getenv("NLG_NO_STAGE")) return;
    if (ha) {
      if (d->pin_sig != sig) return;
      base = (char*)ha->alloc(ha->user, (int64_t)bytes(d->pin_nnz, nrows), 5);
    } else {
      base = own(d, d->pin_nnz, nrows);
    }
    if (!base) return;
    nnz_cap = d->pin_nnz;
    on = true;
  }
  // queue the D2H of a finished piece (its buffers stay alive until emit)
  nlg_status stage(Csr& c) {
    if (!on || used + c.nnz > nnz_cap) {
      on = false;  // out of room: the rest (and everything) is copied at the end
      return NLG_OK;
    }
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, pl->stream));
    CK(cudaStreamWaitEvent(pl->cstream, ev, 0));
    cudaEventDestroy(ev);
    if (g_trace) {  // when each piece's copy starts and ends (NLG_TRACE)
      cudaEvent_t a;
      cudaEventCreate(&a);
      cudaEventRecord(a, pl->cstream);
      tev.push_back(a);
    }
    if (c.nnz) {
      CK(cudaMemcpyAsync(dat() + used, c.data, sizeof(double) * c.nnz, cudaMemcpyDeviceToHost, pl->cstream));
      CK(cudaMemcpyAsync(idx() + used, c.indices, sizeof(int) * c.nnz, cudaMemcpyDeviceToHost, pl->cstream));
    }
    if (g_trace) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecord(b, pl->cstream);
      tev.push_back(b);
      tnnz.push_back(c.nnz);
    }
    c.staged = used;
    used += c.nnz;
    return NLG_OK;
  }
};

// Concatenate row-ordered CSR pieces into the caller's buffers (alloc which
// = 0 indptr, 1 indices, 2 data; or the caller's page-locked block, `ha`);
// frees the pieces.
nlg_status emit_pieces(nlg_plan* pl, DeviceScratch& ds, std::vector<Csr>& pieces, long long row_lo, long long row_hi,
                       int out_on_host, nlg_alloc_fn alloc, void* user, cudaEvent_t e_done, long long* nnz_out,
                       Stager& stg, const HostArena* ha, unsigned long long sig) {
  cudaStream_t s = pl->stream;
  long long nnz = 0;
  for (auto& p : pieces) nnz += p.nnz;
  const long long nrows = row_hi - row_lo;
  long long* u_ptr = nullptr;
  int* u_idx = nullptr;
  double* u_dat = nullptr;
  if (!ha) {
    // a caller's device allocation may fail only because this library holds
    // the memory: the batches' freed scratch in the stream-ordered pool, then
    // the scratch arena itself (sized by the largest call so far; the batches
    // are done with it, and the next call grows it again).  Hand them back
    // and ask again.
    auto ask = [&](size_t n, int which) -> void* {
      void* p = alloc(user, (int64_t)n, which);
      cudaMemPool_t mp;
      if (!p && !out_on_host && cudaDeviceGetDefaultMemPool(&mp, pl->device) == cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(s);
        cudaMemPoolTrimTo(mp, 0);
        p = alloc(user, (int64_t)n, which);
      }
      if (!p && !out_on_host && ds.arena) {
        cudaGetLastError();
        cudaStreamSynchronize(s);
        cudaFree(ds.arena);
        ds.arena = nullptr;
        ds.cap = 0;
        ds.peak = 0;  // (regrown to what the next call needs)
        p = alloc(user, (int64_t)n, which);
      }
      return p;
    };
    u_ptr = (long long*)ask(sizeof(long long) * (nrows + 1), 0);
    u_idx = (int*)ask(sizeof(int) * std::max(nnz, 1LL), 1);
    u_dat = (double*)ask(sizeof(double) * std::max(nnz, 1LL), 2);
    if (!u_ptr || !u_idx || !u_dat) { set_err("output allocation failed"); return NLG_ERR_CUDA; }
  }
  // where the D2H copies land: the caller's buffers (device outputs; or host
  // outputs when no page-locked block is available) or the block
  long long* o_ptr = u_ptr;
  int* o_idx = u_idx;
  double* o_dat = u_dat;
  bool all_staged = false;
  stg.pl = pl;
  stg.ds = &ds;
  if (out_on_host) {
    all_staged = stg.on;
    for (auto& p : pieces) all_staged = all_staged && p.staged >= 0;
    if (!all_staged) {
      // (first call, or the output outgrew the hint): one block of this size
      if (pl->cstream) CK(cudaStreamSynchronize(pl->cstream));
      // (the same 1/8 headroom as the hint of later calls, so a pooled block fits them too)
      stg.nnz_cap = std::max(nnz + nnz / 8, 1LL);
      if (ha) {
        stg.base = (char*)ha->alloc(ha->user, (int64_t)Stager::bytes(stg.nnz_cap, nrows), 5);
        if (!stg.base) { set_err("output allocation failed (page-locked block)"); return NLG_ERR_CUDA; }
      } else {
        stg.base = Stager::own(&ds, stg.nnz_cap, nrows);
      }
    }
    if (stg.base) {
      o_dat = stg.dat();
      o_idx = stg.idx();
      o_ptr = stg.ptr();
    }
    ds.pin_nnz = ds.pin_sig == sig ? std::max(ds.pin_nnz, nnz + nnz / 8) : nnz + nnz / 8;  // the next call stages batch by batch
    ds.pin_sig = sig;
  }
  DevBuf ptrbuf;
  CK(ptrbuf.alloc(sizeof(long long) * (nrows + 1), s));
  long long run = 0;
  for (auto& p : pieces) {
    const long long nr = p.row_hi - p.row_lo;
    if (run) {
      k_add_offset<<<grid_for(nr + 1, 256), 256, 0, s>>>(p.indptr, nr + 1, run);
      LAUNCHED();
    }
    CK(cudaMemcpyAsync(ptrbuf.as<long long>() + (p.row_lo - row_lo), p.indptr, sizeof(long long) * (nr + 1),
                       cudaMemcpyDeviceToDevice, s));
    if (p.nnz && !(out_on_host && all_staged)) {
      CK(cudaMemcpyAsync(o_idx + run, p.indices, sizeof(int) * p.nnz, cudaMemcpyDefault, s));
      CK(cudaMemcpyAsync(o_dat + run, p.data, sizeof(double) * p.nnz, cudaMemcpyDefault, s));
    }
    run += p.nnz;
  }
  if (nrows == 0) CK(cudaMemsetAsync(ptrbuf.p, 0, sizeof(long long), s));
  CK(cudaMemcpyAsync(o_ptr, ptrbuf.p, sizeof(long long) * (nrows + 1), cudaMemcpyDefault, s));
  if (e_done) CK(cudaEventRecord(e_done, s));
  TRACE("outputs queued");
  CK(cudaStreamSynchronize(s));
  if (pl->cstream) CK(cudaStreamSynchronize(pl->cstream));
  TRACE("outputs synced");
  if (g_trace && e_done) {
    for (size_t i = 0; i + 1 < stg.tev.size(); i += 2) {
      float t0 = 0, t1 = 0;
      cudaEventElapsedTime(&t0, stg.tev[i], e_done);
      cudaEventElapsedTime(&t1, stg.tev[i + 1], e_done);
      fprintf(stderr, "[nlg] piece %zu: %.2f GB copied from %.1f to %.1f ms before the end (%.1f GB/s)\n", i / 2,
              12e-9 * stg.tnnz[i / 2], t0, t1, 12e-6 * stg.tnnz[i / 2] / std::max(t0 - t1, 1e-3f));
    }
    for (auto e : stg.tev) cudaEventDestroy(e);
    stg.tev.clear();
    stg.tnnz.clear();
  }
  const size_t b_dat = sizeof(double) * std::max(nnz, 1LL), b_idx = sizeof(int) * std::max(nnz, 1LL),
               b_ptr = sizeof(long long) * (nrows + 1);
  if (ha) {
    ha->out->arena = stg.base;
    ha->out->nnz = nnz;
    ha->out->off_data = 0;
    ha->out->off_indices = (int64_t)Stager::off_idx(stg.nnz_cap);
    ha->out->off_indptr = (int64_t)Stager::off_ptr(stg.nnz_cap);
  } else if (out_on_host && o_dat != u_dat) {  // library staging -> caller buffers
    struct Part { void* dst; const void* src; size_t n; };
    const Part parts[3] = {{u_dat, o_dat, b_dat}, {u_idx, o_idx, b_idx}, {u_ptr, o_ptr, b_ptr}};
    const int nt = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t]() {
        for (const Part& q : parts) {
          const size_t chunk = (q.n + nt - 1) / nt, a = std::min(q.n, chunk * t), b = std::min(q.n, a + chunk);
          if (b > a) memcpy((char*)q.dst + a, (const char*)q.src + a, b - a);
        }
      });
    for (auto& x : th) x.join();
    TRACE("host copy done");
  }

  for (auto& p : pieces) { cudaFreeAsync(p.indptr, s); cudaFreeAsync(p.indices, s); cudaFreeAsync(p.data, s); }
  pieces.clear();
  *nnz_out = nnz;
  return NLG_OK;
}

nlg_status upload_table(const double* h, size_t n, double** d, cudaStream_t s) {
  CK(cudaMallocAsync(d, sizeof(double) * std::max<size_t>(n, 1), s));
  if (n) CK(cudaMemcpyAsync(*d, h, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  return NLG_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

int32_t nlg_abi_version(void) { return NLG_ABI_VERSION; }
const char* nlg_last_error(void) { return g_err.c_str(); }
int64_t nlg_launch_count(void) { return g_launches.load(); }

int64_t nlg_last_batches(const nlg_plan* pl, int64_t* ranges, int64_t cap) {
  if (!pl) return -1;
  const int64_t n = (int64_t)pl->last_batches.size() / 2;
  for (int64_t i = 0; i < std::min(n, cap); ++i) {
    ranges[2 * i] = pl->last_batches[2 * i];
    ranges[2 * i + 1] = pl->last_batches[2 * i + 1];
  }
  return n;
}

nlg_status nlg_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    set_err("cudaGetDeviceCount: %s", cudaGetErrorString(e));
    return NLG_ERR_CUDA;
  }
  *count = n;
  return NLG_OK;
}

nlg_status nlg_plan_create(int32_t device, const nlg_problem* pb, void* stream, nlg_plan** out) {
  *out = nullptr;
  if (!pb) { set_err("null problem"); return NLG_ERR_CONFIG; }
  if (pb->n_outer != 7 || pb->n_inner != 7) { set_err("only the 7-point triangle rule is supported"); return NLG_ERR_CONFIG; }
  if (pb->kernel_id < 0 || pb->kernel_id > 3) { set_err("unknown kernel id %d", pb->kernel_id); return NLG_ERR_CONFIG; }
  const int want_nc = pb->kernel_id == 1 ? 2 : 1;
  if (pb->nc != want_nc) { set_err("kernel id %d needs nc=%d, got %d", pb->kernel_id, want_nc, pb->nc); return NLG_ERR_CONFIG; }
  if ((pb->kernel_id == 3) == (pb->symmetric != 0)) { set_err("kernel id %d has the wrong symmetry flag", pb->kernel_id); return NLG_ERR_CONFIG; }
  if (pb->ball_id < 0 || pb->ball_id > 2 || pb->path_touch < 0 || pb->path_touch > 2) { set_err("bad ball/path id"); return NLG_ERR_CONFIG; }
  if (pb->n_elements < 0 || pb->n_vertices < 0 || pb->n_elements >= (1LL << 30) || pb->n_vertices >= (1LL << 31)) {
    set_err("mesh size out of range"); return NLG_ERR_CONFIG;
  }
  if (pb->n_dofs <= 0 || pb->n_dofs >= (1LL << 31)) { set_err("dof count out of range"); return NLG_ERR_CONFIG; }
  if (pb->has_label_scale)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < a; ++b)
        if (!(pb->label_scale[a * 3 + b] == pb->label_scale[b * 3 + a])) {
          set_err("label_scale must be symmetric (one factor per element pair)");
          return NLG_ERR_CONFIG;
        }
  CK(cudaSetDevice(device));
  nlg_plan* pl = new nlg_plan();
  pl->device = device;
  pl->stream = (cudaStream_t)stream;
  if (cudaStreamCreateWithFlags(&pl->cstream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    pl->cstream = nullptr;
  }
  cudaStream_t s = pl->stream;
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  Params& P = pl->P;
  P.K = (int)pb->n_elements;
  P.V = (int)pb->n_vertices;
  P.nc = pb->nc;
  P.kid = pb->kernel_id;
  P.ball = pb->ball_id;
  P.path = pb->path_touch;
  P.sym = pb->symmetric;
  P.is_dg = pb->is_dg;
  P.s = pb->s;
  P.kexp = -1.0 - pb->s;
  P.cst = pb->scale;
  P.delta = pb->delta;
  P.prer = pb->ball_id == 2 ? pb->delta * sqrt(2.0) : pb->delta;  // _engine.py:445
  P.rskip2 = pb->rskip2;
  P.drop2 = pb->drop2;
  P.kp0 = pb->kp0;
  P.kp1 = pb->kp1;
  P.has_lab = pb->has_label_scale != 0;
  for (int i = 0; i < 9; ++i) P.lab[i] = P.has_lab ? pb->label_scale[i] : 1.0;
  P.J = pb->n_dofs;
  P.dbg = getenv("NLG_DEBUG") ? atoi(getenv("NLG_DEBUG")) : 0;
  // NLG_NO_ANALYTIC: integrate the full pairs of kid 2 / 3 per record (A/B and tests)
  // (nonfinite kernel parameters: every pair is integrated per record, so the
  // failing visit is detected and named -- the analytic sums carry no check)
  pl->use_rows = !(getenv("NLG_MERGE") && !strcmp(getenv("NLG_MERGE"), "sort"));
  // (the analytic visits are enumerated by the stage-W row merge: stage R
  // integrates every pair per record)
  P.analytic = (P.kid == 2 || P.kid == 3) && P.path == 0 && P.nc == 1 && !getenv("NLG_NO_ANALYTIC") &&
               std::isfinite(P.cst) && std::isfinite(P.kp0) && std::isfinite(P.kp1) && pl->use_rows &&
               !P.has_lab;  // (the analytic column factors carry one kernel constant)
  Rule7 hr;
  for (int p = 0; p < 7; ++p) {
    hr.op[p][0] = pb->op[2 * p]; hr.op[p][1] = pb->op[2 * p + 1];
    hr.ip[p][0] = pb->ip[2 * p]; hr.ip[p][1] = pb->ip[2 * p + 1];
    hr.ow[p] = pb->ow[p]; hr.iw[p] = pb->iw[p];
    for (int a = 0; a < 3; ++a) hr.oh[p][a] = pb->oh[3 * p + a];
  }
  // fast-path tables use the outer rule for both sides: they must agree
  for (int p = 0; p < 7; ++p)
    if (hr.op[p][0] != hr.ip[p][0] || hr.op[p][1] != hr.ip[p][1] || hr.ow[p] != hr.iw[p]) {
      set_err("outer and inner rules differ");
      delete pl;
      return NLG_ERR_CONFIG;
    }
  hr.iws = 0.0;
  for (int p = 0; p < 7; ++p) hr.iws += hr.iw[p];
  for (int p = 0; p < 7; ++p)
    for (int a = 0; a < 3; ++a) {
      hr.wh[p][a] = hr.ow[p] * hr.oh[p][a];
      for (int b = 0; b < 3; ++b) hr.whh[p][a * 3 + b] = hr.ow[p] * hr.oh[p][a] * hr.oh[p][b];
    }
  {
    const int tr = g_trace ? 1 : 0;
    cudaMemcpyToSymbolAsync(g_trace_dev, &tr, sizeof tr, 0, cudaMemcpyHostToDevice, s);
  }
  {
    static PowTab ptab;
    static std::once_flag ptab_once;
    std::call_once(ptab_once, [] { pow_tab_fill(&ptab); });
    cudaMemcpyToSymbolAsync(c_powtab, &ptab, sizeof ptab, 0, cudaMemcpyHostToDevice, s);
  }
  if (cudaMemcpyToSymbolAsync(c_rule, &hr, sizeof hr, 0, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    set_err("rule upload failed");
    delete pl;
    return NLG_ERR_CUDA;
  }
  const long long V = pb->n_vertices, K = pb->n_elements;
  nlg_status rc = NLG_OK;
  auto fail = [&](nlg_status r) { nlg_plan_destroy(pl); return r; };
  if (cudaMallocAsync(&pl->vtx, sizeof(double2) * std::max(V, 1LL), s) ||
      cudaMallocAsync(&pl->elem, sizeof(int4) * std::max(K, 1LL), s) ||
      cudaMallocAsync(&pl->dofs, sizeof(int4) * std::max(K, 1LL), s) ||
      cudaMallocAsync(&pl->ctr, sizeof(double2) * std::max(K, 1LL), s) ||
      cudaMallocAsync(&pl->rad, sizeof(double) * std::max(K, 1LL), s) ||
      (P.analytic && cudaMallocAsync(&pl->ftab, sizeof(double4) * std::max(K, 1LL), s)) ||
      cudaMallocAsync(&pl->fmax, 4 * sizeof(unsigned long long), s)) {
    set_err("device allocation failed");
    return fail(NLG_ERR_CUDA);
  }
  {
    // stage inputs on the device (copy when they are host arrays)
    const double* dv = pb->vertices;
    const long long *de = (const long long*)pb->elements, *dl = (const long long*)pb->labels,
                    *dou = (const long long*)pb->outer_mask, *dd = (const long long*)pb->dof_map;
    DevBuf sv, se, sl, so, sd;
    if (!pb->inputs_on_device) {
      if (sv.alloc(sizeof(double) * 2 * V, s) || se.alloc(sizeof(long long) * 3 * K, s) ||
          sl.alloc(sizeof(long long) * K, s) || so.alloc(sizeof(long long) * K, s) ||
          sd.alloc(sizeof(long long) * 3 * K, s)) {
        set_err("device allocation failed");
        return fail(NLG_ERR_CUDA);
      }
      if (V) cudaMemcpyAsync(sv.p, pb->vertices, sizeof(double) * 2 * V, cudaMemcpyHostToDevice, s);
      if (K) {
        cudaMemcpyAsync(se.p, pb->elements, sizeof(long long) * 3 * K, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(sl.p, pb->labels, sizeof(long long) * K, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(so.p, pb->outer_mask, sizeof(long long) * K, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(sd.p, pb->dof_map, sizeof(long long) * 3 * K, cudaMemcpyHostToDevice, s);
      }
      dv = sv.as<double>();
      de = se.as<long long>();
      dl = sl.as<long long>();
      dou = so.as<long long>();
      dd = sd.as<long long>();
    }
    const long long n = std::max(V, K);
    if (n) {
      k_convert<<<grid_for(n, 256), 256, 0, s>>>(dv, (const long long*)de, (const long long*)dl,
                                                 (const long long*)dou, (const long long*)dd, (int)V, (int)K,
                                                 pl->vtx, pl->elem, pl->dofs);
      g_launches += 1;
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { set_err("convert: %s", cudaGetErrorString(e)); return fail(NLG_ERR_CUDA); }
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { set_err("staging inputs: %s", cudaGetErrorString(e)); return fail(NLG_ERR_CUDA); }
  }
  for (int f = 0; f < 3; ++f) {
    const size_t n = (size_t)pb->n_sing[f];
    pl->sing_n[f] = pb->n_sing[f];
    const double* src[5] = {pb->sxs[f], pb->sys[f], pb->sw[f], pb->shx[f], pb->shy[f]};
    const size_t len[5] = {2 * n, 2 * n, n, 3 * n, 3 * n};
    for (int t = 0; t < 5; ++t) {
      if (n && !src[t]) { set_err("missing singular table"); return fail(NLG_ERR_CONFIG); }
      rc = upload_table(src[t], n ? len[t] : 0, &pl->sing_tab[f][t], s);
      if (rc) return fail(rc);
    }
  }
  P.vtx = pl->vtx;
  P.elem = pl->elem;
  P.dofs = pl->dofs;
  P.ctr = pl->ctr;
  P.rad = pl->rad;
  P.ftab = pl->ftab;
  *out = pl;
  return NLG_OK;
}

void nlg_plan_destroy(nlg_plan* pl) {
  if (!pl) return;
  cudaSetDevice(pl->device);
  cudaStream_t s = pl->stream;
  void* ptrs[] = {pl->vtx,        pl->elem,       pl->dofs,     pl->ctr,      pl->rad,     pl->ftab,
                  pl->fmax,       pl->de_start,   pl->de_items, pl->grid_start, pl->grid_items, pl->act,
                  pl->grid_el,    pl->grid_ctr,   pl->grid_rad, pl->grid_ft, pl->grid_dof,
                  pl->col_start,  pl->col_id,     pl->col_pos,  pl->grid_csum};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, s);
  for (auto& f : pl->sing_tab)
    for (double* p : f)
      if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  if (pl->cstream) cudaStreamDestroy(pl->cstream);
  delete pl;
}

static nlg_status assemble_impl(nlg_plan* pl, int64_t row_lo, int64_t row_hi, int32_t out_on_host,
                                nlg_alloc_fn alloc, void* user, int64_t budget, nlg_stats* stats,
                                const HostArena* ha) {
  if (!pl || !alloc) { set_err("null plan or allocator"); return NLG_ERR_CONFIG; }
  if (row_lo < 0 || row_hi > pl->P.J || row_lo > row_hi) { set_err("row range out of bounds"); return NLG_ERR_CONFIG; }
  CK(cudaSetDevice(pl->device));
  cudaStream_t s = pl->stream;
  if (pl->device < 0 || pl->device >= 64) { set_err("device index out of range"); return NLG_ERR_CONFIG; }
  DeviceScratch& ds = g_scratch[pl->device];
  std::lock_guard<std::mutex> scratch_lock(ds.mu);
  // grow the device arena to the peak an earlier call needed
  if (ds.peak > ds.cap) {
    CK(cudaStreamSynchronize(s));
    if (ds.arena) cudaFree(ds.arena);
    ds.arena = nullptr;
    ds.cap = 0;
    const size_t cap = ds.peak + ds.peak / 8;
    if (cudaMalloc((void**)&ds.arena, cap) == cudaSuccess) ds.cap = cap;
    else cudaGetLastError();
  }
  pl->arena_used = 0;
  ds.rb_pending.clear();  // (reads queued by a call that failed midway)
  ds.rb_used = 0;
  struct ArenaActivate {
    ArenaActivate(nlg_plan* p) { g_arena_plan = p; }
    ~ArenaActivate() { g_arena_plan = nullptr; }
  } arena_on(pl);
  nlg_stats st;
  memset(&st, 0, sizeof st);
  st.err_k = st.err_l = -1;
  TRACE("assemble begin");
  if (budget <= 0) {
    // 60 % of the device by default.  Fewer row batches are faster -- a pair
    // whose elements fall in different batches is integrated once per batch
    // (config 5: one batch 768 ms at mem_budget = 75 %, three batches 825 ms)
    // -- but the scratch arena, the stream-ordered pool, the finished pieces
    // and the caller's own buffers share the device, and a process that has
    // assembled other problems before holds more of it: callers that know
    // their process pass a larger mem_budget (bench.py does).
    static thread_local size_t totm = 0;
    if (!totm) {
      size_t fr = 0;
      CK(cudaMemGetInfo(&fr, &totm));
    }
    budget = (long long)(0.6 * (double)totm);
  }
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventRecord(e0, s));
  pl->prepped = false;  // bounds and grid are part of every assembly
  TRACE("prep");
  nlg_status rc = prep(pl);
  TRACE("prep done");
  if (rc) return rc;
  CK(cudaEventRecord(e1, s));
  DevBuf dctr, derr;
  CK(dctr.alloc_pool(sizeof(unsigned long long) * K_NCOUNTERS, s));
  CK(derr.alloc_pool(2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(dctr.p, 0, sizeof(unsigned long long) * K_NCOUNTERS, s));
  CK(cudaMemsetAsync(derr.p, 0xff, 2 * sizeof(unsigned long long), s));
  std::vector<Csr> pieces;
  Stager stg;
  // (the size hint of a caller's block belongs to one problem and row range)
  unsigned long long sig = 1469598103934665603ull;
  for (unsigned long long v : {(unsigned long long)pl->P.K, (unsigned long long)pl->P.J, (unsigned long long)row_lo,
                               (unsigned long long)row_hi, (unsigned long long)pl->P.kid,
                               (unsigned long long)__builtin_bit_cast(long long, pl->P.delta)})
    sig = (sig ^ v) * 1099511628211ull;
  if (out_on_host) stg.begin(pl, &ds, row_hi - row_lo, ha, sig);
  Counters ctr{};
  Timing tm;
  // row batches: a work list of ranges, split in halves when over budget
  struct Range {
    long long first, second;
    bool plain;  // without the analytic enumeration (after a stage-W overflow)
  };
  std::vector<Range> todo;
  if (row_hi > row_lo) todo.push_back({row_lo, row_hi, false});
  // Streamed host output (>= 0.4 GB): a batch's rows are copied while the
  // NEXT batch computes, and nothing overlaps the last batch's copy.  Three
  // row chunks of 62 / 26 / 12 %: each copy fits inside the next chunk's
  // compute (the copy engine is ~3x faster than the rows are produced), and
  // the tail is the copy of the last 12 %.  More chunks would shorten it
  // further but integrate more pairs twice (one chunk per side of a cut).
  if (out_on_host && stg.on && stg.nnz_cap > (1LL << 25) && row_hi - row_lo >= 64 * pl->P.nc) {
    const long long nc = pl->P.nc, n = row_hi - row_lo;
    const long long c1 = row_lo + (long long)(0.62 * (double)n) / nc * nc, c2 = row_lo + (long long)(0.88 * (double)n) / nc * nc;
    todo.clear();
    todo.push_back({c2, row_hi, false});  // (popped last)
    todo.push_back({c1, c2, false});
    todo.push_back({row_lo, c1, false});
  }
  while (!todo.empty()) {
    auto rg = todo.back();
    todo.pop_back();
    bool split = false, an_fb = false;
    std::vector<long long> cuts;
    const bool first_attempt = st.n_batches == 0 && st.n_replans == 0;
    const size_t npieces = pieces.size();
    // (the budget does not shrink with the finished pieces: taking them off
    // cut config 4's shards into 9 batches instead of 6 and cost 8 % -- more
    // cuts, more pairs integrated twice; emit_pieces hands memory back instead)
    rc = run_batch(pl, rg.first, rg.second, budget, first_attempt, pieces, &st, ctr, tm, dctr.as<unsigned long long>(),
                   derr.as<unsigned long long>(), &split, &cuts, rg.plain, &an_fb);
    if (rc) break;
    if (out_on_host && pieces.size() > npieces) {
      rc = stg.stage(pieces.back());
      if (rc) break;
    }
    if (an_fb) {
      todo.push_back({rg.first, rg.second, true});
      st.n_replans += 1;
      continue;
    }
    if (split) {
      if (cuts.empty()) cuts.push_back(rg.first + (rg.second - rg.first) / (2 * pl->P.nc) * pl->P.nc);
      if (cuts.front() <= rg.first) cuts.front() = rg.first + pl->P.nc;
      // ranges pushed in reverse so they run in row order
      long long hi = rg.second;
      for (size_t c = cuts.size(); c-- > 0;) {
        if (cuts[c] > rg.first && cuts[c] < hi) {
          todo.push_back({cuts[c], hi, rg.plain});
          hi = cuts[c];
        }
      }
      todo.push_back({rg.first, hi, rg.plain});
      st.n_replans += 1;
    }
  }
  if (rc) {
    for (auto& p : pieces) { cudaFreeAsync(p.indptr, s); cudaFreeAsync(p.indices, s); cudaFreeAsync(p.data, s); }
    return rc;
  }
  TRACE("batches done");
  pl->last_batches.clear();
  for (const Csr& c : pieces) {
    pl->last_batches.push_back(c.row_lo);
    pl->last_batches.push_back(c.row_hi);
  }
  // pieces are produced in ascending row order (ranges are popped low-first)
  long long nnz = 0;
  rc = emit_pieces(pl, ds, pieces, row_lo, row_hi, out_on_host, alloc, user, e2, &nnz, stg, ha, sig);
  if (rc) return rc;
  unsigned long long hc[K_NCOUNTERS], herr, herr2[2];
  CK(cudaMemcpyAsync(hc, dctr.p, sizeof hc, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(herr2, derr.p, sizeof herr2, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  herr = herr2[0];
  st.err_self_k = herr2[1] == ~0ull ? -1 : (long long)herr2[1];
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  st.ms_prep = ms;
  CK(cudaEventElapsedTime(&ms, e0, e2));
  st.ms_total = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  st.ms_candidates = tm.cand;
  st.ms_full = tm.full;
  st.ms_partial = tm.part;
  st.ms_singular = tm.sing;
  st.ms_merge = tm.merge;
  st.ms_merge_stage_r = tm.stage_r;
  st.ms_integrate_kernels = tm.full + tm.part + tm.sing;
  st.nnz = nnz;
  st.inner_evals = (long long)(hc[K_EVAL_M0] + hc[K_EVAL_M1] + hc[K_EVAL_M2]);
  st.outer_nonempty = (long long)(hc[K_OUT_M0] + hc[K_OUT_M1] + hc[K_OUT_M2]);
  st.sing_points = (long long)(hc[K_SPTS3] + hc[K_SPTS4] + hc[K_SPTS5] + hc[K_SPTS6]);
  TRACE("assemble end");
  if (g_trace)
    fprintf(stderr, "[nlg] clipped: %llu sub-triangles, %llu rounds, %llu chunks -> lane use %.3f\n",
            hc[K_DBG_SUBTRI], hc[K_DBG_ROUNDS], hc[K_DBG_CHUNKS],
            hc[K_DBG_ROUNDS] ? (double)hc[K_DBG_SUBTRI] / (32.0 * kClipWarps * hc[K_DBG_ROUNDS]) : 0.0);
  if (g_trace)
    fprintf(stderr, "[nlg] clipped items: %llu, far %llu, inside %llu, nonempty %llu\n", hc[K_DBG_ITEMS],
            hc[K_DBG_FAR], hc[K_DBG_INSIDE], hc[K_DBG_NONEMPTY]);
  st.alg_flops_full = alg_flops(pl->P, hc, 0);
  st.alg_flops_partial = alg_flops(pl->P, hc, 1);
  st.alg_flops_singular = alg_flops(pl->P, hc, 2);
  st.alg_flops = st.alg_flops_full + st.alg_flops_partial + st.alg_flops_singular;
  if (herr != ~0ull) {
    st.err_k = (long long)(herr / (unsigned long long)pl->P.K);
    st.err_l = (long long)(herr % (unsigned long long)pl->P.K);
  }
  if (stats) *stats = st;
  if (herr != ~0ull) {
    set_err("nonfinite local contribution for element pair (%lld, %lld)", st.err_k, st.err_l);
    return NLG_ERR_NUMERICAL;
  }
  return NLG_OK;
}

nlg_status nlg_assemble(nlg_plan* pl, int64_t row_lo, int64_t row_hi, int32_t out_on_host,
                        nlg_alloc_fn alloc, void* user, int64_t budget, nlg_stats* stats) {
  return assemble_impl(pl, row_lo, row_hi, out_on_host, alloc, user, budget, stats, nullptr);
}

nlg_status nlg_assemble_pinned(nlg_plan* pl, int64_t row_lo, int64_t row_hi, nlg_alloc_fn block_alloc, void* user,
                               int64_t budget, nlg_stats* stats, nlg_host_csr* out) {
  if (!out) { set_err("null result"); return NLG_ERR_CONFIG; }
  memset(out, 0, sizeof *out);
  HostArena ha;
  ha.alloc = block_alloc;
  ha.user = user;
  ha.out = out;
  return assemble_impl(pl, row_lo, row_hi, 1, block_alloc, user, budget, stats, &ha);
}

void* nlg_pinned_alloc(int64_t nbytes) {
  void* p = nullptr;
  if (nbytes <= 0 || cudaHostAlloc(&p, (size_t)nbytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
void nlg_pinned_free(void* p) {
  if (p) cudaFreeHost(p);
}

static nlg_status ensure_active(nlg_plan* pl) {
  if (pl->nact >= 0) return NLG_OK;
  cudaStream_t s = pl->stream;
  const int K = pl->P.K;
  DevBuf flag, idx, n;
  CK(flag.alloc(sizeof(int) * K, s));
  CK(idx.alloc(sizeof(int) * K, s));
  CK(n.alloc(sizeof(int), s));
  CK(cudaMallocAsync(&pl->act, sizeof(int) * std::max(K, 1), s));
  k_active<<<grid_for(K, 256), 256, 0, s>>>(pl->P, flag.as<int>());
  LAUNCHED();
  k_iota<<<grid_for(K, 256), 256, 0, s>>>(idx.as<int>(), K);
  LAUNCHED();
  size_t tb = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, tb, idx.as<int>(), flag.as<int>(), pl->act, n.as<int>(), K, s));
  DevBuf tmp;
  CK(tmp.alloc(tb, s));
  CK(cub::DeviceSelect::Flagged(tmp.p, tb, idx.as<int>(), flag.as<int>(), pl->act, n.as<int>(), K, s));
  int h = 0;
  CK(cudaMemcpyAsync(&h, n.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  TRACE("sync 2445");
  pl->nact = h;
  pl->nbase = (int)(pl->P.J / pl->P.nc);
  return NLG_OK;
}

nlg_status nlg_load_points(nlg_plan* pl, int32_t out_on_host, nlg_alloc_fn alloc, void* user, int64_t* n_points) {
  if (!pl || !alloc) { set_err("null plan or allocator"); return NLG_ERR_CONFIG; }
  CK(cudaSetDevice(pl->device));
  nlg_status rc = ensure_active(pl);
  if (rc) return rc;
  cudaStream_t s = pl->stream;
  const long long np = (long long)pl->nact * 7;
  *n_points = np;
  double* out = (double*)alloc(user, sizeof(double) * 2 * std::max(np, 1LL), 4);
  if (!out) { set_err("output allocation failed"); return NLG_ERR_CUDA; }
  DevBuf tmp;
  double* dst = out;
  if (out_on_host) {
    CK(tmp.alloc(sizeof(double) * 2 * std::max(np, 1LL), s));
    dst = tmp.as<double>();
  }
  if (np) {
    k_load_points<<<grid_for(np, 256), 256, 0, s>>>(pl->P, pl->act, pl->nact, dst);
    LAUNCHED();
  }
  if (out_on_host && np) CK(cudaMemcpyAsync(out, dst, sizeof(double) * 2 * np, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  TRACE("sync 2472");
  (void)out_on_host;
  return NLG_OK;
}

static nlg_status load_impl(nlg_plan* pl, const double* fx, int fx_on_device, int fconst, int32_t out_on_host,
                            nlg_alloc_fn alloc, void* user) {
  if (!pl || !alloc) { set_err("null plan or allocator"); return NLG_ERR_CONFIG; }
  CK(cudaSetDevice(pl->device));
  nlg_status rc = ensure_active(pl);
  if (rc) return rc;
  cudaStream_t s = pl->stream;
  const int nact = pl->nact, nc = pl->P.nc;
  const long long J = pl->P.J;
  DevBuf dfx, contrib, key, item, key2, item2, start, bdev;
  const long long nfx = fconst ? nc : (long long)nact * 7 * nc;
  const double* dptr = fx;
  if (!fx_on_device) {
    CK(dfx.alloc(sizeof(double) * std::max(nfx, 1LL), s));
    CK(cudaMemcpyAsync(dfx.p, fx, sizeof(double) * nfx, cudaMemcpyHostToDevice, s));
    dptr = dfx.as<double>();
  }
  CK(contrib.alloc(sizeof(double) * std::max(3LL * nact * nc, 1LL), s));
  if (nact) {
    k_load_contrib<<<grid_for(nact, 128), 128, 0, s>>>(pl->P, pl->act, nact, dptr, fconst, contrib.as<double>());
    LAUNCHED();
  }
  const long long ni = 3LL * nact;
  CK(key.alloc(sizeof(unsigned) * std::max(ni, 1LL), s));
  CK(item.alloc(sizeof(int) * std::max(ni, 1LL), s));
  CK(key2.alloc(sizeof(unsigned) * std::max(ni, 1LL), s));
  CK(item2.alloc(sizeof(int) * std::max(ni, 1LL), s));
  CK(start.alloc(sizeof(int) * (pl->nbase + 1), s));
  if (ni) {
    k_load_inc<<<grid_for(ni, 256), 256, 0, s>>>(pl->P, pl->act, nact, key.as<unsigned>(), item.as<int>());
    LAUNCHED();
    int bits = 1;
    while ((1ll << bits) <= pl->nbase) ++bits;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<unsigned>(), key2.as<unsigned>(), item.as<int>(),
                                       item2.as<int>(), (int)ni, 0, bits, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<unsigned>(), key2.as<unsigned>(), item.as<int>(),
                                       item2.as<int>(), (int)ni, 0, bits, s));
    g_launches += 3;
  }
  k_cell_ranges<<<grid_for(pl->nbase + 1, 256), 256, 0, s>>>(key2.as<unsigned>(), (int)ni, pl->nbase,
                                                             start.as<int>());
  LAUNCHED();
  double* out = (double*)alloc(user, sizeof(double) * std::max(J, 1LL), 3);
  if (!out) { set_err("output allocation failed"); return NLG_ERR_CUDA; }
  double* dst = out;
  if (out_on_host) {
    CK(bdev.alloc(sizeof(double) * J, s));
    dst = bdev.as<double>();
  }
  k_load_gather<<<grid_for(pl->nbase, 256), 256, 0, s>>>(start.as<int>(), item2.as<int>(), contrib.as<double>(),
                                                         pl->nbase, nc, dst);
  LAUNCHED();
  if (out_on_host) CK(cudaMemcpyAsync(out, dst, sizeof(double) * J, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  TRACE("sync 2533");
  return NLG_OK;
}

nlg_status nlg_load(nlg_plan* pl, const double* fx, int32_t fx_on_device, int32_t out_on_host, nlg_alloc_fn alloc,
                    void* user) {
  return load_impl(pl, fx, fx_on_device, 0, out_on_host, alloc, user);
}

nlg_status nlg_load_const(nlg_plan* pl, const double* fconst, int32_t out_on_host, nlg_alloc_fn alloc, void* user) {
  return load_impl(pl, fconst, 0, 1, out_on_host, alloc, user);
}

nlg_status nlg_mass(nlg_plan* pl, int32_t out_on_host, nlg_alloc_fn alloc, void* user) {
  if (!pl || !alloc) { set_err("null plan or allocator"); return NLG_ERR_CONFIG; }
  CK(cudaSetDevice(pl->device));
  if (pl->device < 0 || pl->device >= 64) { set_err("device index out of range"); return NLG_ERR_CONFIG; }
  DeviceScratch& ds = g_scratch[pl->device];
  std::lock_guard<std::mutex> scratch_lock(ds.mu);
  nlg_status rc = ensure_active(pl);
  if (rc) return rc;
  cudaStream_t s = pl->stream;
  Params P = pl->P;
  P.row_lo = 0;
  P.row_hi = P.J;
  const long long coo = (long long)pl->nact * 9 * P.nc;
  if (coo >= (1LL << 31)) { set_err("mesh too large for one mass-matrix batch"); return NLG_ERR_CONFIG; }
  std::vector<Csr> pieces;
  {
    DevBuf keys, vals;
    CK(keys.alloc(sizeof(unsigned long long) * std::max(coo, 1LL), s));
    CK(vals.alloc(sizeof(double) * std::max(coo, 1LL), s));
    if (pl->nact) {
      k_mass<<<grid_for(pl->nact, 256), 256, 0, s>>>(P, pl->act, pl->nact, keys.as<unsigned long long>(),
                                                     vals.as<double>());
      LAUNCHED();
    }
    Csr piece{0, P.J, 0, nullptr, nullptr, nullptr};
    long long nnz = 0, kept = 0;
    const bool narrow = (unsigned long long)P.J * (unsigned long long)P.J < 0xffffffffull;
    rc = narrow ? merge_csr<unsigned>(s, P, keys.as<unsigned long long>(), vals.as<double>(), coo, P.J, piece, nnz,
                                      &kept, false)
                : merge_csr<unsigned long long>(s, P, keys.as<unsigned long long>(), vals.as<double>(), coo, P.J,
                                                piece, nnz, &kept);
    if (rc) return rc;
    piece.nnz = nnz;
    pieces.push_back(piece);
  }
  long long nnz = 0;
  Stager none;
  return emit_pieces(pl, ds, pieces, 0, P.J, out_on_host, alloc, user, nullptr, &nnz, none, nullptr, 0ull);
}

nlg_status nlg_row_work(nlg_plan* pl, int64_t* work) {
  if (!pl || !work) { set_err("null plan or output"); return NLG_ERR_CONFIG; }
  CK(cudaSetDevice(pl->device));
  DeviceScratch& ds = g_scratch[pl->device];
  std::lock_guard<std::mutex> scratch_lock(ds.mu);
  pl->arena_used = 0;
  cudaStream_t s = pl->stream;
  pl->prepped = false;
  if (nlg_status rc = prep(pl)) return rc;
  Params P = pl->P;
  P.row_lo = 0;
  P.row_hi = P.J;
  const int K = P.K;
  const long long nb = P.J / P.nc;
  DevBuf needA, rflag, roots, nroots, inR, idx, cnt, wk;
  CK(needA.alloc(K, s));
  CK(rflag.alloc(sizeof(int) * K, s));
  CK(roots.alloc(sizeof(int) * K, s));
  CK(nroots.alloc(sizeof(int), s));
  CK(inR.alloc(sizeof(int) * K, s));
  CK(idx.alloc(sizeof(int) * K, s));
  CK(wk.alloc(sizeof(unsigned long long) * std::max(nb, 1LL), s));
  CK(cudaMemsetAsync(wk.p, 0, sizeof(unsigned long long) * std::max(nb, 1LL), s));
  int nR = 0;
  if (K) {
    k_mark_a<<<grid_for(K, 256), 256, 0, s>>>(P, needA.as<unsigned char>());
    LAUNCHED();
    k_mark_roots<<<grid_for(K, 256), 256, 0, s>>>(P, needA.as<unsigned char>(), nullptr, rflag.as<int>());
    LAUNCHED();
    k_iota<<<grid_for(K, 256), 256, 0, s>>>(idx.as<int>(), K);
    LAUNCHED();
    size_t tb = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, tb, idx.as<int>(), rflag.as<int>(), roots.as<int>(), nroots.as<int>(), K, s));
    DevBuf tmp;
    CK(tmp.alloc(tb, s));
    CK(cub::DeviceSelect::Flagged(tmp.p, tb, idx.as<int>(), rflag.as<int>(), roots.as<int>(), nroots.as<int>(), K, s));
    g_launches += 1;
    CK(cudaMemcpyAsync(&nR, nroots.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  if (nR) {
    CK(cudaMemsetAsync(inR.p, 0xff, sizeof(int) * K, s));
    k_rank<<<grid_for(nR, 256), 256, 0, s>>>(roots.as<int>(), nR, inR.as<int>());
    LAUNCHED();
    CK(cnt.alloc(sizeof(int) * (size_t)kCnt * nR, s));
    const int cand_blocks = (int)std::min<long long>((nR * 32LL + 255) / 256, 148 * 16);
    k_candidates<false><<<std::max(cand_blocks, 1), 256, 0, s>>>(P, pl->G, roots.as<int>(), nR,
                                                                 needA.as<unsigned char>(), inR.as<int>(),
                                                                 cnt.as<int>(), nullptr, nullptr, nullptr, nullptr,
                                                                 nullptr, 1);
    LAUNCHED();
    k_base_work<<<grid_for(nR, 256), 256, 0, s>>>(P, roots.as<int>(), nR, cnt.as<int>(),
                                                  wk.as<unsigned long long>());
    LAUNCHED();
  }
  CK(cudaMemcpyAsync(work, wk.p, sizeof(unsigned long long) * nb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return NLG_OK;
}

nlg_status nlg_local_blocks(nlg_plan* pl, int64_t n, const int64_t* pairs, double* blocks, int64_t* dofs,
                            int32_t* dims) {
  if (!pl || n < 0 || (n && (!pairs || !blocks || !dofs || !dims))) { set_err("null plan or output"); return NLG_ERR_CONFIG; }
  const Params& P0 = pl->P;
  const int K = P0.K, NC = P0.nc, NB = 6 * NC;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t k = pairs[2 * i], l = pairs[2 * i + 1];
    if (k < 0 || k >= K || l < 0 || l >= K) {
      set_err("element pair (%lld, %lld) out of range for %d elements", (long long)k, (long long)l, K);
      return NLG_ERR_CONFIG;
    }
  }
  if (!n) return NLG_OK;
  CK(cudaSetDevice(pl->device));
  DeviceScratch& ds = g_scratch[pl->device];
  std::lock_guard<std::mutex> scratch_lock(ds.mu);
  cudaStream_t s = pl->stream;
  Params P = P0;
  P.row_lo = 0;
  P.row_hi = P.J;
  P.narrow = 0;
  std::vector<int4> el(K), dof(K);
  CK(cudaMemcpyAsync(el.data(), pl->elem, sizeof(int4) * K, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(dof.data(), pl->dofs, sizeof(int4) * K, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // the regularizing path's touching pairs use the tensor rules (k_singular,
  // per family), every other pair the retriangulated sweep (k_pair_local)
  std::vector<int2> loc, sing[3];
  std::vector<int64_t> iloc, ising[3];
  for (int64_t i = 0; i < n; ++i) {
    const int k = (int)pairs[2 * i], l = (int)pairs[2 * i + 1];
    const int ea[3] = {el[k].x, el[k].y, el[k].z}, eb[3] = {el[l].x, el[l].y, el[l].z};
    int ns = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) ns += ea[a] == eb[b];
    const bool touching = k == l || ns > 0;
    if (touching && P.path == 2) {
      const int f = k == l ? 0 : (ns == 2 ? 1 : 2);
      sing[f].push_back(make_int2(k, l));
      ising[f].push_back(i);
    } else {
      loc.push_back(make_int2(k, l));
      iloc.push_back(i);
    }
  }
  DevBuf dpairs, dout, derr, dctr, dvmax, demax;
  CK(derr.alloc(2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(derr.p, 0xff, 2 * sizeof(unsigned long long), s));
  CK(dctr.alloc(sizeof(unsigned long long) * K_NCOUNTERS, s));
  CK(cudaMemsetAsync(dctr.p, 0, sizeof(unsigned long long) * K_NCOUNTERS, s));
  CK(dvmax.alloc(sizeof(unsigned long long), s));
  CK(demax.alloc(sizeof(unsigned long long) * K, s));
  CK(cudaMemsetAsync(demax.p, 0, sizeof(unsigned long long) * K, s));
  std::vector<double> hloc((size_t)loc.size() * NB * NB);
  if (!loc.empty()) {
    CK(dpairs.alloc(sizeof(int2) * loc.size(), s));
    CK(dout.alloc(sizeof(double) * hloc.size(), s));
    CK(cudaMemcpyAsync(dpairs.p, loc.data(), sizeof(int2) * loc.size(), cudaMemcpyHostToDevice, s));
    const unsigned g = (unsigned)std::min<size_t>(loc.size(), 1 << 16);
    auto* e = derr.as<unsigned long long>();
    switch (P.kid) {
      case 0: k_pair_local<0><<<g, 32, 0, s>>>(P, dpairs.as<int2>(), (int)loc.size(), dout.as<double>(), e); break;
      case 1: k_pair_local<1><<<g, 32, 0, s>>>(P, dpairs.as<int2>(), (int)loc.size(), dout.as<double>(), e); break;
      case 2: k_pair_local<2><<<g, 32, 0, s>>>(P, dpairs.as<int2>(), (int)loc.size(), dout.as<double>(), e); break;
      default: k_pair_local<3><<<g, 32, 0, s>>>(P, dpairs.as<int2>(), (int)loc.size(), dout.as<double>(), e); break;
    }
    LAUNCHED();
    CK(cudaMemcpyAsync(hloc.data(), dout.p, sizeof(double) * hloc.size(), cudaMemcpyDeviceToHost, s));
  }
  const long long slots = 36LL * NC * NC;
  const long long nsg = (long long)(sing[0].size() + sing[1].size() + sing[2].size());
  std::vector<unsigned long long> hkey((size_t)nsg * slots);
  std::vector<double> hval((size_t)nsg * slots);
  if (nsg) {
    DevBuf dls, dkeys, dvals;
    CK(dls.alloc(sizeof(int2) * nsg, s));
    CK(dkeys.alloc(sizeof(unsigned long long) * nsg * slots, s));
    CK(dvals.alloc(sizeof(double) * nsg * slots, s));
    int2* ls[3];
    long long nS[3], o = 0;
    for (int f = 0; f < 3; ++f) {
      ls[f] = dls.as<int2>() + o;
      nS[f] = (long long)sing[f].size();
      if (nS[f]) CK(cudaMemcpyAsync(ls[f], sing[f].data(), sizeof(int2) * nS[f], cudaMemcpyHostToDevice, s));
      o += nS[f];
    }
    nlg_status rc;
    auto* kk = dkeys.as<unsigned long long>();
    auto* ctr = dctr.as<unsigned long long>();
    auto* e = derr.as<unsigned long long>();
    auto* vm = dvmax.as<unsigned long long>();
    auto* em = demax.as<unsigned long long>();
    switch (P.kid) {
      case 0: rc = run_singular<0>(pl, P, ls, nS, kk, dvals.as<double>(), 0, ctr, e, vm, em); break;
      case 1: rc = run_singular<1>(pl, P, ls, nS, kk, dvals.as<double>(), 0, ctr, e, vm, em); break;
      case 2: rc = run_singular<2>(pl, P, ls, nS, kk, dvals.as<double>(), 0, ctr, e, vm, em); break;
      default: rc = run_singular<3>(pl, P, ls, nS, kk, dvals.as<double>(), 0, ctr, e, vm, em); break;
    }
    if (rc) return rc;
    CK(cudaMemcpyAsync(hkey.data(), dkeys.p, sizeof(unsigned long long) * hkey.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hval.data(), dvals.p, sizeof(double) * hval.size(), cudaMemcpyDeviceToHost, s));
  }
  unsigned long long herr[2];
  CK(cudaMemcpyAsync(herr, derr.p, sizeof herr, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // outputs: each pair's block row-major with stride NB, its dofs, its size
  for (size_t j = 0; j < loc.size(); ++j) {
    const int64_t i = iloc[j];
    memcpy(blocks + i * NB * NB, hloc.data() + j * NB * NB, sizeof(double) * NB * NB);
    const int4 dk = dof[loc[j].x], dl = dof[loc[j].y];
    const int da[3] = {dk.x, dk.y, dk.z}, db[3] = {dl.x, dl.y, dl.z};
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < NC; ++c) {
        dofs[i * NB + a * NC + c] = (int64_t)NC * da[a] + c;
        dofs[i * NB + 3 * NC + a * NC + c] = (int64_t)NC * db[a] + c;
      }
    dims[i] = NB;
  }
  long long o = 0;
  for (int f = 0; f < 3; ++f)
    for (size_t j = 0; j < sing[f].size(); ++j, ++o) {
      const int64_t i = ising[f][j];
      const bool same = sing[f][j].x == sing[f][j].y;
      double* B = blocks + i * NB * NB;
      for (int e = 0; e < NB * NB; ++e) B[e] = 0.0;
      int dim = 0;
      for (long long q = 0; q < slots; ++q) {
        const unsigned long long key = hkey[o * slots + q];
        if (key == kSentinel) continue;
        const int ii = (int)(q / (6 * NC)), jj = (int)(q % (6 * NC));
        // (the engine's unordered-pair block is twice one ordered pair's)
        B[ii * NB + jj] = same ? hval[o * slots + q] : 0.5 * hval[o * slots + q];
        dofs[i * NB + ii] = (int64_t)(key / (unsigned long long)P.J);
        dim = std::max(dim, ii + 1);
      }
      dims[i] = dim;
    }
  if (herr[0] != ~0ull) {
    set_err("nonfinite local contribution for element pair (%lld, %lld)", (long long)(herr[0] / (unsigned long long)K),
            (long long)(herr[0] % (unsigned long long)K));
    return NLG_ERR_NUMERICAL;
  }
  return NLG_OK;
}

nlg_status nlg_fp64_peak(int32_t device, double* tflops) {
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* d;
  CK(cudaMalloc(&d, 8));
  const int bs = 512, grid = sms * 4, iters = 2048;
  k_dfma_peak<<<grid, bs>>>(d, 8, 0.999999, 1e-7);
  LAUNCHED();
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    k_dfma_peak<<<grid, bs>>>(d, iters, 0.999999, 1e-7);
    LAUNCHED();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  *tflops = 2.0 * 8 * 16 * (double)iters * grid * bs / (best * 1e-3) / 1e12;
  return NLG_OK;
}

}  // extern "C"

// ===================================================================== CG solve
// Conjugate gradients on a device CSR (the free block of a Dirichlet split,
// SURVEY.md 8f): warp-per-row SpMV and two-stage dot products with fixed
// reduction trees, so the iteration is run-to-run deterministic.  Scalars
// stay on the device; the host reads the residual every few iterations.
namespace {

constexpr int kCgThreads = 256, kCgBlocks = 592;  // 4 blocks per SM

__global__ void k_cg_spmv(long long n, const long long* __restrict__ ptr, const int* __restrict__ idx,
                          const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double acc = 0.0;
  for (long long j = ptr[row] + lane; j < ptr[row + 1]; j += 32) acc = fma(__ldg(&val[j]), __ldg(&x[idx[j]]), acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = acc;
}

// per-block partial of dot(a, b) (fixed striding and tree)
__global__ void k_cg_dot_part(long long n, const double* __restrict__ a, const double* __restrict__ b, double* part) {
  __shared__ double red[kCgThreads / 32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc = fma(a[i], b[i], acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kCgThreads / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// sum of the partials in block order -> *out (one warp)
__global__ void k_cg_dot_fin(const double* __restrict__ part, int np, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 32) acc += part[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) *out = acc;
}

// s[0] = rr, s[1] = pAp, s[2] = rr_new
__global__ void k_cg_update_xr(long long n, const double* __restrict__ s, const double* __restrict__ p,
                               const double* __restrict__ ap, double* x, double* r) {
  const double alpha = s[1] != 0.0 ? s[0] / s[1] : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    r[i] = fma(-alpha, ap[i], r[i]);
  }
}

__global__ void k_cg_update_p(long long n, double* s, const double* __restrict__ r, double* p) {
  const double beta = s[0] != 0.0 ? s[2] / s[0] : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], r[i]);
}

__global__ void k_cg_shift(double* s) { s[0] = s[2]; }

__global__ void k_cg_residual(long long n, const double* __restrict__ b, const double* __restrict__ ax, double* r,
                              double* p) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = b[i] - ax[i];
    r[i] = v;
    p[i] = v;
  }
}

}  // namespace

extern "C" nlg_status nlg_cg(int32_t device, int64_t n, const int64_t* indptr, const int32_t* indices,
                             const double* data, const double* b, double* x, double rtol, int32_t maxit,
                             int32_t* iters, double* relres) {
  if (n < 0 || !indptr || !indices || !data || !b || !x || !iters || !relres) {
    set_err("nlg_cg: bad arguments");
    return NLG_ERR_CONFIG;
  }
  CK(cudaSetDevice(device));
  *iters = 0;
  *relres = 0.0;
  if (n == 0) return NLG_OK;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
  } sg{st};
  const long long* ptr = (const long long*)indptr;
  double *r, *p, *ap, *part, *sc;
  CK(cudaMallocAsync(&r, sizeof(double) * n, st));
  CK(cudaMallocAsync(&p, sizeof(double) * n, st));
  CK(cudaMallocAsync(&ap, sizeof(double) * n, st));
  CK(cudaMallocAsync(&part, sizeof(double) * kCgBlocks, st));
  CK(cudaMallocAsync(&sc, sizeof(double) * 4, st));
  struct FreeGuard {
    cudaStream_t s;
    void* q[5];
    ~FreeGuard() { for (void* v : q) cudaFreeAsync(v, s); }
  } fg{st, {r, p, ap, part, sc}};
  const unsigned gs = (unsigned)std::min<long long>((n * 32 + 255) / 256, 1LL << 30);
  auto dot = [&](const double* a, const double* c, double* out) {
    k_cg_dot_part<<<kCgBlocks, kCgThreads, 0, st>>>(n, a, c, part);
    k_cg_dot_fin<<<1, 32, 0, st>>>(part, kCgBlocks, out);
    g_launches += 2;
  };
  // r = b - A x, p = r
  k_cg_spmv<<<gs, 256, 0, st>>>(n, ptr, indices, data, x, ap);
  LAUNCHED();
  k_cg_residual<<<kCgBlocks, kCgThreads, 0, st>>>(n, b, ap, r, p);
  LAUNCHED();
  dot(b, b, sc + 3);
  dot(r, r, sc + 0);
  double h[4];
  CK(cudaMemcpyAsync(h, sc, sizeof h, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double bn = sqrt(h[3]) > 0.0 ? sqrt(h[3]) : 1.0;
  double rr = h[0];
  int it = 0;
  const int check = 8;
  while (it < maxit && sqrt(rr) > rtol * bn) {
    for (int k = 0; k < check && it < maxit; ++k, ++it) {
      k_cg_spmv<<<gs, 256, 0, st>>>(n, ptr, indices, data, p, ap);
      dot(p, ap, sc + 1);
      k_cg_update_xr<<<kCgBlocks, kCgThreads, 0, st>>>(n, sc, p, ap, x, r);
      dot(r, r, sc + 2);
      k_cg_update_p<<<kCgBlocks, kCgThreads, 0, st>>>(n, sc, r, p);
      k_cg_shift<<<1, 1, 0, st>>>(sc);
      g_launches += 4;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rr = h[0];
    if (!std::isfinite(rr)) { set_err("nlg_cg: residual is not finite"); return NLG_ERR_NUMERICAL; }
  }
  *iters = it;
  *relres = sqrt(rr) / bn;
  return NLG_OK;
}
