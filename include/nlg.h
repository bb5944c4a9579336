/*
 * nlg.h -- C ABI of the B200 nonlocal stiffness-assembly library (libnlg.so).
 *
 * Drop-in boundary for the reference's assembly hot path
 * (/root/reference/pkg/src/nlfem/assembly.py):
 *
 *   reference seam                                    replaced by
 *   ------------------------------------------------  ----------------------------
 *   bfs_assemble(...)            assembly.py:200-296  nlg_plan_create + nlg_assemble
 *     _element_bounds            assembly.py:130-134    (device bounds kernel)
 *     thread pool over spans     assembly.py:245-283    (device grid hash + kernels)
 *       _engine._chunk           _engine.py:428-600
 *       _engine._visit_pair      _engine.py:188-425
 *       _engine._sweep           _engine.py:46-185
 *       _pyengine.chunk (id 3)   _pyengine.py:327-399
 *     NumericalError on err      assembly.py:285-288    NLG_ERR_NUMERICAL + err pair
 *     _merge_triplets            assembly.py:137-173    (device sort + segmented sum)
 *   assemble_load(...)           assembly.py:451-481  nlg_load_points + nlg_load
 *
 * Conventions
 *   - plain C types only; no exceptions cross the ABI; every call returns an
 *     nlg_status (0 = ok) and nlg_last_error() describes the last failure of
 *     the calling thread;
 *   - problem arrays are HOST or DEVICE pointers (nlg_problem.inputs_on_device)
 *     and are copied/converted into the plan, so the caller keeps ownership;
 *   - outputs (CSR arrays, load vector) are allocated by the caller through
 *     nlg_alloc_fn, on the host or on the device (nlg_assemble's out_on_host),
 *     so e.g. torch's caching allocator or numpy owns them;
 *   - one plan belongs to one device; calls on one plan are serialised by the
 *     caller; plans on different devices may run concurrently;
 *   - a `stream` argument of NULL means the legacy default stream.
 */
#ifndef NLG_H
#define NLG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t nlg_status;
#define NLG_OK 0
#define NLG_ERR_CONFIG 1    /* maps to ConfigurationError */
#define NLG_ERR_NUMERICAL 2 /* maps to NumericalError (nonfinite local contribution) */
#define NLG_ERR_CUDA 3      /* launch / runtime failure, no device, OOM */

#define NLG_ABI_VERSION 5

/* Kernel ids (kernels.py :57-118 built-ins + 3 = nonsymmetric affine). */
#define NLG_KERNEL_FRACTIONAL 0  /* c |x-y|^(-2-2s) */
#define NLG_KERNEL_PERIDYNAMIC 1 /* c (x-y)(x-y)^T/|x-y|^3, nc = 2 */
#define NLG_KERNEL_CONSTANT 2    /* c */
#define NLG_KERNEL_AFFINE 3      /* (1 + p0 x_0) p1, nonsymmetric */

/* Problem description: the arguments _engine._chunk receives
 * (assembly.py:249-264), flattened. */
typedef struct nlg_problem {
  int64_t n_vertices, n_elements;
  const double *vertices;    /* [V][2] */
  const int64_t *elements;   /* [K][3], counterclockwise */
  const int64_t *labels;     /* [K]: 0 inactive, 1 domain, 2 dirichlet */
  const int64_t *outer_mask; /* [K]: 1 = outer element (rows= selection) */
  const int64_t *dof_map;    /* [K][3] scalar dof base of each local hat */
  int64_t n_dofs;            /* J = nc * n_base */
  int32_t nc, is_dg, kernel_id, ball_id, path_touch, symmetric;
  double s, scale, delta, rskip2, drop2, kp0, kp1;
  int32_t n_outer, n_inner; /* must be 7 (QuadratureConfig "7point") */
  const double *op, *ow, *oh, *ip, *iw; /* [n][2], [n], [n][3], [n][2], [n] (host) */
  int32_t n_sing[3];                    /* identical, edge, vertex rule sizes */
  const double *sxs[3], *sys[3], *sw[3], *shx[3], *shy[3]; /* host tables */
  int32_t inputs_on_device;             /* mesh arrays are device pointers */
  /* Label-dependent kernels (KernelSpec.value's label_x, label_y arguments,
   * kernels.py:21-35; _pyengine._pq :38-45 forwards the element labels):
   * value = label_scale[label_x][label_y] x the built-in kernel's value,
   * row-major over labels 0..2.  Must be symmetric. */
  int32_t has_label_scale;
  double label_scale[9];
} nlg_problem;

typedef struct nlg_plan nlg_plan;

/* Allocator for outputs. which: 0 = indptr (int64), 1 = indices (int32),
 * 2 = data (float64), 3 = load vector (float64), 4 = points (float64),
 * 5 = page-locked host block (nlg_assemble_pinned). */
typedef void *(*nlg_alloc_fn)(void *user, int64_t nbytes, int32_t which);

/* Counters and phase times of one nlg_assemble call. */
typedef struct nlg_stats {
  int64_t n_roots;      /* outer elements processed */
  int64_t epi;          /* evaluated element pairs (reference visits passing the reject test) */
  int64_t n_full;       /* non-singular visits whose pair lies fully inside the ball */
  int64_t n_partial;    /* non-singular visits that need clipping */
  int64_t n_singular;   /* touching pairs integrated with the tensor rules */
  int64_t inner_evals;  /* inner-point kernel evaluations on the clipped path */
  int64_t outer_nonempty; /* outer points with a nonempty truncated region (clipped path) */
  int64_t sing_points;  /* singular-rule points evaluated */
  int64_t alg_flops;    /* reference-algorithmic FP64 flops, all phases */
  int64_t alg_flops_full, alg_flops_partial, alg_flops_singular; /* per integration kernel */
  int64_t coo_entries;  /* COO slots emitted by the integration kernels */
  int64_t coo_reduced;  /* entries left after the per-root reduction (globally sorted) */
  int64_t nnz;
  int64_t n_batches;
  int64_t n_replans;    /* batch attempts that did not fit and were re-cut */
  int64_t err_k, err_l; /* first nonfinite pair (lexicographic min), or -1 */
  double ms_prep, ms_candidates, ms_full, ms_partial, ms_singular, ms_merge, ms_total;
  double ms_integrate_kernels; /* full + partial + singular kernel time */
  double ms_merge_stage_r;     /* per-root reduction part of ms_merge */
  int64_t n_row_retries;       /* stage-W rows re-run in a larger table */
  int64_t n_merge_fallbacks;   /* batches merged by stage R + sort instead of stage W */
  int64_t err_self_k;          /* smallest root whose own (k, k) visit was nonfinite, or -1 */
} nlg_stats;

int32_t nlg_abi_version(void);
const char *nlg_last_error(void);
nlg_status nlg_device_count(int32_t *count);

/* Upload/convert the problem onto `device`.  Validates shapes/ids
 * (NLG_ERR_CONFIG) the way bfs_assemble does before its engine runs. */
nlg_status nlg_plan_create(int32_t device, const nlg_problem *problem, void *stream,
                           nlg_plan **out);
void nlg_plan_destroy(nlg_plan *plan);

/* Assemble the CSR rows [row_lo, row_hi) of the J x J stiffness matrix
 * (row_lo = 0, row_hi = J for the whole matrix).  Rows are owner-computed:
 * every outer element that contributes to one of those rows is evaluated
 * and only those rows are emitted, so disjoint row ranges (one per GPU)
 * need no reduction and concatenate into the full matrix.  The CSR
 * (indptr[row_hi-row_lo+1] int64 relative to the block, indices int32
 * column ids, data float64) is written into buffers obtained from `alloc`,
 * on the host when out_on_host != 0.  mem_budget_bytes bounds the scratch
 * of one batch (0 = automatic); larger problems run in row batches. */
nlg_status nlg_assemble(nlg_plan *plan, int64_t row_lo, int64_t row_hi, int32_t out_on_host,
                        nlg_alloc_fn alloc, void *alloc_user, int64_t mem_budget_bytes,
                        nlg_stats *stats);

/* Host CSR without the final host copy.  block_alloc(user, nbytes, 5) must
 * return a PAGE-LOCKED host block of at least nbytes (nlg_pinned_alloc, or
 * the caller's own cudaHostAlloc / registered memory).  The library copies
 * each batch's rows into it while the next batch computes and leaves the CSR
 * there: out->arena is the block used, and indptr (int64[row_hi-row_lo+1]),
 * indices (int32[nnz]), data (float64[nnz]) start at the byte offsets
 * out->off_*.  The callback runs once when the output size is known from an
 * earlier call on the same problem and row range (the size then carries 1/8
 * headroom), else at the end with the exact size; a second time if the
 * first block proved too small -- the caller recycles any block other than
 * out->arena.  Replaces the (data, indices, indptr) arrays the reference
 * builds at assembly.py:294-296 when the consumer is on the host. */
typedef struct nlg_host_csr {
  void *arena;
  int64_t nnz;
  int64_t off_indptr, off_indices, off_data;
} nlg_host_csr;
nlg_status nlg_assemble_pinned(nlg_plan *plan, int64_t row_lo, int64_t row_hi, nlg_alloc_fn block_alloc,
                               void *alloc_user, int64_t mem_budget_bytes, nlg_stats *stats,
                               nlg_host_csr *out);
/* Page-locked host memory for nlg_assemble_pinned (cudaHostAlloc / cudaFreeHost). */
void *nlg_pinned_alloc(int64_t nbytes);
void nlg_pinned_free(void *p);

/* Physical outer quadrature points of the active elements, [K_act][n_outer][2]
 * (assembly.py:463-469), written through alloc (which = 4). */
nlg_status nlg_load_points(nlg_plan *plan, int32_t out_on_host, nlg_alloc_fn alloc, void *user,
                           int64_t *n_points);

/* Load vector b[J] from f evaluated at those points (fx: [K_act*n_outer][nc],
 * host or device per fx_on_device), assembly.py:470-481. */
nlg_status nlg_load(nlg_plan *plan, const double *fx, int32_t fx_on_device, int32_t out_on_host,
                    nlg_alloc_fn alloc, void *user);

/* Load vector for a constant f (one value per component): the whole
 * computation stays on the device. */
nlg_status nlg_load_const(nlg_plan *plan, const double *fconst, int32_t out_on_host,
                          nlg_alloc_fn alloc, void *user);

/* Mass matrix over all dofs, J x J CSR (assembly.py:484-506: the exact P1
 * element mass area * (1 + delta_ab) / 12 on every component of the active
 * elements), written through alloc like nlg_assemble (which = 0, 1, 2). */
nlg_status nlg_mass(nlg_plan *plan, int32_t out_on_host, nlg_alloc_fn alloc, void *alloc_user);

/* Conjugate gradients for A x = b on `device` (all pointers are device
 * memory): A is an n x n CSR (int64 indptr, int32 indices, f64 data), x holds
 * the initial guess and receives the solution.  Stops when
 * ||b - A x|| <= rtol ||b|| or after maxit iterations.  Deterministic
 * (fixed reduction trees).  Used on the free block of a Dirichlet split
 * (SparseSystem.split, assembly.py:102-107). */
nlg_status nlg_cg(int32_t device, int64_t n, const int64_t *indptr, const int32_t *indices, const double *data,
                  const double *b, double *x, double rtol, int32_t maxit, int32_t *iters, double *relres);

/* Local stiffness blocks of n ORDERED element pairs (the reference's
 * local_contribution, assembly.py:327-448): pairs[2i], pairs[2i+1] = (k, l).
 * Block i is written row-major with stride 6 nc into blocks[i][6nc][6nc]; its
 * size (dims[i] x dims[i]) and its global dofs (dofs[i][0..dims[i])) say
 * which part is used:
 *   - the regularizing path's touching pairs: the union-basis block of one
 *     ordered pair (U nc, U = 3 / 4 / 5, or 6 for DG), from the tensor rules;
 *   - every other pair: the 4-term block over (k's 3 nc dofs, l's 3 nc dofs),
 *     the inner element retriangulated against each outer point's ball.
 * Host arrays.  NLG_ERR_CONFIG for a pair out of range, NLG_ERR_NUMERICAL
 * for a nonfinite block. */
nlg_status nlg_local_blocks(nlg_plan *plan, int64_t n, const int64_t *pairs, double *blocks, int64_t *dofs,
                            int32_t *dims);

/* Work estimate per dof base for balancing row shards across GPUs: for
 * every dof base, the summed EPI (visits passing the reject test) of the
 * outer elements incident to it, from the device's candidate count pass;
 * written to the host array work[n_dofs / nc].  Deterministic (integer sums). */
nlg_status nlg_row_work(nlg_plan *plan, int64_t *work);

/* DFMA throughput microbenchmark on `device` (the FP64 roofline denominator). */
nlg_status nlg_fp64_peak(int32_t device, double *tflops);

/* Row ranges of the batches the last nlg_assemble on this plan ran, in row
 * order: writes min(n, cap) pairs (lo, hi) into ranges[2 * cap] and returns
 * n (the batch count), or -1 for a null plan.  Diagnostics / tests: parity at
 * the batch cuts, where each batch re-evaluates its halo roots. */
int64_t nlg_last_batches(const nlg_plan *plan, int64_t *ranges, int64_t cap);

/* Number of kernels this library launched on the calling process so far. */
int64_t nlg_launch_count(void);

/* nlcsr text tokens (host, replaces the token loops of write_nlcsr,
 * assembly.py:509-516): v[0..n) as space-separated tokens, Python int() for
 * the integer arrays and repr(float) for the values, into buf (no trailing
 * separator).  Returns the length, or -1 if cap is too small (33 bytes per
 * token always suffice).  threads <= 0: all hardware threads. */
int64_t nlg_format_f64(const double *v, int64_t n, char *buf, int64_t cap, int32_t threads);
int64_t nlg_format_i64(const int64_t *v, int64_t n, char *buf, int64_t cap, int32_t threads);
int64_t nlg_format_i32(const int32_t *v, int64_t n, char *buf, int64_t cap, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* NLG_H */
