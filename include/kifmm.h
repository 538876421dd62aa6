/*
 * kifmm.h — C-ABI of the B200-native SVD-compressed KIFMM matvec
 * (arXiv 1211.2517, "A SVD accelerated kernel-independent fast multipole method
 * and its application to BEM"; "P:n" = /root/reference/PAPER.md line n).
 *
 * The library computes one FP64 matrix-vector product with the 3D Laplace
 * single-layer kernel G(x, y) = 1 / (4 pi |x - y|):
 *
 *     p_i = sum_{j : x_j != x_i} G(x_i, x_j) q_j            (eq_eval)
 *
 * by the kernel-independent FMM whose translation operators are
 * compressed with the M2L SVD basis, on one B200.
 *
 * Conventions for every entry point:
 *   - Device pointers are CUDA device memory of the plan's device; host pointers
 *     are ordinary host memory.  Points are N x 3 row-major FP64, caller order.
 *   - Streams are cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Return 0 on success or a negative FMM_E* code; the message of the last
 *     error of the calling thread is fmm_last_error().  No exceptions cross the ABI.
 *   - The caller owns every buffer it passes; a plan owns its internal buffers.
 *   - Pairs with |x_i - x_j| == 0 (self pairs, exact duplicates) contribute 0.
 */
#ifndef KIFMM_B200_H
#define KIFMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMM_OK 0
#define FMM_EINVAL (-1)   /* bad argument: null pointer, N < 1, p < 2, k < 1, leaf_size < 1, d outside [0, 2/3) */
#define FMM_ECONFIG (-2)  /* inconsistent operator tables (p, n, k or d do not match the plan) */
#define FMM_ECUDA (-3)    /* a CUDA runtime call or kernel launch failed */
#define FMM_ENOMEM (-4)   /* host allocation failed */

typedef struct fmm_plan fmm_plan;
typedef struct fmm_tables fmm_tables;

/* Operator tables at unit halfwidth, row-major FP64, host memory.
 *   U  n x k   SVD basis of K_fat (= that of K_thin)
 *   C  316 x k x k   C_delta = U^T K_delta U   (offsets in
 *                    lexicographic order of [-3,3]^3 \ [-1,1]^3, delta = source - target)
 *   S  k x n   S' = U^T pinv(E_u)   (S~ = R^T S)
 *   T  n x k   T' = pinv(E_d) U     (T~ = T U)
 *   M  8 x k x k   M~_o, child octant o = x<<2 | y<<1 | z
 *   L  8 x k x k   L~_o
 * Surfaces: UE, DC at halfwidth (1+d) r, UC, DE at (3-2d) r, sampled
 * at the boundary nodes of a p^3 grid in lexicographic order, n = 6(p-1)^2+2. */
typedef struct {
  int p, n, k;
  double d;
  const double *U, *C, *S, *T, *M, *L;
} fmm_tables_view;

typedef struct {
  int p;              /* surface points per cube edge, >= 2 */
  int k;              /* requested rank; raised to k_eff so no singular-value multiplet is split */
  int leaf_size;      /* s: a box is subdivided iff it holds more than s points */
  double d;           /* surface offset, 0 <= d < 2/3; default 0.1 */
  double pinv_rcond;  /* relative cutoff of the equivalent-density pseudo-inverses; default 1e-10 */
  int wx_direct_max;  /* W/X shortcut: evaluate a W/X pair point-to-point when the source
                         subtree (W) or the target leaf (X) holds <= this many points;
                         -1 = n (default), 0 = never */
  const fmm_tables_view* tables;  /* NULL: compute the tables (host precompute);
                                     else use these (e.g. the oracle's, for parity) */
  int profile;        /* 1: record per-phase CUDA events in fmm_matvec (fmm_info.phase_ms) */
  int split_phases;   /* 1: evaluate the near field and the far field in separate passes so that
                         fmm_export_phase can return both; 0 (default): one fused pass */
} fmm_options;

typedef struct {
  int64_t N;
  int p, n, k, kp;            /* k = k_eff; kp = k padded to a multiple of 8 */
  int nboxes, nleaves, nlevels;
  int64_t nU, nV, nW, nX;     /* list sizes (pairs of boxes) */
  int64_t n_s2m, n_xnd, n_l2t, n_wnd;  /* evaluation work items */
  int64_t m2l_tiles, m2l_pairs;
  int64_t launches;           /* kernels of this library launched by the last fmm_matvec */
  double r0, lo_root[3];
  double precompute_ms, tree_ms, lists_ms, schedule_ms;
  float phase_ms[8];          /* last profiled matvec: near (split only), S2M, M2M, M2L, X, L2L, eval (L2T+W[+near]), output */
} fmm_info_t;

/* fmm_options with every default filled in. */
void fmm_default_options(fmm_options* opt);

/* Build a plan on the current CUDA device (Step 1 Setup): operator
 * tables (host precompute, timed separately), then on the device the Morton
 * octree (radix sort) and the U/V/W/X lists.
 *   points     device, N x 3 FP64, caller order (copied and permuted by the plan)
 *   densities  device [N] or NULL: default density for fmm_matvec(density = NULL)
 * Errors: FMM_EINVAL, FMM_ECONFIG, FMM_ECUDA.  *out is NULL on failure. */
int fmm_setup(const double* points, const double* densities, int64_t N, int p, int k, int leaf_size, fmm_plan** out);
int fmm_setup_ex(const double* points, const double* densities, int64_t N, const fmm_options* opt, void* stream,
                 fmm_plan** out);

/* potential = FMM(density), P:482-518 (upward pass, M2L + downward pass, near field).
 *   density    device [N], caller order, or NULL for the setup densities
 *   potential  device [N], caller order; overwritten
 * Asynchronous on `stream`.  One stream at a time per plan. */
int fmm_matvec(fmm_plan* plan, const double* density, double* potential, void* stream);

/* Same with HOST buffers: copies density in, runs fmm_matvec, copies the
 * potential out, all on `stream`; returns after the stream has synchronised. */
int fmm_matvec_host(fmm_plan* plan, const double* h_density, double* h_potential, void* stream);

/* Release every resource of the plan.  NULL is a no-op. */
void fmm_free(fmm_plan* plan);

int fmm_info(const fmm_plan* plan, fmm_info_t* info);

/* Canonical tree dump (host buffers sized from fmm_info): boxes in level-major,
 * Morton-key order.  level/parent/pbeg/pend/leaf per box, key = Morton prefix at
 * the box level, perm[i] = caller index of sorted point i, geom = lo_root[3], r0, scale. */
int fmm_export_tree(const fmm_plan* plan, int32_t* level, uint64_t* key, int32_t* parent, int32_t* pbeg,
                    int32_t* pend, uint8_t* leaf, int32_t* perm, double* geom);

/* Canonical lists (host buffers): U (tgt, src) by (tgt, src); V (tgt, src, offset id)
 * by (offset id, tgt); W and X (tgt, src, direct) by (tgt, src). */
int fmm_export_lists(const fmm_plan* plan, int32_t* U, int32_t* V, int32_t* W, int32_t* X);

/* Phase arrays of the last matvec (host buffers): which = 0 q^' (nboxes x k, level-
 * normalised multipoles q^/r_l), 1 l^ (nboxes x k), 2 near-field potential (N, sorted
 * order), 3 far-field potential (N, sorted order). */
int fmm_export_phase(const fmm_plan* plan, int which, double* out);

/* Host precompute only (no GPU needed): the tables for (p, k, d, rcond). */
int fmm_tables_build(int p, int k, double d, double rcond, fmm_tables** out);
int fmm_tables_view_get(const fmm_tables* t, fmm_tables_view* view, const double** sigma);
void fmm_tables_free(fmm_tables* t);

const char* fmm_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* KIFMM_B200_H */
