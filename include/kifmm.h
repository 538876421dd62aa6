/*
 * kifmm.h — C-ABI of the B200-native SVD-compressed KIFMM matvec
 * (arXiv 1211.2517, "A SVD accelerated kernel-independent fast multipole method
 * and its application to BEM"; "P:n" = /root/reference/PAPER.md line n).
 *
 * The library computes one FP64 matrix-vector product with the 3D Laplace
 * single-layer kernel G(x, y) = 1 / (4 pi |x - y|) — or, with source
 * normals, the double-layer kernel dG/dn(y):
 *
 *     p_i = sum_{j : x_j != x_i} G(x_i, x_j) q_j            (eq_eval)
 *
 * by the kernel-independent FMM whose translation operators are
 * compressed with the M2L SVD basis, on one B200 or
 * partitioned over several (one process per GPU, NCCL over NVLink).
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
#define FMM_ENCCL (-5)    /* NCCL unavailable or an NCCL call failed (multi-GPU plans) */

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
  const double* sigma;  /* n singular values of K_fat, descending (needed by stage 2; may be NULL) */
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
                         fmm_export_phase can return both; 0 (default): one fused pass.
                         Single-GPU plans only. */
  /* Multi-GPU.  nranks > 1 partitions the matvec: every rank passes
     the SAME N points (replicated setup), rank r owns a contiguous Morton range of
     leaves (fmm_owned_range) chosen by a prefix sum of estimated work, and ghost
     multipoles / ghost densities are exchanged inside every matvec.
       nccl_id != NULL: a 128-byte ncclUniqueId shared by all ranks (fmm_nccl_unique_id
                        on one rank, broadcast by the caller); one process per GPU,
                        fmm_setup_ex is collective.
       nccl_id == NULL: a loopback rank: all nranks plans live in one process (any
                        devices) and run together through fmm_matvec_group (tests). */
  int nranks;         /* default 1 */
  int rank;           /* 0 <= rank < nranks */
  const void* nccl_id;
  int leaf_ops;       /* per-leaf S2M and L2T operators built at setup (owned points x kp
                         doubles each): a matvec then streams them from HBM instead of
                         evaluating n kernel values per point and operator.  -1 (default): each
                         while max(16 GB, 10% of the device) stays free; 0 off; 1 on. */
  double m2l_c2;      /* stage 2 of the M2L compression: each core C_o is replaced
                         by its SVD truncated at eps2 ||K_fat||_2 with eps2 = C2 eps1 / k
                         (eq-vareps2; eps1 = sigma_{k+1} / sigma_1, the stage-1 truncation) and
                         M2L runs as two skinny GEMMs (U^_o (V^_o q)).  0 (default) = off. */
  const double* normals; /* device, N x 3 FP64, caller order, or NULL.  Non-NULL: double-layer
                         sources (eq-doubles2m): every evaluation whose source is an
                         input point (near field S2T, the S2M check potential, the X-list check
                         potential) uses dG/dn(y) = (x - y).n(y) / (4 pi |x - y|^3); the
                         translations between surfaces stay single layer.  Copied at setup. */
  const double* triangles; /* device, N x 9 FP64 (3 vertices), caller order, or NULL.  Non-NULL:
                         BEM collocation: source j is the flat triangle j with
                         piecewise-constant density, the points passed to setup are the
                         triangles' centroids (collocation points), and every evaluation whose
                         source is an element integrates G over it (analytic self term, 6-point
                         rule, subdivision: reading R-BEM).  Use d = C_d / sqrt(s);
                         the overhang of elements beyond their leaves is reported in
                         fmm_info.bem_extrusion, setup fails (FMM_EINVAL) if an element reaches
                         its leaf's upward check surface.  The near-field matrix is built at setup
                         (FMM_ENOMEM if it does not fit).  Single GPU. */
  const char* operator_file; /* host path or NULL (ignored when `tables` is set).  The operator
                         tables' versioned binary file (tables_io.cpp): loaded if it exists —
                         FMM_ECONFIG if it was built for another (p, k, d, pinv_rcond), is
                         corrupt or of another version — else computed and written there. */
  int near_mode;      /* near-field (P2P) kernel: -1 (default) = 1; 1 = mutual leaf pairs (k_near:
                         each pair of owned leaves once for both sides, G symmetric);
                         0 = one-sided per target leaf (k_eval); 2 = warp-pair symmetric
                         (k_p2p_sym; single layer only, else 0).  Same result to rounding. */
  int overlap;        /* near field beside the far field on a second plan stream: -1 (default) =
                         3 up to 8M owned points, else 0; 0 = serialised; 3 = k_near (or the
                         BEM near-field SpMV) forked at the densities (NCCL plans: after the
                         ghost exchange); 1 / 2 = the one-sided near field forked at the
                         densities / beside a high-priority M2L stream.  Profiled and
                         split-phase plans: 0. */
} fmm_options;

typedef struct {
  int64_t N;
  int p, n, k, kp;            /* k = k_eff; kp = k padded to a multiple of 8 */
  int nboxes, nleaves, nlevels;
  int64_t nU, nV, nW, nX;     /* list sizes (pairs of boxes) */
  int64_t n_s2m, n_xnd, n_l2t, n_wnd;  /* evaluation work items */
  int64_t m2l_tiles, m2l_pairs;  /* M2L tiles of the sibling-class kernel; V pairs it applies */
  int64_t launches;           /* kernels of this library launched by the last fmm_matvec */
  double r0, lo_root[3];
  double precompute_ms, tree_ms, lists_ms, schedule_ms;
  float phase_ms[9];          /* last profiled matvec (ms): density, S2M, M2M, exchange (straddlers + ghost
                                 multipoles), M2L, X, L2L, eval (L2T + W + near field), output */
  int nranks, rank;
  int64_t own_lo, own_hi;     /* owned sorted points */
  int64_t n_straddle;         /* boxes whose multipole is allreduced */
  int64_t ghost_q_recv, ghost_q_send;  /* ghost multipole rows per matvec */
  int64_t ghost_d_recv, ghost_d_send;  /* ghost densities per matvec (owned mode) */
  int64_t nV_local;           /* V pairs this rank's M2L applies (= nV on one rank) */
  int64_t leaf_op_bytes;      /* device bytes of the per-leaf operators (0: not used) */
  double m2l_flops;           /* algorithmic M2L flops of one matvec on this rank:
                                 sum over V pairs of 2 k^2 (dense cores) or 4 k r_o (stage 2) */
  double m2l_eps2;            /* stage-2 threshold relative to ||K_fat||_2 (0: off) */
  double m2l_rank_mean;       /* mean stage-2 rank over the 316 offsets (k when off) */
  int64_t bem_near_bytes;     /* BEM near-field matrix bytes (0: point sources) */
  double bem_extrusion;       /* BEM: largest element overhang beyond a leaf, in leaf halfwidths
                                 (the surface condition of P:389-411 asks for < d) */
  int64_t near_mutual_leaves; /* target leaves evaluating symmetric (mutual) leaf pairs */
  int64_t near_mutual_pairs;  /* unordered near-field point pairs evaluated once for both sides */
  int64_t near_sym_pairs;     /* leaf pairs of the warp-pair symmetric kernel (KIFMM_SYM=2) */
  double m2l_exec_flops;      /* M2L flops the kernels execute: 2 k^2 per sibling-class column
                                 step (absent children included) + the offset-major pairs */
  int64_t near_pairs;         /* directed near-field point pairs (U + direct W/X, r = 0 pairs
                                 included) delivered by k_near per matvec: own points m^2, 2 per
                                 mutual pair, 1 per one-sided pair (mutual mode; 0 otherwise) */
  double near_ms;             /* last profiled matvec: the near-field (P2P) launches alone, ms
                                 (CUDA events on the launching stream; -1 when not profiled) */
  int64_t overlap;            /* the overlap mode the plan runs (fmm_options.overlap after defaults) */
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

/* Partitioned matvec in OWNED mode (nranks > 1; also valid on one rank, where the
 * owned range is everything):
 *   density_owned    device [own_hi - own_lo], densities of the owned points in
 *                    sorted (Morton) order: density_owned[i] = q[perm[own_lo + i]]
 *                    (perm from fmm_export_tree)
 *   potential_owned  device [own_hi - own_lo], same order; overwritten
 * Ghost densities and multipoles are exchanged over NCCL on `stream`.  fmm_matvec
 * on a multi-GPU plan is the REPLICATED mode: full caller-order density in, full
 * caller-order potential out on every rank (the owned ranges are allgathered). */
int fmm_matvec_owned(fmm_plan* plan, const double* density_owned, double* potential_owned, void* stream);

/* Same with HOST buffers (copies inside; returns after the stream synchronised). */
int fmm_matvec_owned_host(fmm_plan* plan, const double* h_density_owned, double* h_potential_owned, void* stream);

/* `count` matvecs with HOST buffers (pinned host memory for the copies to overlap):
 * h_density[i] -> h_potential[i], each [N] in caller order (the _owned_ form: [own_hi -
 * own_lo] in sorted order, as fmm_matvec_owned).  Same results as `count` calls of
 * fmm_matvec_host, but pipelined: the density of matvec i + 1 is copied in (one copy
 * stream) and the potential of matvec i - 1 copied out (another) while matvec i computes
 * on `stream`, through two device staging pairs allocated on first use (2 N doubles).
 * Buffers may repeat (the same density for every i).  Returns after all copies have
 * landed.  FMM_EINVAL for a null buffer or count < 0. */
int fmm_matvec_host_batch(fmm_plan* plan, const double* const* h_density, double* const* h_potential, int count,
                          void* stream);
int fmm_matvec_owned_host_batch(fmm_plan* plan, const double* const* h_density_owned,
                                double* const* h_potential_owned, int count, void* stream);

/* Solve A x = rhs with restarted GMRES(restart) (the paper's solver,
 * P:528, tolerance 1e-6 at P:539), A = the plan's matvec (single-GPU plans; with BEM
 * triangles, the collocation operator).  Device vectors in caller order; x holds the
 * initial guess on entry and the solution on return.  Stops when ||rhs - A x|| <=
 * tol ||rhs|| or after maxit iterations.  Arnoldi by classical Gram-Schmidt applied twice
 * on the device; Givens rotations on the host.  Outputs: *iters iterations (= matvecs
 * in the Krylov loop), *relres the final true relative residual, *t_matvec_ms (may be
 * NULL) the mean matvec time.  Synchronises `stream` before returning. */
int fmm_gmres(fmm_plan* plan, const double* rhs, double* x, int restart, int maxit, double tol, void* stream, int* iters,
              double* relres, double* t_matvec_ms);

/* Owned sorted-point range [*begin, *end) of the plan's rank. */
int fmm_owned_range(const fmm_plan* plan, int64_t* begin, int64_t* end);

/* 128-byte NCCL unique id for fmm_options.nccl_id. */
int fmm_nccl_unique_id(void* id128);

/* Loopback group: one matvec of the nplans plans of one partition (plans[r] built
 * with nranks = nplans, rank = r, nccl_id = NULL), run stage by stage with the
 * ghost exchanges done as device copies between the plans, all on `stream`.
 *   owned = 1: densities[r] / potentials[r] as in fmm_matvec_owned for rank r
 *   owned = 0: densities[r] / potentials[r] as in fmm_matvec (full, caller order)
 * The exchanges are the same buffers and lists the NCCL transport sends. */
int fmm_matvec_group(fmm_plan* const* plans, int nplans, const double* const* densities, double* const* potentials,
                     int owned, void* stream);

/* Host-only partition (no GPU): the partition rank `rank` of `nranks` derives from a
 * tree and its lists in the fmm_export_tree / fmm_export_lists formats
 * (U: nU x 2, V, W, X: n x 3 int32).  n = surface points, k = rank (work model). */
typedef struct fmm_partition fmm_partition;
int fmm_partition_host(int nboxes, const int32_t* level, const int32_t* parent, const int32_t* pbeg,
                       const int32_t* pend, const uint8_t* leaf, int64_t nU, const int32_t* U, int64_t nV,
                       const int32_t* V, int64_t nW, const int32_t* W, int64_t nX, const int32_t* X, int n, int k,
                       int nranks, int rank, fmm_partition** out);
/* Arrays of a partition (owned by it), what =
 *   0 bnd[nranks+1] (sorted-point boundaries)   1 inD[nboxes] (0/1: point range meets the owned range)
 *   2 straddling boxes                           3 full[nboxes] (0/1: point range inside the owned range)
 *   4 q send boxes, 5 q send offsets[nranks+1]   6 q recv boxes, 7 q recv offsets
 *   8 density send points, 9 offsets             10 density recv points, 11 offsets  */
int fmm_partition_get(const fmm_partition* part, int what, int64_t* count, const int32_t** data);
void fmm_partition_free(fmm_partition* part);
/* The partition of a plan (owned by the plan; valid until fmm_free). */
const fmm_partition* fmm_plan_partition(const fmm_plan* plan);

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
/* The tables' versioned binary file (see fmm_options.operator_file): write (FMM_EINVAL if
 * the path cannot be written) / read (FMM_ECONFIG: missing, corrupt or another version). */
int fmm_tables_save(const fmm_tables* t, const char* path);
int fmm_tables_load(const char* path, fmm_tables** out);

const char* fmm_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* KIFMM_B200_H */
