// Internal structures of the B200 KIFMM library (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace kifmm {

constexpr int kNumOffsets = 316;  // M2L offsets per level

struct HostTables {
  int p = 0, n = 0, k = 0;
  double d = 0.1, rcond = 1e-10;
  std::vector<double> sigma;   // singular values of K_fat (n)
  std::vector<double> surf;    // unit surface grid (n x 3)
  std::vector<double> U;       // n x k
  std::vector<double> C;       // 316 x k x k
  std::vector<double> S;       // k x n
  std::vector<double> T;       // n x k
  std::vector<double> M;       // 8 x k x k
  std::vector<double> L;       // 8 x k x k
  // stage 2: per-offset low-rank factors of C, empty when off
  double eps2 = 0;
  int rmax = 0;
  std::vector<int> ranks;                 // 316
  std::vector<std::vector<double>> Uh, Vh;  // k x r_o, r_o x k
};

int build_tables(int p, int k, double d, double rcond, HostTables* out);
int save_tables(const HostTables& H, int k_req, const std::string& path);
int load_tables(const std::string& path, HostTables* H, int* k_req);  // 1: no file
int build_stage2(HostTables& H, double C2);

// One launch of the grouped gather-GEMM-scatter kernel: Y[tgt] (+)= scale * Op * X[src].
struct GemmTile {
  int op;        // operator index within the op array
  int begin;     // first pair
  int count;     // pairs in this tile (<= tile width)
  int pad;
  double scale;  // level factor applied to the product
};

struct GemmLaunch {
  int ntiles = 0;
  GemmTile* d_tiles = nullptr;
  int2* d_pairs = nullptr;  // (src row, tgt row)
  int npairs = 0;
};

// Sibling-grouped M2L (k_m2l_sib): tiles (class, first column, count, 0); columns
// (target, src[8]); classes (nvalid, b[8], offset id[8]) for class = delta * 8 + a.
struct SibLaunch {
  int ntiles = 0, ncols = 0;
  int4* d_tiles = nullptr;   // sorted by decreasing work (operators per column)
  int* d_cols = nullptr;
  int* d_classes = nullptr;
  int* d_counter = nullptr;  // dynamic tile scheduler (reset before every launch)
};

// Stage-2 low-rank M2L factors on the device (k_m2l_lr), zero padded: Uh[316][kp][rp],
// Vh[316][rp][kp] with rp = max rank rounded up to 16; rank[316].
struct LowRank {
  bool on = false;
  int rp = 0;
  double* d_Uh = nullptr;
  double* d_Vh = nullptr;
  int* d_rank = nullptr;
};

struct Tree {
  int64_t N = 0;
  int nboxes = 0, nleaves = 0, nlevels = 0;
  double lo_root[3] = {0, 0, 0}, r0 = 1, scale = 1;
  std::vector<int> level_begin;       // nlevels + 1
  // device
  uint64_t* d_key = nullptr;          // per box: Morton prefix at its level
  int* d_level = nullptr;
  int* d_parent = nullptr;
  int* d_pbeg = nullptr;
  int* d_pend = nullptr;
  int* d_child_begin = nullptr;       // first child (children contiguous), -1 for leaves
  int* d_nchild = nullptr;
  uint8_t* d_leaf = nullptr;
  double4* d_geom = nullptr;          // (cx, cy, cz, r)
  int32_t* d_perm = nullptr;          // sorted -> caller
  int32_t* d_iperm = nullptr;         // caller -> sorted
  double4* d_pts = nullptr;           // sorted points (x, y, z, q)
  // host mirrors (setup-time copies)
  std::vector<uint64_t> key;
  std::vector<int> level, parent, pbeg, pend, child_begin, nchild;
  std::vector<uint8_t> leaf;
};

struct Lists {
  // canonical device lists
  int nU = 0, nV = 0, nW = 0, nX = 0;
  int2* d_U = nullptr;     // (tgt, src) by (tgt, src)
  int4* d_V = nullptr;     // (tgt, src, off, 0) by (off, tgt)
  int4* d_W = nullptr;     // (tgt, src, direct, 0) by (tgt, src)
  int4* d_X = nullptr;     // (tgt, src, direct, 0) by (tgt, src)
};

// Host-side view of a tree and its canonical lists (partition input).  Lists are
// strided int32 records: U (tgt, src), V (tgt, src, offset id), W / X (tgt, src, direct).
struct PartitionInput {
  int nboxes = 0;
  const int* level = nullptr;
  const int* parent = nullptr;
  const int* pbeg = nullptr;
  const int* pend = nullptr;
  const uint8_t* leaf = nullptr;
  int64_t nU = 0, nV = 0, nW = 0, nX = 0;
  const int* U = nullptr; int ustride = 2;
  const int* V = nullptr; int vstride = 3;
  const int* W = nullptr; int wstride = 3;
  const int* X = nullptr; int xstride = 3;
  int n = 0, k = 0;
};

// Morton-range partition of one matvec over nranks (partition.cpp).
struct DistPlan {
  int nranks = 1, rank = 0;
  std::vector<int> bnd;              // nranks + 1 sorted-point boundaries
  int own_lo = 0, own_hi = 0;        // owned sorted points [own_lo, own_hi)
  std::vector<double> work;          // estimated work per rank
  std::vector<uint8_t> inD, full;    // per box: range meets / lies in the owned range
  std::vector<int> straddle;         // boxes spanning >= 2 ranks (all ranks agree)
  std::vector<int> q_send, q_send_off, q_recv, q_recv_off;  // ghost q^' boxes, CSR by peer
  std::vector<int> d_send, d_send_off, d_recv, d_recv_off;  // ghost density points, CSR by peer
};

int build_partition(const PartitionInput& in, int nranks, int rank, DistPlan* out);

// Device side of one ghost exchange (rows of `row` doubles).
struct Exchange {
  int row = 0;
  std::vector<int> send_off, recv_off;  // per peer, in rows
  int nsend = 0, nrecv = 0;
  int* d_send_idx = nullptr;
  int* d_recv_idx = nullptr;
  double* d_send = nullptr;
  double* d_recv = nullptr;
};

// bulk-copy streamed leaf-operator GEMV (stream.cu): items (first row, rows, first weight /
// output point, output box) and per-CTA item ranges
struct StreamPlan {
  int4* d_items = nullptr;
  int* d_cta = nullptr;
  int nitems = 0, ncta = 0;
  int64_t rows = 0;
};

struct Plan {
  int device = 0;
  int p = 0, k = 0, kp = 0, n = 0, leaf_size = 0, wx = 0;
  double d = 0.1, rcond = 1e-10;
  Tree tree;
  Lists lists;
  HostTables tables;   // host copy (unpadded)
  // device operator tables, zero-padded to kp
  double* d_C = nullptr;    // 316 x kp x kp
  double* d_M = nullptr;    // 8 x kp x kp
  double* d_L = nullptr;    // 8 x kp x kp
  double* d_S = nullptr;    // kp x n    (S')
  double* d_Ut = nullptr;   // kp x n    (U^T)
  double* d_T = nullptr;    // n x kp    (T')
  double* d_Ue = nullptr;   // n x kp    (U)
  double* d_surf = nullptr; // n x 3 unit surface grid
  LowRank lr;               // stage-2 M2L (fmm_options.m2l_c2 > 0)
  double4* d_nrm = nullptr; // sorted source normals: double-layer sources, else NULL
  // BEM elements: sorted triangles (3 x double4 each), near-field block matrix
  bool bem = false;
  double4* d_tri = nullptr;
  double* d_bem_A = nullptr;
  int64_t* d_bem_moff = nullptr;  // matrix offset per near segment
  int64_t bem_near_bytes = 0;
  double bem_extrusion = 0;       // max over leaves of (vertex distance / r) - 1 (surface condition)
  double m2l_flops = 0;     // algorithmic M2L flops per matvec on this rank
  // work buffers
  double* d_qhat = nullptr;     // nboxes x kp (level-normalised q^')
  double* d_lhat = nullptr;     // nboxes x kp
  double* d_chk_s2m = nullptr;  // n_s2m x n  check potentials of leaves (S2M stage 1)
  double* d_chk_x = nullptr;    // n_xnd x n  check potentials of non-direct X pairs
  double* d_eqd_l2t = nullptr;  // n_l2t x n  downward equivalent densities
  double* d_eqd_w = nullptr;    // n_wnd x n  upward equivalent densities of W sources
  double* d_pot_near = nullptr; // N (sorted)
  double* d_pot_far = nullptr;  // N (sorted)
  double* d_io = nullptr;       // N staging for host-buffer matvec
  // batched host-buffer matvecs (fmm_matvec_host_batch): a second staging pair, copy
  // streams and per-buffer events, created on first use
  double* d_io2 = nullptr;
  cudaStream_t stream_h2d = nullptr, stream_d2h = nullptr;
  cudaEvent_t ev_io[7] = {};  // in[2], done[2], out[2], start
  // evaluation work lists (k_eval items: (box, out row, 0, 0); CSR of segments (kind, a, b, len))
  int np = 0;                                  // n rounded up to a multiple of 8
  int n_tleaf = 0; int4* d_tleaf_items = nullptr;
  int n_sym = 0; int2* d_sym = nullptr;   // symmetric near-field leaf pairs (both owned), k_p2p_sym
  int sym_opt = -1;                        // -1 / 1 mutual segments (k_evalm), 2 warp pairs (k_p2p_sym), 0 off
  // near field by k_near (near.cu; mutual leaf pairs, sym_opt -1 / 1): per target leaf
  // (first point, m, chunk begin, chunk end), grouped by pass shape; chunks (first
  // source slot, n | nchk << 10 | ml << 20, mh, 0); source slots (point indices)
  bool nr_on = false;
  int nr_table = 0;                        // k_near shape table: 0 single layer, 3 double layer
  int n_tleaf_mut = 0;                     // target leaves with mutual segments
  int64_t n_mut_pairs = 0;                 // unordered point pairs of the mutual segments
  int64_t n_near_pairs = 0;               // directed near-field point pairs (k_near mode)
  double m2l_exec_flops = 0;               // M2L flops executed incl. absent sibling children
  int4* d_nr_items = nullptr;
  int4* d_nr_chunks = nullptr;
  int* d_nr_src = nullptr;
  int* d_nr_counters = nullptr;            // work counters per k_near launch (2 per group)
  int nr_spare = 0;                        // overlap mode 3: CTA slots per SM left to the kernels beside k_near
  double nr_split = 1.0;                   // overlap mode 3: share of each group's units launched at the fork (rest after M2L)
  int64_t nr_src_bytes = 0;
  std::vector<int3> nr_groups;             // (pass shape, first item, count) per k_near launch
  int* d_near_off = nullptr; int4* d_near_seg = nullptr; int n_near_seg = 0;
  int* d_far_off = nullptr;  int4* d_far_seg = nullptr;  int n_far_seg = 0;
  int n_fitems = 0; int4* d_fitems = nullptr;      // target leaves with far segments (compact far pass)
  int* d_fitem_off = nullptr; int4* d_fitem_seg = nullptr;
  int* d_all_off = nullptr;  int4* d_all_seg = nullptr;  // near + far segments (fused pass)
  bool split_phases = false;  // separate near / far passes (phase exports)
  // per-leaf operators (leaf-op mode): S2M  q^'_B = S_B q_B  with S_B = S' G(UC_B, x_B)
  // (point-major rows of kp), L2T  pot_B = T_B l^_B  with T_B = r_l G(x_B, DE_B) T'
  // (kp-major within a leaf block); both indexed by sorted point - own_lo
  int leaf_ops_opt = -1;      // -1 auto, 0 off, 1 on
  bool leaf_s2m = false, leaf_l2t = false;  // which of the two operators are used
  // X-list operators (same budget): per non-direct X pair (target B, source leaf A) the
  // k x m_A matrix U^T G_src(DC_B, sources of A), point-major rows of kp at x_moff[row]
  bool leaf_x = false;
  double* d_x_mat = nullptr;
  int64_t* d_x_moff = nullptr;
  int n_xt = 0;
  int4* d_xt_items = nullptr;   // (target box, first row, end row, 0)
  double* d_s2m_mat = nullptr;
  double* d_l2t_mat = nullptr;
  // the upward leaf-operator GEMVs (S2M, X) streamed by bulk copies (stream.cu): one rank,
  // S2M (and X, if any) operators built
  bool stream_ok = false;
  StreamPlan sw_s2m, sw_x;
  double* d_q_sorted = nullptr;  // N + 2 densities in sorted order (the streamed weights)
  int64_t leaf_op_bytes = 0;
  int n_s2m = 0; int4* d_s2m_items = nullptr; int* d_s2m_off = nullptr; int4* d_s2m_seg = nullptr;
  int n_xnd = 0; int4* d_x_items = nullptr;   int* d_x_off = nullptr;   int4* d_x_seg = nullptr;
  int n_l2t = 0, n_wnd = 0;
  std::vector<void*> allocations;              // everything cudaMalloc'ed for the plan
  // dense-algebra launches
  GemmLaunch g_s2m, g_x, g_l2t, g_w;
  SibLaunch g_m2l_sib;        // M2L columns whose sources are complete on this rank (all, one rank)
  SibLaunch g_m2l_sib_ghost;  // the rest: ghost / straddling sources (multi-rank plans)
  bool m2l_local_done = false;  // this matvec already ran the local M2L tiles (overlapped exchange)
  double sib_min_density = 0.5;   // sibling groups at least this full go to k_m2l_sib
  std::vector<GemmLaunch> g_m2m;   // per child level (descending)
  std::vector<GemmLaunch> g_l2l;   // per parent level (ascending)
  // timing of the last matvec (ms per phase), filled when profiling is on
  std::vector<float> phase_ms;
  cudaStream_t stream = nullptr;
  int overlap = 0;                    // near field on stream_near: 1 from the upward pass, 2 beside M2L
  cudaStream_t stream_near = nullptr;
  cudaStream_t stream_m2l = nullptr;  // overlap 2: high-priority stream of the M2L kernel
  cudaEvent_t ev_m2l = nullptr;
  cudaEvent_t ev_near[2] = {nullptr, nullptr};  // profiled plans: around the near-field launches
  bool near_timed = false;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // k_near's second launch stream (near_launch alternates the pass-shape launches)
  cudaStream_t stream_nr2 = nullptr;
  cudaEvent_t ev_nr_fork = nullptr, ev_nr_join = nullptr;
  // NCCL plans: the straddler allreduce and the ghost exchange on their own stream, beside
  // the M2L of the local sources (matvec_device)
  cudaStream_t stream_comm = nullptr;
  cudaEvent_t ev_up = nullptr, ev_comm = nullptr;
  std::vector<cudaEvent_t> ev_phase;
  std::vector<cudaEvent_t> ev_trace;  // KIFMM_TRACE=1 diagnostics (kernels.cu)
  bool profile = false;
  bool profiled = false;
  int launches = 0;       // kernels of this library launched by the last matvec
  int launch_acc = 0;     // running count across the stages of the current matvec
  // ---- multi-GPU; nranks == 1: everything owned, exchanges empty
  DistPlan dist;
  Exchange xq, xd;                 // ghost q^' rows / ghost densities
  int n_straddle = 0;
  int64_t nV_local = 0;            // V pairs with a target in D (this rank's M2L work)
  int* d_straddle = nullptr;       // straddling boxes
  double* d_straddle_buf = nullptr;  // n_straddle x kp partial multipoles
  void* nccl_comm = nullptr;       // ncclComm_t (NULL: single GPU or loopback group)
};

// matvec stages; between them the transport runs the exchanges:
//   0 densities (+ pack ghost densities)            -> exchange xd (owned mode)
//   1 unpack densities, S2M, M2M, pack straddlers   -> allreduce straddlers
//   2 unpack straddlers, pack ghost q^'             -> exchange xq
//   3 unpack ghost q^', M2L, X, L2L, L2T, W, P2P, owned output
//                                                   -> allgather potentials (replicated mode)
//   4 potential in caller order (replicated mode)
int build_leaf_ops(Plan& P, cudaStream_t st);
int build_x_ops(Plan& P, cudaStream_t st);
int sort_normals(Plan& P, const double* d_normals, cudaStream_t st);
int bem_sort_triangles(Plan& P, const double* d_tri_caller, cudaStream_t st);
int bem_check_enclosure(Plan& P, cudaStream_t st);
int bem_build_near(Plan& P, const std::vector<int4>& blocks, cudaStream_t st);
int bem_near_matvec(const Plan& P, cudaStream_t st);
int gmres_solve(Plan& P, const double* b, double* x, int m, int maxit, double tol, cudaStream_t st, int* iters,
                double* relres, double* t_matvec_ms);
int matvec_stage(Plan& P, int stage, const double* d_density, double* d_pot, bool owned, cudaStream_t st);
constexpr int kNumStages = 5;
int matvec_device(Plan& P, const double* d_density, double* d_pot, bool owned, cudaStream_t st);

// NCCL transport (nccl_transport.cpp; libnccl.so.2 resolved at run time)
int nccl_unique_id(void* id128);
int nccl_comm_init(Plan& P, const void* id128);
void nccl_comm_destroy(Plan& P);
int nccl_exchange(Plan& P, Exchange& X, cudaStream_t st);
int nccl_allreduce_sum(Plan& P, double* buf, size_t count, cudaStream_t st);
int nccl_allgather_ranges(Plan& P, double* buf, cudaStream_t st);

// error helpers (thread-local last error)
void set_error(const std::string& msg);
const char* last_error();

#define KIFMM_CUDA(call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::kifmm::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                         ":" + std::to_string(__LINE__));                                   \
      return -3;                                                                            \
    }                                                                                       \
  } while (0)

// setup stages (tree.cu, lists.cu) and matvec launches (kernels.cu)
int build_tree_device(Plan& P, const double* d_points_caller, cudaStream_t st);
int build_lists_device(Plan& P, cudaStream_t st);
// k_near sources per chunk for a pass shape of cap = TB x MQ targets (static shared memory <= 48 KB)
__host__ __device__ constexpr int near_ch(int cap, bool dl = false) { return dl ? 128 : cap <= 128 ? 512 : 256; }
int near_shape_count(int tab);           // k_near pass shapes of table tab, by capacity
int near_shape_cap(int tab, int shape);  // TB x MQ targets per pass
extern int g_num_sms;
extern int g_launches;
int near_launch(const Plan& P, double* out, cudaStream_t st, int part = 0, int spare = 0);
int build_schedules(Plan& P, cudaStream_t st);
int stream_plan(Plan& P, StreamPlan& S, const std::vector<int4>& items, cudaStream_t st);
int stream_s2m(const Plan& P, cudaStream_t st);
int stream_x(const Plan& P, cudaStream_t st);
int upload_tables(Plan& P);
int kernels_init();
int ggs_tile_width(int M, int K);
int sib_tile_width(int kp, bool lowrank = false);

}  // namespace kifmm
