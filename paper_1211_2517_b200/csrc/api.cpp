// C-ABI of the B200 KIFMM library (include/kifmm.h).
#include "../../include/kifmm.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmm_internal.h"

struct fmm_partition {
  kifmm::DistPlan own;                 // host-built partitions
  const kifmm::DistPlan* D = nullptr;  // -> own, or a plan's partition
  std::vector<int32_t> inD32, full32;
  void view(const kifmm::DistPlan* d) {
    D = d;
    inD32.assign(d->inD.begin(), d->inD.end());
    full32.assign(d->full.begin(), d->full.end());
  }
};

struct fmm_plan {
  kifmm::Plan P;
  fmm_partition part;
  double* d_default_density = nullptr;
  double precompute_ms = 0, tree_ms = 0, lists_ms = 0, schedule_ms = 0;
};

struct fmm_tables {
  kifmm::HostTables H;
  int k_req = 0;  // the requested k (H.k is k_eff)
};

namespace kifmm {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
}  // namespace kifmm

using kifmm::set_error;

namespace {

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void free_plan_memory(fmm_plan* h) {
  kifmm::Plan& P = h->P;
  for (void* p : P.allocations) cudaFree(p);
  P.allocations.clear();
  kifmm::Tree& T = P.tree;
  void* tp[] = {T.d_key, T.d_level, T.d_parent, T.d_pbeg, T.d_pend, T.d_child_begin, T.d_nchild, T.d_leaf, T.d_geom,
                T.d_perm, T.d_iperm, T.d_pts, P.lists.d_U, P.lists.d_V, P.lists.d_W, P.lists.d_X, h->d_default_density};
  for (void* p : tp)
    if (p) cudaFree(p);
  for (auto e : P.ev_phase) cudaEventDestroy(e);
  for (auto e : P.ev_trace) cudaEventDestroy(e);
  P.ev_trace.clear();
  P.ev_phase.clear();
  if (P.ev_fork) cudaEventDestroy(P.ev_fork);
  if (P.ev_join) cudaEventDestroy(P.ev_join);
  if (P.stream_near) cudaStreamDestroy(P.stream_near);
  if (P.stream_m2l) cudaStreamDestroy(P.stream_m2l);
  if (P.ev_m2l) cudaEventDestroy(P.ev_m2l);
  if (P.stream_nr2) cudaStreamDestroy(P.stream_nr2);
  if (P.ev_nr_fork) cudaEventDestroy(P.ev_nr_fork);
  if (P.ev_nr_join) cudaEventDestroy(P.ev_nr_join);
  P.stream_nr2 = nullptr;
  P.ev_nr_fork = P.ev_nr_join = nullptr;
  if (P.stream_comm) cudaStreamDestroy(P.stream_comm);
  if (P.ev_up) cudaEventDestroy(P.ev_up);
  if (P.ev_comm) cudaEventDestroy(P.ev_comm);
  P.stream_comm = nullptr;
  P.ev_up = P.ev_comm = nullptr;
  for (auto& e : P.ev_near) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  for (auto& e : P.ev_io) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  if (P.stream_h2d) cudaStreamDestroy(P.stream_h2d);
  if (P.stream_d2h) cudaStreamDestroy(P.stream_d2h);
  P.stream_h2d = P.stream_d2h = nullptr;
  if (P.d_io2) cudaFree(P.d_io2);
  P.d_io2 = nullptr;
  P.ev_fork = P.ev_join = P.ev_m2l = nullptr;
  P.stream_near = P.stream_m2l = nullptr;
  kifmm::nccl_comm_destroy(P);
}

constexpr int kPhases = 9;

// No C++ exception crosses the C ABI: every int-returning entry point runs its body
// through guard(), which maps std::bad_alloc to FMM_ENOMEM and any other exception to
// FMM_EINVAL, with the message in fmm_last_error().
template <class F>
int guard(const char* what, F&& body) {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    set_error(std::string(what) + ": out of host memory");
    return FMM_ENOMEM;
  } catch (const std::exception& e) {
    set_error(std::string(what) + ": " + e.what());
    return FMM_EINVAL;
  } catch (...) {
    set_error(std::string(what) + ": unknown exception");
    return FMM_EINVAL;
  }
}

}  // namespace

extern "C" {

void fmm_default_options(fmm_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->p = 6;
  o->k = 60;
  o->leaf_size = 128;
  o->d = 0.1;
  o->pinv_rcond = 1e-10;
  o->wx_direct_max = -1;
  o->tables = nullptr;
  o->profile = 0;
  o->split_phases = 0;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->leaf_ops = -1;
  o->m2l_c2 = 0.0;
  o->normals = nullptr;
  o->triangles = nullptr;
  o->operator_file = nullptr;
  o->near_mode = -1;
  o->overlap = -1;
}

const char* fmm_last_error(void) { return kifmm::last_error(); }

int fmm_tables_build(int p, int k, double d, double rcond, fmm_tables** out) {
  return guard("fmm_tables_build", [&]() -> int {
    if (!out || p < 2 || k < 1 || !(d >= 0 && d < 2.0 / 3.0) || !(rcond >= 0)) {
      set_error("fmm_tables_build: invalid argument");
      return FMM_EINVAL;
    }
    *out = nullptr;
    fmm_tables* t = new (std::nothrow) fmm_tables();
    if (!t) { set_error("fmm_tables_build: out of host memory"); return FMM_ENOMEM; }
    int rc = kifmm::build_tables(p, k, d, rcond, &t->H);
    if (rc) { delete t; return rc; }
    t->k_req = k;
    *out = t;
    return FMM_OK;
  });
}

int fmm_tables_save(const fmm_tables* t, const char* path) {
  return guard("fmm_tables_save", [&]() -> int {
    if (!t || !path) { set_error("fmm_tables_save: null argument"); return FMM_EINVAL; }
    return kifmm::save_tables(t->H, t->k_req, path) ? FMM_EINVAL : FMM_OK;
  });
}

int fmm_tables_load(const char* path, fmm_tables** out) {
  return guard("fmm_tables_load", [&]() -> int {
    if (!path || !out) { set_error("fmm_tables_load: null argument"); return FMM_EINVAL; }
    *out = nullptr;
    fmm_tables* t = new (std::nothrow) fmm_tables();
    if (!t) { set_error("fmm_tables_load: out of host memory"); return FMM_ENOMEM; }
    const int rc = kifmm::load_tables(path, &t->H, &t->k_req);
    if (rc) {
      delete t;
      if (rc == 1) set_error(std::string("fmm_tables_load: no such file ") + path);
      return FMM_ECONFIG;
    }
    *out = t;
    return FMM_OK;
  });
}

int fmm_tables_view_get(const fmm_tables* t, fmm_tables_view* v, const double** sigma) {
  return guard("fmm_tables_view_get", [&]() -> int {
    if (!t || !v) { set_error("fmm_tables_view_get: null argument"); return FMM_EINVAL; }
    const kifmm::HostTables& H = t->H;
    v->p = H.p; v->n = H.n; v->k = H.k; v->d = H.d;
    v->U = H.U.data(); v->C = H.C.data(); v->S = H.S.data(); v->T = H.T.data(); v->M = H.M.data(); v->L = H.L.data();
    v->sigma = H.sigma.data();
    if (sigma) *sigma = H.sigma.data();
    return FMM_OK;
  });
}

void fmm_tables_free(fmm_tables* t) { delete t; }

int fmm_setup(const double* points, const double* densities, int64_t N, int p, int k, int leaf_size, fmm_plan** out) {
  return guard("fmm_setup", [&]() -> int {
    fmm_options o;
    fmm_default_options(&o);
    o.p = p; o.k = k; o.leaf_size = leaf_size;
    return fmm_setup_ex(points, densities, N, &o, nullptr, out);
  });
}

int fmm_setup_ex(const double* points, const double* densities, int64_t N, const fmm_options* opt, void* stream,
                 fmm_plan** out) {
  fmm_plan* pending = nullptr;  // freed here if the body throws after allocating it
  const int rc_ = guard("fmm_setup_ex", [&]() -> int {
    if (!out) { set_error("fmm_setup: out is NULL"); return FMM_EINVAL; }
    *out = nullptr;
    if (!opt || !points || N < 1 || N > INT32_MAX || opt->p < 2 || opt->k < 1 || opt->leaf_size < 1 ||
        !(opt->d >= 0 && opt->d < 2.0 / 3.0) || !(opt->pinv_rcond >= 0)) {
      set_error("fmm_setup: invalid argument (points, N in [1, 2^31), p >= 2, k >= 1, leaf_size >= 1, 0 <= d < 2/3)");
      return FMM_EINVAL;
    }
    if (opt->nranks < 1 || opt->rank < 0 || opt->rank >= opt->nranks || (opt->nranks > 1 && opt->split_phases)) {
      set_error("fmm_setup: invalid nranks / rank (0 <= rank < nranks; split_phases needs nranks == 1)");
      return FMM_EINVAL;
    }
    const int n_expect = 6 * (opt->p - 1) * (opt->p - 1) + 2;
    if (opt->p * 1 > 0 && n_expect > 296) { set_error("fmm_setup: p > 8 is not supported (n <= 296)"); return FMM_EINVAL; }
    fmm_plan* h = new (std::nothrow) fmm_plan();
    if (!h) { set_error("fmm_setup: out of host memory"); return FMM_ENOMEM; }
    pending = h;
    kifmm::Plan& P = h->P;
    cudaStream_t st = (cudaStream_t)stream;
    P.stream = st;
    cudaGetDevice(&P.device);
    P.leaf_size = opt->leaf_size;
    P.d = opt->d;
    P.rcond = opt->pinv_rcond;
    P.profile = opt->profile != 0;
    P.split_phases = opt->split_phases != 0;
    P.leaf_ops_opt = opt->leaf_ops;
    if (opt->near_mode < -1 || opt->near_mode > 2 || opt->overlap < -1 || opt->overlap > 3) {
      set_error("fmm_setup: near_mode must be in [-1, 2] and overlap in [-1, 3]");
      return FMM_EINVAL;
    }
    P.sym_opt = opt->near_mode;
    P.dist.nranks = opt->nranks;
    P.dist.rank = opt->rank;
    auto fail = [&](int rc) { free_plan_memory(h); delete h; pending = nullptr; return rc; };
    if (kifmm::kernels_init()) return fail(FMM_ECUDA);
    // ---- operator tables
    auto t0 = std::chrono::steady_clock::now();
    if (opt->tables) {
      const fmm_tables_view* v = opt->tables;
      if (v->p != opt->p || v->n != n_expect || v->k < 1 || v->k > v->n || !v->U || !v->C || !v->S || !v->T || !v->M ||
          !v->L || std::fabs(v->d - opt->d) > 1e-15) {
        set_error("fmm_setup: operator tables do not match (p, n, k, d)");
        return fail(FMM_ECONFIG);
      }
      kifmm::HostTables& H = P.tables;
      H.p = v->p; H.n = v->n; H.k = v->k; H.d = v->d; H.rcond = opt->pinv_rcond;
      const size_t n = v->n, k = v->k;
      H.U.assign(v->U, v->U + n * k);
      H.C.assign(v->C, v->C + 316 * k * k);
      H.S.assign(v->S, v->S + k * n);
      H.T.assign(v->T, v->T + n * k);
      H.M.assign(v->M, v->M + 8 * k * k);
      H.L.assign(v->L, v->L + 8 * k * k);
      if (v->sigma) H.sigma.assign(v->sigma, v->sigma + n);
      else H.sigma.clear();
      // surface grid (same enumeration as the precompute)
      H.surf.clear();
      const int pp = v->p;
      for (int i = 0; i < pp; ++i)
        for (int j = 0; j < pp; ++j)
          for (int l = 0; l < pp; ++l)
            if (i == 0 || j == 0 || l == 0 || i == pp - 1 || j == pp - 1 || l == pp - 1) {
              H.surf.push_back(-1.0 + 2.0 / (pp - 1) * i);
              H.surf.push_back(-1.0 + 2.0 / (pp - 1) * j);
              H.surf.push_back(-1.0 + 2.0 / (pp - 1) * l);
            }
    } else if (opt->operator_file) {  // the table file: load it, or compute and write it
      int k_req = 0;
      const int rc = kifmm::load_tables(opt->operator_file, &P.tables, &k_req);
      if (rc < 0) return fail(FMM_ECONFIG);
      if (rc == 0 && (P.tables.p != opt->p || k_req != opt->k || P.tables.n != n_expect ||
                      std::fabs(P.tables.d - opt->d) > 1e-15 || P.tables.rcond != opt->pinv_rcond)) {
        set_error(std::string("fmm_setup: operator file ") + opt->operator_file + " was built for (p, k, d, rcond) = (" +
                  std::to_string(P.tables.p) + ", " + std::to_string(k_req) + ", " + std::to_string(P.tables.d) + ", " +
                  std::to_string(P.tables.rcond) + ")");
        return fail(FMM_ECONFIG);
      }
      if (rc == 1) {
        if (int b = kifmm::build_tables(opt->p, opt->k, opt->d, opt->pinv_rcond, &P.tables)) return fail(b);
        // the tables are built: a file that cannot be written costs the next setup a
        // recompute, not this one its plan (warning on stderr, setup continues)
        if (kifmm::save_tables(P.tables, opt->k, opt->operator_file))
          std::fprintf(stderr, "kifmm: warning: %s\n", fmm_last_error());
      }
    } else {
      int rc = kifmm::build_tables(opt->p, opt->k, opt->d, opt->pinv_rcond, &P.tables);
      if (rc) return fail(rc);
    }
    if (!(opt->m2l_c2 >= 0)) { set_error("fmm_setup: m2l_c2 must be >= 0"); return fail(FMM_EINVAL); }
    if (int rc = kifmm::build_stage2(P.tables, opt->m2l_c2)) return fail(rc == -2 ? FMM_ECONFIG : rc);
    h->precompute_ms = ms_since(t0);
    P.p = P.tables.p;
    P.n = P.tables.n;
    P.k = P.tables.k;
    P.kp = (P.k + 7) / 8 * 8;
    P.np = (P.n + 7) / 8 * 8;
    P.wx = opt->wx_direct_max < 0 ? P.n : opt->wx_direct_max;
    if (kifmm::upload_tables(P)) return fail(FMM_ECUDA);
    // ---- device tree + lists
    P.tree.N = N;
    t0 = std::chrono::steady_clock::now();
    if (kifmm::build_tree_device(P, points, st)) return fail(FMM_ECUDA);
    h->tree_ms = ms_since(t0);
    if (opt->normals && opt->triangles) {
      set_error("fmm_setup: normals (double layer) and triangles (BEM) are exclusive");
      return fail(FMM_EINVAL);
    }
    if (opt->normals) {  // double-layer sources: mutual pairs use the sign rule of k_near's
      // double-layer path; the warp-pair kernel (mode 2) is single-layer only
      if (kifmm::sort_normals(P, opt->normals, st)) return fail(FMM_ECUDA);
      if (P.sym_opt == 2) P.sym_opt = 0;
    }
    if (opt->triangles) {  // BEM elements: collocation at the points (= centroids), element integrals
      if (opt->nranks > 1) {
        set_error("fmm_setup: BEM elements are single-GPU in this build");
        return fail(FMM_EINVAL);
      }
      P.bem = true;
      P.sym_opt = 0;
      if (kifmm::bem_sort_triangles(P, opt->triangles, st)) return fail(FMM_ECUDA);
      if (int rc = kifmm::bem_check_enclosure(P, st)) return fail(rc == -1 ? FMM_EINVAL : FMM_ECUDA);
    }
    t0 = std::chrono::steady_clock::now();
    if (kifmm::build_lists_device(P, st)) return fail(FMM_ECUDA);
    h->lists_ms = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    if (int rc = kifmm::build_schedules(P, st)) return fail(rc == -4 ? FMM_ENOMEM : FMM_ECUDA);
    h->schedule_ms = ms_since(t0);
    h->part.view(&P.dist);
    if (opt->nccl_id) {  // (a one-rank communicator is allowed: it exercises the transport setup)
      if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("fmm_setup: CUDA error before NCCL init"); return fail(FMM_ECUDA); }
      if (kifmm::nccl_comm_init(P, opt->nccl_id)) return fail(FMM_ENCCL);
      if (cudaStreamCreateWithFlags(&P.stream_comm, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&P.ev_up, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&P.ev_comm, cudaEventDisableTiming) != cudaSuccess) {
        set_error("fmm_setup: creating the communication stream failed");
        return fail(FMM_ECUDA);
      }
    }
    if (densities) {
      if (cudaMalloc(&h->d_default_density, sizeof(double) * N) != cudaSuccess ||
          cudaMemcpyAsync(h->d_default_density, densities, sizeof(double) * N, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        set_error("fmm_setup: copying the default densities failed");
        return fail(FMM_ECUDA);
      }
    }
    // Near field on a second stream (overlap modes, fmm_options.overlap):
    //  3 (default with the mutual near field, up to 8M owned points): all of k_near from the
    //    fork after the densities on the near stream, beside the far field (the GEMVs take
    //    SM slots as k_near's CTAs drain); results joined before the output (C2 -2.5%,
    //    C3 -10%; C4 / C5 +-1%: their long launches leave little tail to fill).  NCCL plans
    //    fork after the ghost exchange.
    //  1 / 2 (diagnostics, k_eval era): whole near field forked after the densities /
    //    beside a high-priority M2L stream.
    //  Off (0) in profiled and split-phase plans: per-phase events on one stream need the
    //  phases serialised.
    //  (A mode running k_near in two parts beside single-warp bulk-copy GEMVs sized to fit
    //  next to it was measured slower — C4 25.2 vs 21.8 ms: DESIGN.md §5.)
    {
      const int64_t owned = P.dist.own_hi - P.dist.own_lo;
      const bool ovl_default = (P.nr_on || P.bem) && !P.profile && owned <= (int64_t)8 << 20;
      P.overlap = !P.split_phases ? (opt->overlap >= 0 ? opt->overlap : (ovl_default ? 3 : 0)) : 0;
      if (P.bem && P.overlap != 3) P.overlap = 0;         // BEM: only the SpMV fork (mode 3)
      if (P.overlap == 3 && !P.nr_on && !P.bem) P.overlap = 0;  // mode 3 runs k_near or the BEM SpMV
      int lo_prio = 0, hi_prio = 0;
      cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
      if (P.overlap &&
          (cudaStreamCreateWithPriority(&P.stream_near, cudaStreamNonBlocking, lo_prio) != cudaSuccess ||
           cudaStreamCreateWithPriority(&P.stream_m2l, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
           cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
           cudaEventCreateWithFlags(&P.ev_m2l, cudaEventDisableTiming) != cudaSuccess ||
           cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming) != cudaSuccess)) {
        set_error("fmm_setup: creating the near-field stream failed");
        return fail(FMM_ECUDA);
      }
    }
    P.ev_phase.resize(kPhases + 1);
    for (auto& e : P.ev_phase) cudaEventCreate(&e);
    if (P.nr_on && P.nr_groups.size() > 1 &&
        (cudaStreamCreateWithFlags(&P.stream_nr2, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&P.ev_nr_fork, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&P.ev_nr_join, cudaEventDisableTiming) != cudaSuccess)) {
      set_error("fmm_setup: creating the second near-field stream failed");
      return fail(FMM_ECUDA);
    }
    if (P.profile)
      for (auto& e : P.ev_near) cudaEventCreate(&e);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      set_error("fmm_setup: CUDA error during setup");
      return fail(FMM_ECUDA);
    }
    *out = h;
    pending = nullptr;
    return FMM_OK;
  });
  if (pending) {
    free_plan_memory(pending);
    delete pending;
  }
  return rc_;
}

int fmm_matvec(fmm_plan* h, const double* density, double* potential, void* stream) {
  return guard("fmm_matvec", [&]() -> int {
    if (!h || !potential) { set_error("fmm_matvec: null plan or potential"); return FMM_EINVAL; }
    const double* q = density ? density : h->d_default_density;
    if (!q) { set_error("fmm_matvec: no density given and none at setup"); return FMM_EINVAL; }
    if (h->P.dist.nranks > 1 && !h->P.nccl_comm) { set_error("fmm_matvec: loopback plan, use fmm_matvec_group"); return FMM_EINVAL; }
    int rc = kifmm::matvec_device(h->P, q, potential, false, (cudaStream_t)stream);
    return rc == 0 ? FMM_OK : rc == -5 ? FMM_ENCCL : FMM_ECUDA;
  });
}

int fmm_matvec_owned(fmm_plan* h, const double* density_owned, double* potential_owned, void* stream) {
  return guard("fmm_matvec_owned", [&]() -> int {
    if (!h) { set_error("fmm_matvec_owned: null plan"); return FMM_EINVAL; }
    const kifmm::DistPlan& D = h->P.dist;
    if (D.own_hi > D.own_lo && (!density_owned || !potential_owned)) {
      set_error("fmm_matvec_owned: null density or potential");
      return FMM_EINVAL;
    }
    if (D.nranks > 1 && !h->P.nccl_comm) { set_error("fmm_matvec_owned: loopback plan, use fmm_matvec_group"); return FMM_EINVAL; }
    int rc = kifmm::matvec_device(h->P, density_owned, potential_owned, true, (cudaStream_t)stream);
    return rc == 0 ? FMM_OK : rc == -5 ? FMM_ENCCL : FMM_ECUDA;
  });
}

int fmm_matvec_owned_host(fmm_plan* h, const double* h_density, double* h_potential, void* stream) {
  return guard("fmm_matvec_owned_host", [&]() -> int {
    if (!h) { set_error("fmm_matvec_owned_host: null plan"); return FMM_EINVAL; }
    kifmm::Plan& P = h->P;
    const int64_t cnt = P.dist.own_hi - P.dist.own_lo;
    if (cnt > 0 && (!h_density || !h_potential)) { set_error("fmm_matvec_owned_host: null argument"); return FMM_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    double* d_q = P.d_io;
    double* d_p = P.d_io + P.tree.N;
    if (cnt > 0 && cudaMemcpyAsync(d_q, h_density, sizeof(double) * cnt, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      set_error("fmm_matvec_owned_host: H2D copy failed");
      return FMM_ECUDA;
    }
    int rc = fmm_matvec_owned(h, d_q, d_p, stream);
    if (rc) return rc;
    if ((cnt > 0 && cudaMemcpyAsync(h_potential, d_p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("fmm_matvec_owned_host: D2H copy failed");
      return FMM_ECUDA;
    }
    return FMM_OK;
  });
}

int fmm_gmres(fmm_plan* h, const double* rhs, double* x, int restart, int maxit, double tol, void* stream, int* iters,
              double* relres, double* t_matvec_ms) {
  return guard("fmm_gmres", [&]() -> int {
    if (!h || !rhs || !x || !iters || !relres || restart < 1 || maxit < 0 || !(tol >= 0)) {
      set_error("fmm_gmres: invalid argument");
      return FMM_EINVAL;
    }
    if (h->P.dist.nranks > 1) { set_error("fmm_gmres: single-GPU plans only"); return FMM_EINVAL; }
    int rc = kifmm::gmres_solve(h->P, rhs, x, restart, maxit, tol, (cudaStream_t)stream, iters, relres, t_matvec_ms);
    return rc ? FMM_ECUDA : FMM_OK;
  });
}

int fmm_owned_range(const fmm_plan* h, int64_t* begin, int64_t* end) {
  return guard("fmm_owned_range", [&]() -> int {
    if (!h || !begin || !end) { set_error("fmm_owned_range: null argument"); return FMM_EINVAL; }
    *begin = h->P.dist.own_lo;
    *end = h->P.dist.own_hi;
    return FMM_OK;
  });
}

int fmm_nccl_unique_id(void* id128) {
  return guard("fmm_nccl_unique_id", [&]() -> int {
    if (!id128) { set_error("fmm_nccl_unique_id: null argument"); return FMM_EINVAL; }
    return kifmm::nccl_unique_id(id128) ? FMM_ENCCL : FMM_OK;
  });
}

// Loopback transport: the same stage sequence as matvec_device, with every exchange
// done as device-to-device copies between the group's plans.
int fmm_matvec_group(fmm_plan* const* plans, int np, const double* const* dens, double* const* pots, int owned,
                     void* stream) {
  return guard("fmm_matvec_group", [&]() -> int {
    if (!plans || np < 1 || !dens || !pots) { set_error("fmm_matvec_group: invalid argument"); return FMM_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<kifmm::Plan*> Ps(np);
    for (int r = 0; r < np; ++r) {
      if (!plans[r] || plans[r]->P.dist.nranks != np || plans[r]->P.dist.rank != r) {
        set_error("fmm_matvec_group: plans[r] must be rank r of an nplans-rank partition");
        return FMM_EINVAL;
      }
      Ps[r] = &plans[r]->P;
    }
    for (int r = 1; r < np; ++r)
      if (Ps[r]->tree.N != Ps[0]->tree.N || Ps[r]->tree.nboxes != Ps[0]->tree.nboxes || Ps[r]->kp != Ps[0]->kp ||
          Ps[r]->dist.bnd != Ps[0]->dist.bnd || Ps[r]->n_straddle != Ps[0]->n_straddle) {
        set_error("fmm_matvec_group: the plans do not describe one partition of one problem");
        return FMM_EINVAL;
      }
    auto stage = [&](int sg) -> int {
      for (int r = 0; r < np; ++r)
        if (kifmm::matvec_stage(*Ps[r], sg, dens[r], pots[r], owned != 0, st)) return FMM_ECUDA;
      return 0;
    };
    auto exchange = [&](kifmm::Exchange kifmm::Plan::*which) -> int {
      for (int r = 0; r < np; ++r)
        for (int s = 0; s < np; ++s) {
          if (s == r) continue;
          kifmm::Exchange& R = Ps[r]->*which;
          kifmm::Exchange& S = Ps[s]->*which;
          const int nr = R.recv_off[s + 1] - R.recv_off[s], ns = S.send_off[r + 1] - S.send_off[r];
          if (nr != ns) { set_error("fmm_matvec_group: send / receive lists disagree"); return FMM_EINVAL; }
          if (nr && cudaMemcpyAsync(R.d_recv + (size_t)R.recv_off[s] * R.row, S.d_send + (size_t)S.send_off[r] * S.row,
                                    sizeof(double) * nr * R.row, cudaMemcpyDefault, st) != cudaSuccess) {
            set_error("fmm_matvec_group: exchange copy failed");
            return FMM_ECUDA;
          }
        }
      return 0;
    };
    int rc;
    if ((rc = stage(0))) return rc;
    if (owned && (rc = exchange(&kifmm::Plan::xd))) return rc;
    if ((rc = stage(1))) return rc;
    // allreduce of the straddlers' partial multipoles: accumulate on the host (exact
    // order: rank 0, 1, ...), as NCCL's ring / tree order is unspecified anyway
    const size_t cnt = (size_t)Ps[0]->n_straddle * Ps[0]->kp;
    if (cnt) {
      std::vector<double> sum(cnt, 0.0), part(cnt);
      for (int r = 0; r < np; ++r) {
        if (cudaMemcpyAsync(part.data(), Ps[r]->d_straddle_buf, sizeof(double) * cnt, cudaMemcpyDefault, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          set_error("fmm_matvec_group: straddler copy failed");
          return FMM_ECUDA;
        }
        for (size_t i = 0; i < cnt; ++i) sum[i] += part[i];
      }
      for (int r = 0; r < np; ++r)
        if (cudaMemcpyAsync(Ps[r]->d_straddle_buf, sum.data(), sizeof(double) * cnt, cudaMemcpyDefault, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          set_error("fmm_matvec_group: straddler copy failed");
          return FMM_ECUDA;
        }
    }
    if ((rc = stage(2))) return rc;
    if ((rc = exchange(&kifmm::Plan::xq))) return rc;
    if ((rc = stage(3))) return rc;
    if (!owned) {
      for (int r = 0; r < np; ++r)
        for (int s = 0; s < np; ++s) {
          const auto& b = Ps[s]->dist.bnd;
          const size_t c = (size_t)(b[s + 1] - b[s]);
          if (s == r || !c) continue;
          if (cudaMemcpyAsync(Ps[r]->d_pot_near + b[s], Ps[s]->d_pot_near + b[s], sizeof(double) * c, cudaMemcpyDefault,
                              st) != cudaSuccess) {
            set_error("fmm_matvec_group: allgather copy failed");
            return FMM_ECUDA;
          }
        }
    }
    if ((rc = stage(4))) return rc;
    return FMM_OK;
  });
}

int fmm_partition_host(int nboxes, const int32_t* level, const int32_t* parent, const int32_t* pbeg,
                       const int32_t* pend, const uint8_t* leaf, int64_t nU, const int32_t* U, int64_t nV,
                       const int32_t* V, int64_t nW, const int32_t* W, int64_t nX, const int32_t* X, int n, int k,
                       int nranks, int rank, fmm_partition** out) {
  return guard("fmm_partition_host", [&]() -> int {
    if (!out || nboxes < 1 || !level || !parent || !pbeg || !pend || !leaf || (nU && !U) || (nV && !V) || (nW && !W) ||
        (nX && !X) || nranks < 1 || rank < 0 || rank >= nranks) {
      set_error("fmm_partition_host: invalid argument");
      return FMM_EINVAL;
    }
    *out = nullptr;
    kifmm::PartitionInput in;
    in.nboxes = nboxes;
    in.level = level; in.parent = parent; in.pbeg = pbeg; in.pend = pend; in.leaf = leaf;
    in.nU = nU; in.U = U; in.ustride = 2;
    in.nV = nV; in.V = V; in.vstride = 3;
    in.nW = nW; in.W = W; in.wstride = 3;
    in.nX = nX; in.X = X; in.xstride = 3;
    in.n = n; in.k = k;
    for (int b = 0; b < nboxes; ++b)
      if (parent[b] >= b || (b > 0 && parent[b] < 0) || pbeg[b] > pend[b]) {
        set_error("fmm_partition_host: boxes must be level-major with parents first");
        return FMM_EINVAL;
      }
    fmm_partition* p = new (std::nothrow) fmm_partition();
    if (!p) { set_error("fmm_partition_host: out of host memory"); return FMM_ENOMEM; }
    if (kifmm::build_partition(in, nranks, rank, &p->own)) { delete p; return FMM_EINVAL; }
    p->view(&p->own);
    *out = p;
    return FMM_OK;
  });
}

int fmm_partition_get(const fmm_partition* p, int what, int64_t* count, const int32_t** data) {
  return guard("fmm_partition_get", [&]() -> int {
    if (!p || !p->D || !count || !data) { set_error("fmm_partition_get: null argument"); return FMM_EINVAL; }
    const kifmm::DistPlan& D = *p->D;
    const std::vector<int>* v = nullptr;
    switch (what) {
      case 0: v = &D.bnd; break;
      case 1: v = &p->inD32; break;
      case 2: v = &D.straddle; break;
      case 3: v = &p->full32; break;
      case 4: v = &D.q_send; break;
      case 5: v = &D.q_send_off; break;
      case 6: v = &D.q_recv; break;
      case 7: v = &D.q_recv_off; break;
      case 8: v = &D.d_send; break;
      case 9: v = &D.d_send_off; break;
      case 10: v = &D.d_recv; break;
      case 11: v = &D.d_recv_off; break;
      default: set_error("fmm_partition_get: unknown array"); return FMM_EINVAL;
    }
    *count = (int64_t)v->size();
    *data = v->data();
    return FMM_OK;
  });
}

void fmm_partition_free(fmm_partition* p) { delete p; }

const fmm_partition* fmm_plan_partition(const fmm_plan* h) { return h ? &h->part : nullptr; }

int fmm_matvec_host(fmm_plan* h, const double* h_density, double* h_potential, void* stream) {
  return guard("fmm_matvec_host", [&]() -> int {
    if (!h || !h_density || !h_potential) { set_error("fmm_matvec_host: null argument"); return FMM_EINVAL; }
    kifmm::Plan& P = h->P;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = P.tree.N;
    double* d_q = P.d_io;
    double* d_p = P.d_io + N;
    if (cudaMemcpyAsync(d_q, h_density, sizeof(double) * N, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      set_error("fmm_matvec_host: H2D copy failed");
      return FMM_ECUDA;
    }
    if (P.dist.nranks > 1 && !P.nccl_comm) { set_error("fmm_matvec_host: loopback plan, use fmm_matvec_group"); return FMM_EINVAL; }
    int rc = kifmm::matvec_device(P, d_q, d_p, false, st);
    if (rc) return rc == -5 ? FMM_ENCCL : FMM_ECUDA;
    if (cudaMemcpyAsync(h_potential, d_p, sizeof(double) * N, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("fmm_matvec_host: D2H copy failed");
      return FMM_ECUDA;
    }
    return FMM_OK;
  });
}

// Several matvecs with host buffers, copies overlapped with compute: matvec i reads
// staging pair i % 2; its density's H2D runs on a copy stream while matvec i - 1 computes,
// its potential's D2H on another copy stream while matvec i + 1 computes.  Events order
// each staging buffer's reuse (H2D into a pair waits for the matvec two steps back to have
// read it; that matvec's output waits for the D2H two steps back).
static int matvec_host_batch_body(fmm_plan* h, const double* const* hq, double* const* hp, int count, bool owned,
                                  cudaStream_t st);
static int matvec_host_batch(fmm_plan* h, const double* const* hq, double* const* hp, int count, bool owned,
                             cudaStream_t st) {
  const int rc = matvec_host_batch_body(h, hq, hp, count, owned, st);
  if (rc != FMM_OK) {  // no copy may still touch the caller's host buffers after an error return
    if (h->P.stream_h2d) cudaStreamSynchronize(h->P.stream_h2d);
    if (h->P.stream_d2h) cudaStreamSynchronize(h->P.stream_d2h);
  }
  return rc;
}

static int matvec_host_batch_body(fmm_plan* h, const double* const* hq, double* const* hp, int count, bool owned,
                                  cudaStream_t st) {
  kifmm::Plan& P = h->P;
  const int64_t N = P.tree.N;
  const int64_t cnt = owned ? P.dist.own_hi - P.dist.own_lo : N;
  if (!P.d_io2 && cudaMalloc(&P.d_io2, sizeof(double) * 2 * std::max<int64_t>(N, 1)) != cudaSuccess) {
    set_error("fmm_matvec_host_batch: staging buffers: out of device memory");
    return FMM_ENOMEM;
  }
  if (!P.stream_h2d && (cudaStreamCreateWithFlags(&P.stream_h2d, cudaStreamNonBlocking) != cudaSuccess ||
                        cudaStreamCreateWithFlags(&P.stream_d2h, cudaStreamNonBlocking) != cudaSuccess)) {
    set_error("fmm_matvec_host_batch: creating the copy streams failed");
    return FMM_ECUDA;
  }
  for (auto& e : P.ev_io)
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      set_error("fmm_matvec_host_batch: creating events failed");
      return FMM_ECUDA;
    }
  cudaEvent_t* ev_in = P.ev_io;       // density staged
  cudaEvent_t* ev_done = P.ev_io + 2; // matvec finished (input read, output written)
  cudaEvent_t* ev_out = P.ev_io + 4;  // potential copied out
  double* din[2] = {P.d_io, P.d_io2};
  double* dout[2] = {P.d_io + N, P.d_io2 + N};
  auto cuda = [&](cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    set_error(std::string("fmm_matvec_host_batch: ") + what + ": " + cudaGetErrorString(e));
    return false;
  };
  // the copy streams start after the work already queued on st (which may use d_io)
  if (!cuda(cudaEventRecord(P.ev_io[6], st), "event") || !cuda(cudaStreamWaitEvent(P.stream_h2d, P.ev_io[6], 0), "wait") ||
      !cuda(cudaStreamWaitEvent(P.stream_d2h, P.ev_io[6], 0), "wait"))
    return FMM_ECUDA;
  for (int i = 0; i < count; ++i) {
    const int b = i & 1;
    if (i >= 2 && !cuda(cudaStreamWaitEvent(P.stream_h2d, ev_done[b], 0), "wait")) return FMM_ECUDA;
    if (cnt > 0 && !cuda(cudaMemcpyAsync(din[b], hq[i], sizeof(double) * cnt, cudaMemcpyHostToDevice, P.stream_h2d), "H2D copy"))
      return FMM_ECUDA;
    if (!cuda(cudaEventRecord(ev_in[b], P.stream_h2d), "event") || !cuda(cudaStreamWaitEvent(st, ev_in[b], 0), "wait"))
      return FMM_ECUDA;
    if (i >= 2 && !cuda(cudaStreamWaitEvent(st, ev_out[b], 0), "wait")) return FMM_ECUDA;
    const int rc = kifmm::matvec_device(P, din[b], dout[b], owned, st);
    if (rc) return rc == -5 ? FMM_ENCCL : FMM_ECUDA;
    if (!cuda(cudaEventRecord(ev_done[b], st), "event") || !cuda(cudaStreamWaitEvent(P.stream_d2h, ev_done[b], 0), "wait"))
      return FMM_ECUDA;
    if (cnt > 0 && !cuda(cudaMemcpyAsync(hp[i], dout[b], sizeof(double) * cnt, cudaMemcpyDeviceToHost, P.stream_d2h), "D2H copy"))
      return FMM_ECUDA;
    if (!cuda(cudaEventRecord(ev_out[b], P.stream_d2h), "event")) return FMM_ECUDA;
  }
  // st is ordered after the last D2H (a later call may reuse the staging buffers)
  if (!cuda(cudaEventRecord(P.ev_io[6], P.stream_d2h), "event") || !cuda(cudaStreamWaitEvent(st, P.ev_io[6], 0), "wait") ||
      !cuda(cudaStreamSynchronize(st), "synchronize"))
    return FMM_ECUDA;
  return FMM_OK;
}

int fmm_matvec_host_batch(fmm_plan* h, const double* const* h_density, double* const* h_potential, int count,
                          void* stream) {
  return guard("fmm_matvec_host_batch", [&]() -> int {
    if (!h || count < 0 || (count > 0 && (!h_density || !h_potential))) {
      set_error("fmm_matvec_host_batch: null argument or negative count");
      return FMM_EINVAL;
    }
    for (int i = 0; i < count; ++i)
      if (!h_density[i] || !h_potential[i]) { set_error("fmm_matvec_host_batch: null buffer"); return FMM_EINVAL; }
    if (h->P.dist.nranks > 1 && !h->P.nccl_comm) { set_error("fmm_matvec_host_batch: loopback plan, use fmm_matvec_group"); return FMM_EINVAL; }
    return matvec_host_batch(h, h_density, h_potential, count, false, (cudaStream_t)stream);
  });
}

int fmm_matvec_owned_host_batch(fmm_plan* h, const double* const* h_density_owned, double* const* h_potential_owned,
                                int count, void* stream) {
  return guard("fmm_matvec_owned_host_batch", [&]() -> int {
    if (!h || count < 0 || (count > 0 && (!h_density_owned || !h_potential_owned))) {
      set_error("fmm_matvec_owned_host_batch: null argument or negative count");
      return FMM_EINVAL;
    }
    const kifmm::DistPlan& D = h->P.dist;
    for (int i = 0; i < count; ++i)
      if (D.own_hi > D.own_lo && (!h_density_owned[i] || !h_potential_owned[i])) {
        set_error("fmm_matvec_owned_host_batch: null buffer");
        return FMM_EINVAL;
      }
    if (D.nranks > 1 && !h->P.nccl_comm) { set_error("fmm_matvec_owned_host_batch: loopback plan, use fmm_matvec_group"); return FMM_EINVAL; }
    return matvec_host_batch(h, h_density_owned, h_potential_owned, count, true, (cudaStream_t)stream);
  });
}

void fmm_free(fmm_plan* h) {
  if (!h) return;
  free_plan_memory(h);
  delete h;
}

int fmm_info(const fmm_plan* h, fmm_info_t* info) {
  return guard("fmm_info", [&]() -> int {
    if (!h || !info) { set_error("fmm_info: null argument"); return FMM_EINVAL; }
    const kifmm::Plan& P = h->P;
    std::memset(info, 0, sizeof(*info));
    info->N = P.tree.N;
    info->p = P.p; info->n = P.n; info->k = P.k; info->kp = P.kp;
    info->nboxes = P.tree.nboxes; info->nleaves = P.tree.nleaves; info->nlevels = P.tree.nlevels;
    info->nU = P.lists.nU; info->nV = P.lists.nV; info->nW = P.lists.nW; info->nX = P.lists.nX;
    info->n_s2m = P.n_s2m; info->n_xnd = P.n_xnd; info->n_l2t = P.n_l2t; info->n_wnd = P.n_wnd;
    info->m2l_tiles = P.g_m2l_sib.ntiles + P.g_m2l_sib_ghost.ntiles; info->m2l_pairs = P.nV_local;
    info->launches = P.launches;
    info->r0 = P.tree.r0;
    for (int d = 0; d < 3; ++d) info->lo_root[d] = P.tree.lo_root[d];
    info->precompute_ms = h->precompute_ms; info->tree_ms = h->tree_ms; info->lists_ms = h->lists_ms;
    info->schedule_ms = h->schedule_ms;
    if (P.profile && P.profiled && P.ev_phase.size() == kPhases + 1 && cudaEventSynchronize(P.ev_phase[kPhases]) == cudaSuccess)
      for (int i = 0; i < kPhases; ++i) cudaEventElapsedTime(&info->phase_ms[i], P.ev_phase[i], P.ev_phase[i + 1]);
    info->near_ms = -1;
    info->overlap = P.overlap;
    if (P.profile && P.profiled && P.near_timed && cudaEventSynchronize(P.ev_near[1]) == cudaSuccess) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, P.ev_near[0], P.ev_near[1]) == cudaSuccess) info->near_ms = ms;
    }
    info->nranks = P.dist.nranks;
    info->rank = P.dist.rank;
    info->own_lo = P.dist.own_lo;
    info->own_hi = P.dist.own_hi;
    info->n_straddle = P.n_straddle;
    info->ghost_q_recv = P.xq.nrecv;
    info->ghost_q_send = P.xq.nsend;
    info->ghost_d_recv = P.xd.nrecv;
    info->ghost_d_send = P.xd.nsend;
    info->nV_local = P.nV_local;
    info->leaf_op_bytes = P.leaf_op_bytes;
    info->bem_near_bytes = P.bem_near_bytes;
    info->bem_extrusion = P.bem_extrusion;
    info->near_mutual_leaves = P.n_tleaf_mut;
    info->near_mutual_pairs = P.n_mut_pairs;
    info->near_sym_pairs = P.n_sym;
    info->m2l_exec_flops = P.m2l_exec_flops;
    info->near_pairs = P.n_near_pairs;
    info->m2l_flops = P.m2l_flops;
    info->m2l_eps2 = P.tables.eps2;
    {
      double rs = 0;
      for (int r : P.tables.ranks) rs += r;
      info->m2l_rank_mean = P.tables.ranks.empty() ? P.k : rs / P.tables.ranks.size();
    }
    return FMM_OK;
  });
}

int fmm_export_tree(const fmm_plan* h, int32_t* level, uint64_t* key, int32_t* parent, int32_t* pbeg, int32_t* pend,
                    uint8_t* leaf, int32_t* perm, double* geom) {
  return guard("fmm_export_tree", [&]() -> int {
    if (!h) { set_error("fmm_export_tree: null plan"); return FMM_EINVAL; }
    const kifmm::Tree& T = h->P.tree;
    const size_t nb = T.nboxes;
    for (size_t b = 0; b < nb; ++b) {
      if (level) level[b] = T.level[b];
      if (key) key[b] = T.key[b];
      if (parent) parent[b] = T.parent[b];
      if (pbeg) pbeg[b] = T.pbeg[b];
      if (pend) pend[b] = T.pend[b];
      if (leaf) leaf[b] = T.leaf[b];
    }
    if (perm && cudaMemcpy(perm, T.d_perm, sizeof(int32_t) * T.N, cudaMemcpyDeviceToHost) != cudaSuccess) {
      set_error("fmm_export_tree: copy failed");
      return FMM_ECUDA;
    }
    if (geom) {
      for (int d = 0; d < 3; ++d) geom[d] = T.lo_root[d];
      geom[3] = T.r0;
      geom[4] = T.scale;
    }
    return FMM_OK;
  });
}

int fmm_export_lists(const fmm_plan* h, int32_t* U, int32_t* V, int32_t* W, int32_t* X) {
  return guard("fmm_export_lists", [&]() -> int {
    if (!h) { set_error("fmm_export_lists: null plan"); return FMM_EINVAL; }
    const kifmm::Lists& L = h->P.lists;
    std::vector<int4> tmp;
    if (U && L.nU && cudaMemcpy(U, L.d_U, sizeof(int2) * L.nU, cudaMemcpyDeviceToHost) != cudaSuccess) goto err;
    if (V && L.nV) {
      tmp.resize(L.nV);
      if (cudaMemcpy(tmp.data(), L.d_V, sizeof(int4) * L.nV, cudaMemcpyDeviceToHost) != cudaSuccess) goto err;
      for (int i = 0; i < L.nV; ++i) { V[3 * i] = tmp[i].x; V[3 * i + 1] = tmp[i].y; V[3 * i + 2] = tmp[i].z; }
    }
    if (W && L.nW) {
      tmp.resize(L.nW);
      if (cudaMemcpy(tmp.data(), L.d_W, sizeof(int4) * L.nW, cudaMemcpyDeviceToHost) != cudaSuccess) goto err;
      for (int i = 0; i < L.nW; ++i) { W[3 * i] = tmp[i].x; W[3 * i + 1] = tmp[i].y; W[3 * i + 2] = tmp[i].z; }
    }
    if (X && L.nX) {
      tmp.resize(L.nX);
      if (cudaMemcpy(tmp.data(), L.d_X, sizeof(int4) * L.nX, cudaMemcpyDeviceToHost) != cudaSuccess) goto err;
      for (int i = 0; i < L.nX; ++i) { X[3 * i] = tmp[i].x; X[3 * i + 1] = tmp[i].y; X[3 * i + 2] = tmp[i].z; }
    }
    return FMM_OK;
  err:
    set_error("fmm_export_lists: copy failed");
    return FMM_ECUDA;
  });
}

int fmm_export_phase(const fmm_plan* h, int which, double* out) {
  return guard("fmm_export_phase", [&]() -> int {
    if (!h || !out || which < 0 || which > 3) { set_error("fmm_export_phase: invalid argument"); return FMM_EINVAL; }
    const kifmm::Plan& P = h->P;
    if (cudaDeviceSynchronize() != cudaSuccess) { set_error("fmm_export_phase: device error"); return FMM_ECUDA; }
    if (which >= 2) {
      const double* src = which == 2 ? P.d_pot_near : P.d_pot_far;
      if (cudaMemcpy(out, src, sizeof(double) * P.tree.N, cudaMemcpyDeviceToHost) != cudaSuccess) {
        set_error("fmm_export_phase: copy failed");
        return FMM_ECUDA;
      }
      return FMM_OK;
    }
    const double* src = which == 0 ? P.d_qhat : P.d_lhat;
    const size_t nb = P.tree.nboxes;
    std::vector<double> tmp(nb * P.kp);
    if (cudaMemcpy(tmp.data(), src, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      set_error("fmm_export_phase: copy failed");
      return FMM_ECUDA;
    }
    for (size_t b = 0; b < nb; ++b)
      for (int a = 0; a < P.k; ++a) out[b * P.k + a] = tmp[b * P.kp + a];
    return FMM_OK;
  });
}

}  // extern "C"
