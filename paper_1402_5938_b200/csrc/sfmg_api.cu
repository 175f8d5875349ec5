// C ABI of libsfmg (include/sfmg.h): argument checking, workspace carving, and the host-side
// orchestration of the kernels (Chebyshev recurrence scalars, V-cycle recursion, Algorithm 1).
// Host code only launches kernels on the caller's stream; no arithmetic of the method runs here
// except the scalar Chebyshev recurrence coefficients (R7).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "sfmg_internal.h"

namespace sfmg {

static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }

static sfmg_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return SFMG_E_CUDA;
}

#define CK(call)                                         \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static sfmg_status check_problem(const sfmg_problem* pr) {
  if (!pr) { set_error("null problem"); return SFMG_E_ARG; }
  if (pr->order < 1 || pr->order > kMaxOrder) { set_error("order must be 1..16"); return SFMG_E_ORDER; }
  if (pr->dim != 0 && pr->dim != 2 && pr->dim != 3) { set_error("dim must be 0, 2 or 3"); return SFMG_E_ARG; }
  const bool two = pr->dim == 2;
  if (two && pr->nez > 1) { set_error("2-D problems have nez = 0 or 1"); return SFMG_E_MESH; }
  if (pr->nex < 1 || pr->ney < 1 || (!two && pr->nez < 1)) { set_error("element counts must be >= 1"); return SFMG_E_MESH; }
  long long Mx = (long long)pr->nex * pr->order + 1, My = (long long)pr->ney * pr->order + 1,
            Mz = two ? 1 : (long long)pr->nez * pr->order + 1;
  if (Mx * My * Mz >= (1LL << 31)) { set_error("lattice exceeds 2^31 nodes"); return SFMG_E_MESH; }
  if (pr->warp != 0 && pr->warp != 1) { set_error("warp must be 0 or 1"); return SFMG_E_ARG; }
  if (pr->coeff < 0 || pr->coeff > (two ? 4 : 3)) { set_error("coeff must be 0..3 (2-D: 0..4)"); return SFMG_E_ARG; }
  if (pr->quadrature != 0 && pr->quadrature != 1) { set_error("quadrature must be 0 or 1"); return SFMG_E_ARG; }
  return SFMG_OK;
}

static MeshDev make_mesh(const sfmg_problem* pr) {
  MeshDev m;
  m.nex = pr->nex; m.ney = pr->ney; m.nez = pr->nez; m.p = pr->order;
  m.Mx = pr->nex * pr->order + 1; m.My = pr->ney * pr->order + 1; m.Mz = pr->nez * pr->order + 1;
  m.E = (long long)pr->nex * pr->ney * pr->nez;
  m.N = (long long)m.Mx * m.My * m.Mz;
  m.warp = pr->warp; m.coeff = pr->coeff;
  m.amp = pr->warp_amp; m.c0 = pr->c0; m.c1 = pr->c1;
  m.quad = pr->quadrature;
  m.Kb0 = 0; m.Kb1 = m.Mz - 1;
  if (pr->dim == 2) {   // quadrilaterals: one lattice plane, no z boundary (NEXT-2)
    m.dim = 2;
    m.nez = 1;
    m.Mz = 1;
    m.E = (long long)m.nex * m.ney;
    m.N = (long long)m.Mx * m.My;
    m.Kb0 = m.Kb1 = -1;
  }
  return m;
}

struct LevelLayout {
  size_t G, dinv, y, t0, t1, t2, partials, scalars, counter, bad, total;
};

static LevelLayout level_layout(const MeshDev& m) {
  LevelLayout L;
  const long long n3 = (long long)(m.p + 1) * (m.p + 1) * (m.p + 1);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes); return o; };
  if (m.dim == 2) L.G = take(sizeof(double) * 3 * (size_t)m.E * (m.p + 1) * (m.p + 1));   // [E][3][n^2]
  else L.G = take(sizeof(double) * 6 * (size_t)geometry_elems(m.p, m.E) * n3);
  L.dinv = take(sizeof(double) * m.N);
  L.y = take(sizeof(double) * m.N);
  L.t0 = take(sizeof(double) * m.N);
  L.t1 = take(sizeof(double) * m.N);
  L.t2 = take(sizeof(double) * m.N);
  L.partials = take(sizeof(double) * kRedBlocks * kRedSlots);
  L.scalars = take(sizeof(double) * 32);
  L.counter = take(sizeof(unsigned int));
  L.bad = take(sizeof(int));
  L.total = off;
  return L;
}

static sfmg_status level_build(const sfmg_problem* pr, void* d_ws, size_t ws_bytes, cudaStream_t s,
                               sfmg_level_s** out) {
  MeshDev m = make_mesh(pr);
  LevelLayout L = level_layout(m);
  if (!d_ws || ((uintptr_t)d_ws & 255) || ws_bytes < L.total) {
    set_error("workspace too small or not 256-byte aligned");
    return SFMG_E_WORKSPACE;
  }
  char* base = (char*)d_ws;
  sfmg_level_s* lv = new (std::nothrow) sfmg_level_s();
  if (!lv) { set_error("host allocation failed"); return SFMG_E_ARG; }
  lv->prob = *pr; lv->m = m; lv->p = m.p; lv->n = m.p + 1;
  lv->n3 = (long long)lv->n * lv->n * (m.dim == 2 ? 1 : lv->n); lv->E = m.E; lv->N = m.N;
  lv->G = (double*)(base + L.G);
  lv->dinv = (double*)(base + L.dinv);
  lv->y = (double*)(base + L.y);
  lv->t0 = (double*)(base + L.t0);
  lv->t1 = (double*)(base + L.t1);
  lv->t2 = (double*)(base + L.t2);
  lv->red.partials = (double*)(base + L.partials);
  lv->red.scalars = (double*)(base + L.scalars);
  lv->red.counter = (unsigned int*)(base + L.counter);
  lv->bad = (int*)(base + L.bad);
  lv->ws_bytes = L.total;
  lv->owned_by_hier = false;
  auto fail = [&](sfmg_status st) { delete lv; return st; };
  cudaError_t e;
  if ((e = upload_order_tables(m.p, s))) return fail(cuda_fail(e, "upload_order_tables"));
  if (m.dim == 2 && (e = upload_2d_tables(m.p, m.quad))) return fail(cuda_fail(e, "upload_2d_tables"));
  if ((e = cudaMemsetAsync(lv->red.counter, 0, sizeof(unsigned int), s))) return fail(cuda_fail(e, "memset"));
  if ((e = cudaMemsetAsync(lv->bad, 0, sizeof(int), s))) return fail(cuda_fail(e, "memset"));
  if ((e = launch_geometry(m, lv->G, lv->bad, s))) return fail(cuda_fail(e, "geometry"));
  int bad = 0;
  if ((e = cudaMemcpyAsync(&bad, lv->bad, sizeof(int), cudaMemcpyDeviceToHost, s))) return fail(cuda_fail(e, "copy"));
  if ((e = cudaStreamSynchronize(s))) return fail(cuda_fail(e, "geometry sync"));
  if (bad > 0) {
    set_error("det J <= 0 at " + std::to_string(bad) + " quadrature points");
    return fail(SFMG_E_GEOMETRY);
  }
  if ((e = launch_diag(m, 0, lv->G, lv->t0, s))) return fail(cuda_fail(e, "diag"));
  if ((e = launch_recip(lv->t0, lv->dinv, m.N, s))) return fail(cuda_fail(e, "recip"));
  *out = lv;
  return SFMG_OK;
}

// y <- A_D u (bc 0) or A u (bc 1).  p <= 2: zero fill, then the thread-per-element kernel whose
// canonical owner elements also store the boundary pass-through values (I - M) u.  p >= 3: the
// boundary/zero init kernel, then the persistent kernel launched as its programmatic dependent
// (its factor prefetches overlap the init).  Both orders were measured; each is the faster for
// its kernel family.
// The element (operator) kernel, with optional event timing for benchmarks (sfmg_profile_*).
static cudaError_t element_kernel(sfmg_level_s* lv, int bc, const double* u, double* v, int wait_mode,
                                  int write_bnd, cudaStream_t s) {
  if (!lv->prof) return launch_apply(lv->m, bc, lv->G, u, v, wait_mode, write_bnd, s);
  if (lv->prof_used + 2 > lv->prof_ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t ev;
      cudaError_t e = cudaEventCreate(&ev);
      if (e) return e;
      lv->prof_ev.push_back(ev);
    }
  }
  cudaEvent_t a = lv->prof_ev[lv->prof_used], b = lv->prof_ev[lv->prof_used + 1];
  lv->prof_used += 2;
  cudaError_t e = cudaEventRecord(a, s);
  if (e) return e;
  e = launch_apply(lv->m, bc, lv->G, u, v, wait_mode, write_bnd, s);
  if (e) return e;
  return cudaEventRecord(b, s);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

static cudaError_t op_apply(sfmg_level_s* lv, int bc, const double* u, double* v, cudaStream_t s) {
  cudaError_t e;
  // opt-in (SFMG_FUSED=1): one fused kernel, A_D u accumulated in an L2-resident plane ring inside lv->y
  // and copied out one element layer behind (no v init, no RED traffic to HBM)
  if (bc == 0 && v != lv->y && u != lv->y && !lv->prof && fused_available(lv->m) && aligned16(u) && aligned16(v)) {
    if ((e = fused_zero_ring(lv->m, lv->y, s))) return e;
    return launch_fused_step(lv->m, lv->G, u, nullptr, v, nullptr, nullptr, lv->y, 0.0, 0.0, 1, s);
  }
  if (lv->p <= 2 && !lv->m.quad && lv->m.dim == 3) {   // zero v, then the thread-per-element kernel, whose
                                                       // canonical owner elements store (I - M) u
    if ((e = launch_zero(v, lv->N, s))) return e;
    return element_kernel(lv, bc, u, v, 1, 1, s);
  }
  e = launch_init(lv->m, bc, u, 0.0, v, s);
  if (e) return e;
  return element_kernel(lv, bc, u, v, 1, 0, s);
}

// Degree-K Chebyshev application, iterate form of R7:
//   x1 = x0 + (1/theta) D^{-1} (b - A x0)
//   x_{k+1} = x_k + rho_k rho_{k-1} (x_k - x_{k-1}) + (2 rho_k / delta) D^{-1} (b - A x_k)
// with rho_0 = 1/sigma, rho_k = 1/(2 sigma - rho_{k-1}), sigma = theta/delta.  K applies.
static cudaError_t op_cheb(sfmg_level_s* lv, const double* b, double* x, int K, double lo, double hi,
                           cudaStream_t s) {
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  double rho_prev = 1.0 / sigma;
  const bool fused = !lv->prof && fused_available(lv->m) && aligned16(b) && aligned16(x) && b != lv->y && x != lv->y;
  cudaError_t e = fused ? fused_zero_ring(lv->m, lv->y, s) : op_apply(lv, 0, x, lv->y, s);
  if (e) return e;
  double* A = x;
  double* B = lv->t0;
  double* cur = A;
  double* prev = nullptr;
  for (int k = 0; k < K; ++k) {
    double c1 = 0.0, c2 = 1.0 / theta;
    if (k > 0) {
      const double rho = 1.0 / (2.0 * sigma - rho_prev);
      c1 = rho * rho_prev;
      c2 = 2.0 * rho / delta;
      rho_prev = rho;
    }
    double* out = (k == K - 1) ? A : (k == 0 ? B : prev);
    if (fused) {   // one kernel per step: apply + recurrence, y = A_D x_k never leaves L2
      e = launch_fused_step(lv->m, lv->G, cur, prev ? prev : cur, out, b, lv->dinv, lv->y, c1, c2, 0, s);
      if (e) return e;
      prev = cur;
      cur = out;
      continue;
    }
    if (k > 0) {
      e = element_kernel(lv, 0, cur, lv->y, 2, 0, s);   // y was re-initialised by the last update
      if (e) return e;
    }
    e = launch_cheb_update(lv->m, cur, prev ? prev : cur, out, b, lv->y, lv->dinv, c1, c2, s);
    if (e) return e;
    prev = cur;
    cur = out;
  }
  return cudaSuccess;
}

// `steps` damped point-Jacobi steps x += omega D^{-1} (b - A_D x): the
// Chebyshev update kernel with c1 = 0, c2 = omega (it also re-initialises y for the next apply).
static cudaError_t op_jacobi(sfmg_level_s* lv, const double* b, double* x, int steps, double omega,
                             cudaStream_t s) {
  if (!lv->prof && fused_available(lv->m) && aligned16(b) && aligned16(x) && b != lv->y && x != lv->y) {
    cudaError_t e = fused_zero_ring(lv->m, lv->y, s);
    for (int k = 0; k < steps && !e; ++k)
      e = launch_fused_step(lv->m, lv->G, x, x, x, b, lv->dinv, lv->y, 0.0, omega, 0, s);
    return e;
  }
  for (int k = 0; k < steps; ++k) {
    cudaError_t e = (k == 0) ? op_apply(lv, 0, x, lv->y, s) : element_kernel(lv, 0, x, lv->y, 2, 0, s);
    if (e) return e;
    if ((e = launch_cheb_update(lv->m, x, x, x, b, lv->y, lv->dinv, 0.0, omega, s))) return e;
  }
  return cudaSuccess;
}

// Largest eigenvalue of the symmetric tridiagonal matrix (a[0..k), off-diagonal b[0..k-1)) by
// Sturm-sequence bisection (count of negative pivots of T - x I = number of eigenvalues < x).
static double tridiag_max_eig(const std::vector<double>& a, const std::vector<double>& b) {
  const int k = (int)a.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {   // Gershgorin interval
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto below = [&](double x) {
    int c = 0;
    double q = 1.0;
    for (int i = 0; i < k; ++i) {
      q = (a[i] - x) - (i > 0 ? b[i - 1] * b[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 300 && hi - lo > 4e-16 * std::max(std::fabs(lo), std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (below(mid) == k) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

// lambda_max(D^{-1} A_D) from m Arnoldi steps in the D-inner product (R26):
// modified Gram-Schmidt repeated once per step, coefficients kept on the device between kernels
// (slots 14.. of the level's scalars) and read back once per pass to accumulate H.  work: (m + 2) N.
static sfmg_status arnoldi_lambda(sfmg_level_s* lv, int m, uint64_t seed, double* work, double* lam,
                                  cudaStream_t s) {
  const long long N = lv->N;
  double* Q = work;                   // q_0 .. q_m
  double* w = work + (size_t)(m + 1) * N;
  double* sc = lv->red.scalars;
  double host[32];
  CK(launch_power_start(lv->m, seed, Q, lv->y, s));           // q_0: seeded, boundary zero (R9)
  CK(launch_dotw(lv->red, Q, Q, lv->dinv, N, 14, s));
  CK(cudaMemcpyAsync(host, sc + 14, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!(host[0] > 0.0)) { set_error("Arnoldi start vector is zero (no interior dofs)"); return SFMG_E_ARG; }
  CK(launch_scale_mul(1.0 / std::sqrt(host[0]), Q, nullptr, Q, N, s));
  std::vector<double> H((size_t)(m + 1) * m, 0.0);
  int k = 0;
  for (int j = 0; j < m; ++j) {
    double* qj = Q + (size_t)j * N;
    CK(op_apply(lv, 0, qj, lv->y, s));
    CK(launch_scale_mul(1.0, lv->y, lv->dinv, w, N, s));      // w = D^{-1} A_D q_j
    CK(launch_dotw(lv->red, w, w, lv->dinv, N, 13, s));
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i <= j; ++i) {
        CK(launch_dotw(lv->red, w, Q + (size_t)i * N, lv->dinv, N, 14 + i, s));
        CK(launch_sub_scaled_dev(lv->red, 14 + i, Q + (size_t)i * N, w, N, s));
      }
      CK(cudaMemcpyAsync(host, sc + 14, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] += host[i];
    }
    CK(launch_dotw(lv->red, w, w, lv->dinv, N, 12, s));
    CK(cudaMemcpyAsync(host, sc + 12, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double hn = std::sqrt(host[0]), wn0 = std::sqrt(host[1]);
    k = j + 1;
    H[(size_t)(j + 1) * m + j] = hn;
    if (hn <= 1e-10 * wn0) break;   // Krylov space exhausted
    CK(launch_scale_mul(1.0 / hn, w, nullptr, Q + (size_t)(j + 1) * N, N, s));
  }
  std::vector<double> a(k), b(k > 0 ? k - 1 : 0);
  for (int i = 0; i < k; ++i) a[i] = H[(size_t)i * m + i];
  for (int i = 0; i + 1 < k; ++i) b[i] = 0.5 * (H[(size_t)i * m + i + 1] + H[(size_t)(i + 1) * m + i]);
  *lam = tridiag_max_eig(a, b);
  return SFMG_OK;
}

}  // namespace sfmg

using namespace sfmg;

extern "C" {

const char* sfmg_version(void) { return "sfmg 0.1 (sm_100a, fp64)"; }
const char* sfmg_last_error(void) { return g_err.c_str(); }

sfmg_status sfmg_level_query(const sfmg_problem* prob, int64_t* n_dofs, int64_t* n_elem, size_t* ws_bytes) {
  sfmg_status st = check_problem(prob);
  if (st) return st;
  MeshDev m = make_mesh(prob);
  if (n_dofs) *n_dofs = m.N;
  if (n_elem) *n_elem = m.E;
  if (ws_bytes) *ws_bytes = level_layout(m).total;
  return SFMG_OK;
}

sfmg_status sfmg_level_create(const sfmg_problem* prob, void* d_ws, size_t ws_bytes, void* stream, sfmg_level* out) {
  sfmg_status st = check_problem(prob);
  if (st) return st;
  if (!out) { set_error("null output handle"); return SFMG_E_ARG; }
  return level_build(prob, d_ws, ws_bytes, (cudaStream_t)stream, out);
}

static void free_prof(sfmg_level_s* lv) {
  for (cudaEvent_t ev : lv->prof_ev) cudaEventDestroy(ev);
  lv->prof_ev.clear();
  lv->prof_used = 0;
  for (cudaEvent_t ev : lv->hp_ev) cudaEventDestroy(ev);
  lv->hp_ev.clear();
  if (lv->hp_h2d) cudaStreamDestroy(lv->hp_h2d);
  if (lv->hp_d2h) cudaStreamDestroy(lv->hp_d2h);
  lv->hp_h2d = lv->hp_d2h = nullptr;
  if (lv->cgc_exec) cudaGraphExecDestroy(lv->cgc_exec);
  for (cudaEvent_t& ev : lv->cgc_ev)
    if (ev) cudaEventDestroy(ev), ev = nullptr;
  if (lv->cgc_s) cudaStreamDestroy(lv->cgc_s);
  lv->cgc_exec = nullptr;
  lv->cgc_s = nullptr;
  lv->cgc_x = lv->cgc_r = nullptr;
}

sfmg_status sfmg_level_destroy(sfmg_level lv) {
  if (!lv) return SFMG_E_ARG;
  if (lv->owned_by_hier) { set_error("level is owned by a hierarchy"); return SFMG_E_ARG; }
  free_prof(lv);
  delete lv;
  return SFMG_OK;
}

sfmg_status sfmg_profile_enable(sfmg_level lv, int32_t enable) {
  if (!lv) return SFMG_E_ARG;
  lv->prof = enable != 0;
  return SFMG_OK;
}

sfmg_status sfmg_profile_read(sfmg_level lv, double* ms, int64_t* launches, int32_t reset) {
  if (!lv) return SFMG_E_ARG;
  double tot = 0.0;
  for (size_t i = 0; i + 1 < lv->prof_used; i += 2) {
    CK(cudaEventSynchronize(lv->prof_ev[i + 1]));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, lv->prof_ev[i], lv->prof_ev[i + 1]));
    tot += t;
  }
  if (ms) *ms = tot;
  if (launches) *launches = (int64_t)(lv->prof_used / 2);
  if (reset) lv->prof_used = 0;
  return SFMG_OK;
}

sfmg_status sfmg_level_info(sfmg_level lv, int64_t* n_dofs, int64_t* n_elem, int32_t* order) {
  if (!lv) return SFMG_E_ARG;
  if (n_dofs) *n_dofs = lv->N;
  if (n_elem) *n_elem = lv->E;
  if (order) *order = lv->p;
  return SFMG_OK;
}

sfmg_status sfmg_export_l2g(sfmg_level lv, int32_t* d_l2g, void* stream) {
  if (!lv || !d_l2g || lv->m.dim == 2) return SFMG_E_ARG;
  CK(launch_export_maps(lv->m, d_l2g, nullptr, nullptr, (cudaStream_t)stream));
  return SFMG_OK;
}
sfmg_status sfmg_export_mask(sfmg_level lv, uint8_t* d_mask, void* stream) {
  if (!lv || !d_mask || lv->m.dim == 2) return SFMG_E_ARG;
  CK(launch_export_maps(lv->m, nullptr, d_mask, nullptr, (cudaStream_t)stream));
  return SFMG_OK;
}
sfmg_status sfmg_export_colors(sfmg_level lv, uint8_t* d_col, void* stream) {
  if (!lv || !d_col || lv->m.dim == 2) return SFMG_E_ARG;
  CK(launch_export_maps(lv->m, nullptr, nullptr, d_col, (cudaStream_t)stream));
  return SFMG_OK;
}
sfmg_status sfmg_export_geometry(sfmg_level lv, double* d_G, void* stream) {
  if (!lv || !d_G || lv->m.dim == 2) return SFMG_E_ARG;
  CK(launch_export_geometry(lv->m, lv->G, d_G, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_apply(sfmg_level lv, int32_t bc, const double* d_u, double* d_v, int64_t n, void* stream) {
  if (!lv || !d_u || !d_v || d_u == d_v || (bc != 0 && bc != 1)) { set_error("bad argument to sfmg_apply"); return SFMG_E_ARG; }
  if (n != lv->N) { set_error("vector length != N"); return SFMG_E_ARG; }
  CK(op_apply(lv, bc, d_u, d_v, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_diag(sfmg_level lv, int32_t bc, double* d_diag, int64_t n, void* stream) {
  if (!lv || !d_diag || (bc != 0 && bc != 1)) return SFMG_E_ARG;
  if (n != lv->N) { set_error("vector length != N"); return SFMG_E_ARG; }
  CK(launch_diag(lv->m, bc, lv->G, d_diag, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_lambda_max(sfmg_level lv, int32_t iters, uint64_t seed, double* h_lambda, void* stream) {
  if (!lv || !h_lambda || iters < 1) return SFMG_E_ARG;
  if ((long long)(lv->m.Mx - 2) * (lv->m.My - 2) * (lv->m.dim == 2 ? 1 : lv->m.Mz - 2) <= 0) {
    set_error("level has no interior dofs: D^{-1} A_D is the identity on the boundary");
    return SFMG_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* x = lv->t1;
  double* y = lv->y;
  CK(launch_power_start(lv->m, seed, x, y, s));
  for (int it = 0; it < iters; ++it) {
    CK(launch_apply(lv->m, 0, lv->G, x, y, 2, 0, s));
    CK(launch_power_step(lv->m, lv->red, x, y, lv->dinv, s));
  }
  CK(cudaMemcpyAsync(h_lambda, lv->red.scalars + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SFMG_OK;
}

sfmg_status sfmg_cheb(sfmg_level lv, const double* d_b, double* d_x, int64_t n, int32_t degree, double lam_lo,
                      double lam_hi, void* stream) {
  if (!lv || !d_b || !d_x || d_b == d_x || degree < 1 || !(lam_hi > lam_lo) || !(lam_lo > 0.0)) {
    set_error("bad argument to sfmg_cheb (b and x must be distinct vectors)");
    return SFMG_E_ARG;
  }
  if (n != lv->N) { set_error("vector length != N"); return SFMG_E_ARG; }
  CK(op_cheb(lv, d_b, d_x, degree, lam_lo, lam_hi, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_lambda_arnoldi(sfmg_level lv, int32_t steps, uint64_t seed, double* d_work, double* h_lambda,
                                void* stream) {
  if (!lv || !h_lambda || !d_work || steps < 1 || steps > 16) {
    set_error("bad argument to sfmg_lambda_arnoldi (steps 1..16, work of (steps + 2) N doubles)");
    return SFMG_E_ARG;
  }
  return arnoldi_lambda(lv, steps, seed, d_work, h_lambda, (cudaStream_t)stream);
}

sfmg_status sfmg_jacobi(sfmg_level lv, const double* d_b, double* d_x, int64_t n, int32_t steps, double omega,
                        void* stream) {
  if (!lv || !d_b || !d_x || d_b == d_x || steps < 0 || !(omega > 0.0 && omega < 2.0)) {
    set_error("bad argument to sfmg_jacobi");
    return SFMG_E_ARG;
  }
  if (n != lv->N) { set_error("vector length != N"); return SFMG_E_ARG; }
  CK(op_jacobi(lv, d_b, d_x, steps, omega, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_load_vector(sfmg_level lv, int32_t rhs_id, double* d_f, int64_t n, void* stream) {
  if (!lv || !d_f || rhs_id != 1) return SFMG_E_ARG;
  if (n != lv->N) return SFMG_E_ARG;
  CK(launch_load(lv->m, rhs_id, d_f, (cudaStream_t)stream));
  return SFMG_OK;
}

// Host-buffer apply, pipelined over z-slabs of element layers: the H2D copy of slab c+1, the
// kernels of slab c and the D2H copy of slab c-1 overlap (copy engines in both directions + SMs).
// Slab c = element layers [L_c, L_{c+1}) reads u planes [L_c p, L_{c+1} p] and adds into the same
// v planes; its kernels run on a z-slab view of the lattice whose cut planes are not Dirichlet
// planes (MeshDev::Kb0/Kb1).  v plane L_{c+1} p also receives slab c+1, so slab c ships v planes
// [L_c p, L_{c+1} p) after its kernels and the last slab the rest.  Same arithmetic as sfmg_apply.
static constexpr int kHostChunks = 8;

static int host_chunks(const sfmg_level_s* lv) {
  if (lv->m.quad || lv->m.dim == 2) return 1;
  if (lv->p <= 2 && ((long long)lv->m.nex * lv->m.ney) % 32 != 0) return 1;   // interleaved G blocks of 32
  if (lv->hp_slabs > 0) return std::min(std::min(lv->hp_slabs, kHostChunks), lv->m.nez);
  const long long plane_bytes = (long long)lv->m.Mx * lv->m.My * 8;
  long long S = std::min<long long>(lv->m.nez, kHostChunks);
  S = std::min<long long>(S, std::max<long long>(1, plane_bytes * lv->m.Mz / (1 << 20)));   // >= ~1 MB per slab
  return (int)std::max<long long>(S, 1);
}

static cudaError_t host_pipe_ready(sfmg_level_s* lv) {
  cudaError_t e;
  if (!lv->hp_h2d && (e = cudaStreamCreateWithFlags(&lv->hp_h2d, cudaStreamNonBlocking))) return e;
  if (!lv->hp_d2h && (e = cudaStreamCreateWithFlags(&lv->hp_d2h, cudaStreamNonBlocking))) return e;
  while (lv->hp_ev.size() < 1 + 3 * (size_t)kHostChunks) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return e;
    lv->hp_ev.push_back(ev);
  }
  return cudaSuccess;
}

// z-slab view of planes [K0, K0 + planes) (Kb0/Kb1 keep only the true boundary planes)
static MeshDev slab_view(const MeshDev& m, int K0, int planes, int nez) {
  MeshDev v = m;
  v.nez = nez;
  v.Mz = planes;
  v.E = (long long)m.nex * m.ney * nez;
  v.N = (long long)m.Mx * m.My * planes;
  v.Kb0 = (K0 == 0) ? 0 : -1;
  v.Kb1 = (K0 + planes == m.Mz) ? planes - 1 : -1;
  return v;
}

sfmg_status sfmg_apply_host(sfmg_level lv, int32_t bc, const double* h_u, double* h_v, int64_t n, void* stream) {
  if (!lv || !h_u || !h_v || (bc != 0 && bc != 1)) return SFMG_E_ARG;
  if (n != lv->N) return SFMG_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * lv->N;
  const int S = host_chunks(lv);
  if (S <= 1) {
    CK(cudaMemcpyAsync(lv->t1, h_u, bytes, cudaMemcpyHostToDevice, s));
    CK(op_apply(lv, bc, lv->t1, lv->t2, s));
    CK(cudaMemcpyAsync(h_v, lv->t2, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return SFMG_OK;
  }
  CK(host_pipe_ready(lv));
  const MeshDev& m = lv->m;
  const int p = lv->p;
  const long long sxy = (long long)m.Mx * m.My;
  const long long n3 = lv->n3;
  int L[kHostChunks + 1];
  for (int c = 0; c <= S; ++c) L[c] = (int)((long long)m.nez * c / S);
  cudaEvent_t* ev = lv->hp_ev.data();
  CK(cudaEventRecord(ev[0], s));   // the copies start after the caller's prior work on s
  CK(cudaStreamWaitEvent(lv->hp_h2d, ev[0], 0));
  CK(cudaStreamWaitEvent(lv->hp_d2h, ev[0], 0));
  for (int c = 0; c < S; ++c) {   // H2D: u planes not yet on the device
    const long long k0 = (c == 0) ? 0 : (long long)L[c] * p + 1, k1 = (long long)L[c + 1] * p;
    CK(cudaMemcpyAsync(lv->t1 + k0 * sxy, h_u + k0 * sxy, sizeof(double) * (k1 - k0 + 1) * sxy,
                       cudaMemcpyHostToDevice, lv->hp_h2d));
    CK(cudaEventRecord(ev[1 + 3 * c], lv->hp_h2d));
  }
  for (int c = 0; c < S; ++c) {   // kernels of slab c on the caller's stream
    CK(cudaStreamWaitEvent(s, ev[1 + 3 * c], 0));
    const int K0 = L[c] * p, K1 = L[c + 1] * p;
    const int i0 = (c == 0) ? 0 : K0 + 1;   // plane K0 was initialised (and partly summed) by slab c-1
    const MeshDev mi = slab_view(m, i0, K1 - i0 + 1, L[c + 1] - L[c]);
    const MeshDev ma = slab_view(m, K0, K1 - K0 + 1, L[c + 1] - L[c]);
    const double* Ga = lv->G + (long long)L[c] * m.nex * m.ney * 6 * n3;
    if (p <= 2) {
      CK(cudaMemsetAsync(lv->t2 + i0 * sxy, 0, sizeof(double) * (K1 - i0 + 1) * sxy, s));
      CK(launch_apply(ma, bc, Ga, lv->t1 + K0 * sxy, lv->t2 + K0 * sxy, 1, 1, s));
    } else {
      CK(launch_init(mi, bc, lv->t1 + i0 * sxy, 0.0, lv->t2 + i0 * sxy, s));
      CK(launch_apply(ma, bc, Ga, lv->t1 + K0 * sxy, lv->t2 + K0 * sxy, 1, 0, s));
    }
    CK(cudaEventRecord(ev[2 + 3 * c], s));
  }
  for (int c = 0; c < S; ++c) {   // D2H: v planes complete after slab c
    const long long k0 = (c == 0) ? 0 : (long long)L[c] * p, k1 = (c == S - 1) ? m.Mz : (long long)L[c + 1] * p;
    CK(cudaStreamWaitEvent(lv->hp_d2h, ev[2 + 3 * c], 0));
    CK(cudaMemcpyAsync(h_v + k0 * sxy, lv->t2 + k0 * sxy, sizeof(double) * (k1 - k0) * sxy, cudaMemcpyDeviceToHost,
                       lv->hp_d2h));
    CK(cudaEventRecord(ev[3 + 3 * c], lv->hp_d2h));
  }
  CK(cudaStreamWaitEvent(s, ev[3 + 3 * (S - 1)], 0));
  CK(cudaStreamSynchronize(s));
  return SFMG_OK;
}

sfmg_status sfmg_host_pipeline(sfmg_level lv, int32_t slabs) {
  if (!lv || slabs < 0) return SFMG_E_ARG;
  lv->hp_slabs = slabs;
  return SFMG_OK;
}

sfmg_status sfmg_cheb_host(sfmg_level lv, const double* h_b, double* h_x, int64_t n, int32_t degree, double lam_lo,
                           double lam_hi, void* stream) {
  if (!lv || !h_b || !h_x || degree < 1 || !(lam_hi > lam_lo) || !(lam_lo > 0.0)) return SFMG_E_ARG;
  if (n != lv->N) return SFMG_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * lv->N;
  CK(cudaMemcpyAsync(lv->t1, h_b, bytes, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(lv->t2, h_x, bytes, cudaMemcpyHostToDevice, s));
  CK(op_cheb(lv, lv->t1, lv->t2, degree, lam_lo, lam_hi, s));
  CK(cudaMemcpyAsync(h_x, lv->t2, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SFMG_OK;
}

// 1: p pair (fine.p = 2 coarse.p <= 16, same element grid); 2: h pair (same p, fine ne = 2 coarse ne;
// p = 1: NEXT-1 trilinear gathers, p > 1: NEXT-4 high-order h-transfer)
static int pair_kind(const MeshDev& c, const MeshDev& f) {
  if (c.dim != f.dim) return 0;
  const bool two = f.dim == 2;
  if (f.p == 2 * c.p && c.p <= 8 && f.nex == c.nex && f.ney == c.ney && f.nez == c.nez) return 1;
  if (c.p == f.p && f.nex == 2 * c.nex && f.ney == 2 * c.ney && (two || f.nez == 2 * c.nez)) return 2;
  return 0;
}

static sfmg_status check_pair(sfmg_level c, sfmg_level f, int* kind) {
  if (!c || !f) return SFMG_E_ARG;
  *kind = pair_kind(c->m, f->m);
  if (!*kind) {
    set_error("levels are neither (p/2, p) on one element grid nor (ne/2, ne) at one order");
    return SFMG_E_PCOARSEN;
  }
  return SFMG_OK;
}

static cudaError_t transfer_prolong(const MeshDev& c, const MeshDev& f, const double* uc, double* uf, int add,
                                    cudaStream_t s) {
  if (f.dim == 2) return launch_transfer_2d(c, f, pair_kind(c, f), 0, uc, uf, add, s);
  if (pair_kind(c, f) == 2)
    return f.p == 1 ? launch_prolong_h(c, f, uc, uf, add, s) : launch_prolong_hp(c, f, uc, uf, add, s);
  return launch_prolong(c, f, uc, uf, add, s);
}
static cudaError_t transfer_restrict(const MeshDev& c, const MeshDev& f, const double* rf, double* rc,
                                     cudaStream_t s) {
  if (f.dim == 2) return launch_transfer_2d(c, f, pair_kind(c, f), 1, rf, rc, 0, s);
  if (pair_kind(c, f) == 2) return f.p == 1 ? launch_restrict_h(c, f, rf, rc, s) : launch_restrict_hp(c, f, rf, rc, s);
  return launch_restrict(c, f, rf, rc, s);
}

sfmg_status sfmg_prolong(sfmg_level coarse, sfmg_level fine, const double* d_uc, double* d_uf, void* stream) {
  int kind = 0;
  sfmg_status st = check_pair(coarse, fine, &kind);
  if (st) return st;
  if (!d_uc || !d_uf) return SFMG_E_ARG;
  if (kind == 1) CK(upload_interp_tables(coarse->p, (cudaStream_t)stream));
  CK(transfer_prolong(coarse->m, fine->m, d_uc, d_uf, 0, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_restrict(sfmg_level coarse, sfmg_level fine, const double* d_rf, double* d_rc, void* stream) {
  int kind = 0;
  sfmg_status st = check_pair(coarse, fine, &kind);
  if (st) return st;
  if (!d_rf || !d_rc) return SFMG_E_ARG;
  if (kind == 1) CK(upload_interp_tables(coarse->p, (cudaStream_t)stream));
  CK(transfer_restrict(coarse->m, fine->m, d_rf, d_rc, (cudaStream_t)stream));
  return SFMG_OK;
}

// ------------------------------------------------------------------------------ hierarchy

// Level problems of the hierarchy: orders p, p/2, ..., 1 on the fine mesh, then
// mg->h_levels p = 1 levels on meshes ne/2, ne/4, ....  mg->coarsen = 1
// (NEXT-4, high-order h-multigrid): order p on meshes ne, ne/2, ..., ne/2^h_levels.
static sfmg_status hier_specs(const sfmg_problem* fine, const sfmg_mg_params* mg, std::vector<sfmg_problem>& out) {
  out.clear();
  for (int q = fine->order;; q /= 2) {
    sfmg_problem pr = *fine;
    pr.order = q;
    out.push_back(pr);
    if (q == 1 || mg->coarsen == 1) break;
    if (q % 2) { set_error("order cannot be p-coarsened to 1 by halving"); return SFMG_E_PCOARSEN; }
  }
  for (int j = 1; j <= mg->h_levels; ++j) {
    sfmg_problem pr = out.back();
    const bool two = pr.dim == 2;
    if (pr.nex % 2 || pr.ney % 2 || (!two && pr.nez % 2)) {
      set_error("mesh cannot be h-coarsened h_levels times (element counts must be divisible by 2^h_levels)");
      return SFMG_E_PCOARSEN;
    }
    pr.nex /= 2; pr.ney /= 2;
    if (!two) pr.nez /= 2;
    out.push_back(pr);
  }
  return SFMG_OK;
}

static sfmg_status check_mg(const sfmg_mg_params* mg) {
  if (!mg || mg->nu_pre < 0 || mg->nu_post < 0 || mg->cheb_degree < 1 || !(mg->eig_hi_frac > mg->eig_lo_frac) ||
      !(mg->eig_lo_frac > 0) || mg->power_iters < 1 || !(mg->coarse_rtol > 0) || mg->coarse_max_iter < 1 ||
      (mg->smoother != 0 && mg->smoother != 1) || (mg->smoother == 1 && !(mg->jacobi_omega > 0 && mg->jacobi_omega < 2)) ||
      (mg->lambda_method != 0 && mg->lambda_method != 1) || (mg->lambda_method == 1 && mg->power_iters > 16) ||
      mg->h_levels < 0 || mg->h_levels > 20 || (mg->coarsen != 0 && mg->coarsen != 1) ||
      (mg->coarsen == 1 && mg->h_levels < 1)) {
    set_error("bad multigrid parameters");
    return SFMG_E_ARG;
  }
  return SFMG_OK;
}

sfmg_status sfmg_hier_query(const sfmg_problem* fine, const sfmg_mg_params* mg, size_t* ws_bytes) {
  sfmg_status st = check_problem(fine);
  if (st) return st;
  if ((st = check_mg(mg))) return st;
  std::vector<sfmg_problem> specs;
  if ((st = hier_specs(fine, mg, specs))) return st;
  size_t total = 0;
  for (size_t l = 0; l < specs.size(); ++l) {
    MeshDev m = make_mesh(&specs[l]);
    total += level_layout(m).total + 3 * align_up(sizeof(double) * m.N);
    if (l == 0) total += 4 * align_up(sizeof(double) * m.N);
    if (l == 0 && mg->lambda_method == 1) total += align_up(sizeof(double) * (size_t)(mg->power_iters + 2) * m.N);
  }
  if (ws_bytes) *ws_bytes = total;
  return SFMG_OK;
}

sfmg_status sfmg_hier_destroy(sfmg_hier h) {
  if (!h) return SFMG_E_ARG;
  for (sfmg_level_s* lv : h->lv) {
    free_prof(lv);
    delete lv;
  }
  if (h->vc_exec) cudaGraphExecDestroy(h->vc_exec);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  delete h;
  return SFMG_OK;
}

sfmg_status sfmg_hier_create(const sfmg_problem* fine, const sfmg_mg_params* mg, void* d_ws, size_t ws_bytes,
                             void* stream, sfmg_hier* out) {
  size_t need = 0;
  sfmg_status st = sfmg_hier_query(fine, mg, &need);
  if (st) return st;
  if (!out) return SFMG_E_ARG;
  if (!d_ws || ((uintptr_t)d_ws & 255) || ws_bytes < need) { set_error("workspace too small"); return SFMG_E_WORKSPACE; }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<sfmg_problem> specs;
  hier_specs(fine, mg, specs);
  sfmg_hier_s* h = new sfmg_hier_s();
  h->mg = *mg;
  h->fine_applies = 0;
  char* base = (char*)d_ws;
  double* arn_work = nullptr;
  for (size_t l = 0; l < specs.size(); ++l) {
    const sfmg_problem& q = specs[l];
    MeshDev m = make_mesh(&q);
    LevelLayout L = level_layout(m);
    sfmg_level_s* lv = nullptr;
    st = level_build(&q, base, L.total, s, &lv);
    if (st) { sfmg_hier_destroy(h); return st; }
    lv->owned_by_hier = true;
    h->lv.push_back(lv);
    base += L.total;
    const size_t vb = align_up(sizeof(double) * m.N);
    h->b.push_back((double*)base); base += vb;
    h->x.push_back((double*)base); base += vb;
    h->r.push_back((double*)base); base += vb;
    if (l == 0) {
      h->pr = (double*)base; base += vb;
      h->pz = (double*)base; base += vb;
      h->pp = (double*)base; base += vb;
      h->ph = (double*)base; base += vb;
      if (mg->lambda_method == 1) {
        arn_work = (double*)base;
        base += align_up(sizeof(double) * (size_t)(mg->power_iters + 2) * m.N);
      }
    }
    if (l + 1 < specs.size() && specs[l + 1].order * 2 == q.order) {
      cudaError_t e = upload_interp_tables(q.order / 2, s);
      if (e) { sfmg_hier_destroy(h); return cuda_fail(e, "interp tables"); }
    }
    if (l + 1 < specs.size() && specs[l + 1].order == q.order && q.order > 1) {
      cudaError_t e = upload_h_tables(q.order);
      if (e) { sfmg_hier_destroy(h); return cuda_fail(e, "h tables"); }
    }
  }
  {
    const MeshDev& mc = h->lv.back()->m;
    h->host_coarse = !((mc.p == 1 || mc.p == 2)) || mc.dim == 2;   // single-CTA device CG: 3-D, p <= 2
  }
  h->lam.assign(h->lv.size(), 0.0);
  for (size_t l = 0; l + 1 < h->lv.size(); ++l) {
    double lam = 0.0;
    st = (mg->lambda_method == 1) ? arnoldi_lambda(h->lv[l], mg->power_iters, mg->power_seed, arn_work, &lam, s)
                                  : sfmg_lambda_max(h->lv[l], mg->power_iters, mg->power_seed, &lam, stream);
    if (st) { sfmg_hier_destroy(h); return st; }
    h->lam[l] = lam;
  }
  *out = h;
  return SFMG_OK;
}

sfmg_status sfmg_hier_info(sfmg_hier h, int32_t* n_levels, int64_t* n_dofs_fine) {
  if (!h) return SFMG_E_ARG;
  if (n_levels) *n_levels = (int32_t)h->lv.size();
  if (n_dofs_fine) *n_dofs_fine = h->lv[0]->N;
  return SFMG_OK;
}

sfmg_status sfmg_hier_level(sfmg_hier h, int32_t l, sfmg_level* out) {
  if (!h || !out || l < 0 || l >= (int32_t)h->lv.size()) return SFMG_E_ARG;
  *out = h->lv[l];
  return SFMG_OK;
}

sfmg_status sfmg_hier_lambda(sfmg_hier h, int32_t l, double* lam) {
  if (!h || !lam || l < 0 || l >= (int32_t)h->lv.size()) return SFMG_E_ARG;
  *lam = h->lam[l];
  return SFMG_OK;
}

}  // extern "C"

namespace sfmg {

// Coarse solve of a level whose order is > 2 (high-order h-multigrid, NEXT-4): unpreconditioned CG
// (R13) on the level's own apply and reduction kernels, x0 = 0, ||r|| <= rtol ||b||.  Convergence is
// decided on the device after every iteration (a flag then freezes x, r, p); the iterations are
// queued in batches of kCgcBatch and the host reads the flag between batches (syncs).
static constexpr int kCgcBatch = 8;

static cudaError_t coarse_cg_any(sfmg_level_s* lv, const double* b, double* x, double* r, double rtol, int maxit,
                                 cudaStream_t s) {
  const long long N = lv->N;
  double* p = lv->t0;
  double* q = lv->t1;
  cudaError_t e;
  if ((e = cudaMemsetAsync(x, 0, sizeof(double) * N, s))) return e;
  if ((e = launch_copy(b, r, N, s))) return e;
  if ((e = launch_copy(b, p, N, s))) return e;
  if ((e = launch_dot(lv->red, b, b, N, kCgcBB, s))) return e;
  if ((e = launch_cgc_start(lv->red, s))) return e;
  double flag = 0.0;
  auto batch = [&](cudaStream_t st) -> cudaError_t {
    cudaError_t be;
    for (int k = 0; k < kCgcBatch; ++k) {
      if ((be = op_apply(lv, 0, p, q, st))) return be;
      if ((be = launch_dot(lv->red, p, q, N, kCgcPQ, st))) return be;
      if ((be = launch_cgc_iter_tail(lv->red, x, r, p, q, N, rtol, maxit, st))) return be;
    }
    return cudaSuccess;
  };
  // a batch is ~6 small kernels per iteration on a small level: replay it as one captured graph on the
  // level's own stream (the caller's stream may be the legacy one, which cannot be captured)
  static const bool no_graph = getenv("SFMG_NO_GRAPH") && getenv("SFMG_NO_GRAPH")[0] == '1';
  bool use_graph = !no_graph && !lv->prof;
  if (use_graph && (!lv->cgc_exec || lv->cgc_x != x || lv->cgc_r != r || lv->cgc_rtol != rtol ||
                    lv->cgc_maxit != maxit)) {
    if (!lv->cgc_s && (e = cudaStreamCreateWithFlags(&lv->cgc_s, cudaStreamNonBlocking))) return e;
    for (cudaEvent_t& ev : lv->cgc_ev)
      if (!ev && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return e;
    if (lv->cgc_exec) {
      cudaGraphExecDestroy(lv->cgc_exec);
      lv->cgc_exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    if ((e = cudaStreamBeginCapture(lv->cgc_s, cudaStreamCaptureModeThreadLocal))) return e;
    const cudaError_t ce = batch(lv->cgc_s);
    const cudaError_t ee = cudaStreamEndCapture(lv->cgc_s, &g);
    if (ce || ee) {
      if (g) cudaGraphDestroy(g);
      return ce ? ce : ee;
    }
    e = cudaGraphInstantiate(&lv->cgc_exec, g, 0);
    cudaGraphDestroy(g);
    if (e) return e;
    lv->cgc_x = x;
    lv->cgc_r = r;
    lv->cgc_rtol = rtol;
    lv->cgc_maxit = maxit;
  }
  for (int it = 0; it < maxit; it += kCgcBatch) {
    if (use_graph) {
      if ((e = cudaEventRecord(lv->cgc_ev[0], s))) return e;
      if ((e = cudaStreamWaitEvent(lv->cgc_s, lv->cgc_ev[0], 0))) return e;
      if ((e = cudaGraphLaunch(lv->cgc_exec, lv->cgc_s))) return e;
      if ((e = cudaEventRecord(lv->cgc_ev[1], lv->cgc_s))) return e;
      if ((e = cudaStreamWaitEvent(s, lv->cgc_ev[1], 0))) return e;
    } else if ((e = batch(s))) {
      return e;
    }
    if ((e = cudaMemcpyAsync(&flag, lv->red.scalars + kCgcFlag, sizeof(double), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if (flag != 0.0) break;
  }
  return cudaSuccess;
}

static cudaError_t vcycle_level(sfmg_hier_s* h, size_t l, const double* b, double* x, cudaStream_t s) {
  sfmg_level_s* lv = h->lv[l];
  const sfmg_mg_params& mg = h->mg;
  cudaError_t e;
  if (l + 1 == h->lv.size()) {
    if (h->host_coarse) return coarse_cg_any(lv, b, x, h->r[l], mg.coarse_rtol, mg.coarse_max_iter, s);
    return launch_coarse_cg(lv->m, lv->G, b, x, lv->t0, lv->t1, lv->y, lv->red.scalars, mg.coarse_rtol,
                            mg.coarse_max_iter, s);
  }
  const double lo = mg.eig_lo_frac * h->lam[l], hi = mg.eig_hi_frac * h->lam[l];
  // one smoothing application: a degree-K Chebyshev polynomial or one damped Jacobi step
  auto smooth = [&]() -> cudaError_t {
    if (mg.smoother == 1) {
      if (l == 0) h->fine_applies += 1;
      return op_jacobi(lv, b, x, 1, mg.jacobi_omega, s);
    }
    if (l == 0) h->fine_applies += mg.cheb_degree;
    return op_cheb(lv, b, x, mg.cheb_degree, lo, hi, s);
  };
  if ((e = cudaMemsetAsync(x, 0, sizeof(double) * lv->N, s))) return e;
  for (int i = 0; i < mg.nu_pre; ++i)
    if ((e = smooth())) return e;
  if ((e = op_apply(lv, 0, x, lv->y, s))) return e;
  if (l == 0) h->fine_applies += 1;
  if ((e = launch_residual(b, lv->y, h->r[l], lv->N, s))) return e;
  sfmg_level_s* c = h->lv[l + 1];
  if ((e = transfer_restrict(c->m, lv->m, h->r[l], h->b[l + 1], s))) return e;
  if ((e = vcycle_level(h, l + 1, h->b[l + 1], h->x[l + 1], s))) return e;
  if ((e = transfer_prolong(c->m, lv->m, h->x[l + 1], x, 1, s))) return e;
  for (int i = 0; i < mg.nu_post; ++i)
    if ((e = smooth())) return e;
  return cudaSuccess;
}

// The V-cycle is a fixed sequence of ~10^2 small launches (most levels are latency-bound), so it is
// replayed as a CUDA graph: the first call per (b, x) pair runs eagerly (it also completes every lazy
// per-kernel setup), the second captures the sequence on a private stream (relaxed mode) and every
// later call launches the instantiated graph on the caller's stream.  SFMG_NO_GRAPH=1 disables it.
static cudaError_t vcycle(sfmg_hier_s* h, const double* b, double* x, cudaStream_t s) {
  static const bool no_graph = getenv("SFMG_NO_GRAPH") && getenv("SFMG_NO_GRAPH")[0] == '1';
  bool prof = false;   // per-launch event timing (sfmg_profile_*) cannot be recorded inside a capture
  for (const sfmg_level_s* L : h->lv) prof = prof || L->prof;
  if (no_graph || h->host_coarse || prof) return vcycle_level(h, 0, b, x, s);   // eager
  if (h->vc_exec && h->vc_b == b && h->vc_x == x) {
    h->fine_applies += h->vc_fine_applies;
    return cudaGraphLaunch(h->vc_exec, s);
  }
  if (h->vc_b != b || h->vc_x != x) {
    h->vc_b = b;
    h->vc_x = x;
    h->vc_eager_runs = 0;
    if (h->vc_exec) {
      cudaGraphExecDestroy(h->vc_exec);
      h->vc_exec = nullptr;
    }
  }
  if (h->vc_eager_runs < 1) {
    ++h->vc_eager_runs;
    return vcycle_level(h, 0, b, x, s);
  }
  cudaError_t e;
  if (!h->cap_stream && (e = cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking))) return e;
  // order the capture after the caller's pending work: the graph itself is launched on s below
  const int64_t fa0 = h->fine_applies;
  if ((e = cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeRelaxed))) return e;
  cudaError_t ev = vcycle_level(h, 0, b, x, h->cap_stream);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(h->cap_stream, &graph);
  if (ev) { if (graph) cudaGraphDestroy(graph); return ev; }
  if (e) return e;
  h->vc_fine_applies = h->fine_applies - fa0;
  h->fine_applies = fa0;
  e = cudaGraphInstantiate(&h->vc_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e) return e;
  h->fine_applies += h->vc_fine_applies;
  return cudaGraphLaunch(h->vc_exec, s);
}

}  // namespace sfmg

extern "C" {

sfmg_status sfmg_vcycle(sfmg_hier h, const double* d_b, double* d_x, void* stream) {
  if (!h || !d_b || !d_x || d_b == d_x) return SFMG_E_ARG;
  CK(vcycle(h, d_b, d_x, (cudaStream_t)stream));
  return SFMG_OK;
}

sfmg_status sfmg_solve(sfmg_hier h, int32_t mode, const double* d_b, double* d_x, double rtol, int32_t max_iter,
                       sfmg_report* rep, void* stream) {
  if (!h || !d_b || !d_x || (mode != 0 && mode != 1) || !(rtol > 0) || max_iter < 0) return SFMG_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  sfmg_level_s* lv = h->lv[0];
  const long long N = lv->N;
  double* sc = lv->red.scalars;
  h->fine_applies = 0;
  int64_t vcycles = 0;
  CK(cudaMemsetAsync(d_x, 0, sizeof(double) * N, s));
  CK(cudaMemcpyAsync(h->pr, d_b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  CK(launch_dot(lv->red, h->pr, h->pr, N, 7, s));
  double host[2] = {0, 0};
  CK(cudaMemcpyAsync(host, sc + 7, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const double r0 = std::sqrt(host[0]);
  double rn = r0;
  int it = 0, converged = 0;
  sfmg_status result = SFMG_OK;
  if (rep && rep->history && rep->history_cap > 0) rep->history[0] = r0;
  if (r0 == 0.0) {
    converged = 1;
  } else if (mode == 0) {
    while (it < max_iter) {
      if (rn <= rtol * r0) { converged = 1; break; }
      if (rn > 10.0 * r0) break;
      CK(vcycle(h, h->pr, h->pz, s));
      ++vcycles;
      CK(launch_axpy1(d_x, h->pz, N, s));
      CK(op_apply(lv, 0, d_x, h->ph, s));
      h->fine_applies += 1;
      CK(launch_residual(d_b, h->ph, h->pr, N, s));
      CK(launch_dot(lv->red, h->pr, h->pr, N, 7, s));
      CK(cudaMemcpyAsync(host, sc + 7, sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      rn = std::sqrt(host[0]);
      ++it;
      if (rep && rep->history && it < rep->history_cap) rep->history[it] = rn;
    }
    if (rn <= rtol * r0) converged = 1;
  } else {
    // Algorithm 1 with slots: 12/13 rho_r (alternating), 6 (p,h), 7 |r|^2
    int sa = 12, sb = 13;
    CK(vcycle(h, h->pr, h->pz, s));
    ++vcycles;
    CK(launch_copy(h->pz, h->pp, N, s));
    CK(launch_dot(lv->red, h->pz, h->pr, N, sa, s));
    while (it < max_iter) {
      CK(op_apply(lv, 0, h->pp, h->ph, s));                       // h = A p
      h->fine_applies += 1;
      CK(launch_dot(lv->red, h->pp, h->ph, N, 6, s));              // (p, h)
      CK(launch_pcg_xr(lv->red, d_x, h->pr, h->pp, h->ph, sa, 6, 7, N, s));  // u += a p, r -= a h
      CK(cudaMemcpyAsync(host, sc + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      ++it;
      if (!(host[0] > 0.0)) { result = SFMG_E_BREAKDOWN; set_error("(p, A p) <= 0 in CG"); break; }
      rn = std::sqrt(host[1]);
      if (rep && rep->history && it < rep->history_cap) rep->history[it] = rn;
      if (rn <= rtol * r0) { converged = 1; break; }                // convergence test
      if (rn > 10.0 * r0) break;
      CK(vcycle(h, h->pr, h->pz, s));                     // rho = M r
      ++vcycles;
      CK(launch_dot(lv->red, h->pz, h->pr, N, sb, s));             // (rho, r)
      CK(launch_pcg_p(lv->red, h->pp, h->pz, sb, sa, N, s));       // p = rho + beta p
      std::swap(sa, sb);
    }
  }
  if (rep) {
    rep->iterations = it;
    rep->converged = converged;
    rep->r0_norm = r0;
    rep->r_norm = rn;
    rep->fine_applies = h->fine_applies;
    rep->vcycles = vcycles;
  }
  return result;
}

}  // extern "C"
