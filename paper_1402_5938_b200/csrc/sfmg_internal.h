// Internal declarations of libsfmg (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "sfmg.h"

namespace sfmg {

constexpr int kMaxOrder = 16;
constexpr int kRedBlocks = 592;   // 4 x 148 SMs: fixed grid of the deterministic reductions
constexpr int kRedSlots = 4;      // partial sums per reduction pass
// scalar slots of the general (flag-gated) coarse CG
constexpr int kCgcBB = 20, kCgcRho = 21, kCgcPQ = 22, kCgcRn = 23, kCgcBeta = 24, kCgcFlag = 25, kCgcIt = 26;

// Per-device lazy state.  __constant__ tables, kernel attributes and occupancy figures exist once per
// device (CUDA context), so every "done" flag and cached number is keyed by the ordinal of the calling
// thread's current device, and first-time work runs under a mutex (thread-safe; a level built on a
// second GPU of the same process uploads its own tables).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
// f() -> cudaError_t runs until it first succeeds on each device
struct OncePerDevice {
  std::mutex mu;
  std::atomic<bool> done[kMaxDevices] = {};
  template <class F>
  cudaError_t run(F f) {
    const int d = current_device();
    if (done[d].load(std::memory_order_acquire)) return cudaSuccess;
    std::lock_guard<std::mutex> g(mu);
    if (done[d].load(std::memory_order_relaxed)) return cudaSuccess;
    cudaError_t e = f();
    if (e == cudaSuccess) done[d].store(true, std::memory_order_release);
    return e;
  }
};
// an int computed once per device by f(int& out) -> cudaError_t (occupancy, SM counts)
struct IntPerDevice {
  std::mutex mu;
  std::atomic<int> val[kMaxDevices] = {};
  template <class F>
  cudaError_t get(int& out, F f) {
    const int d = current_device();
    out = val[d].load(std::memory_order_acquire);
    if (out) return cudaSuccess;
    std::lock_guard<std::mutex> g(mu);
    out = val[d].load(std::memory_order_relaxed);
    if (out) return cudaSuccess;
    int v = 0;
    cudaError_t e = f(v);
    if (e) return e;
    if (v < 1) v = 1;
    val[d].store(v, std::memory_order_release);
    out = v;
    return cudaSuccess;
  }
};
inline int num_sms() {
  static IntPerDevice cache;
  int n = 0;
  cache.get(n, [](int& v) { return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device()); });
  return n;
}

// Mesh + problem description passed by value to kernels.
struct MeshDev {
  int nex, ney, nez, p;
  int Mx, My, Mz;          // lattice sizes (nex p + 1, ...)
  long long E, N;          // elements, dofs
  int warp, coeff;
  double amp, c0, c1;
  int quad;                // 0 collocated LGL quadrature, 1 Gauss-Legendre (NEXT-3)
  // lattice planes K that lie on the Dirichlet boundary z = 0 / z = 1: 0 and Mz - 1 for a whole
  // mesh; a z-slab view (pipelined host apply) marks an interior cut plane with -1.  Used by the
  // apply and init kernels only.
  int Kb0, Kb1;
  int dim = 3;             // 3 hexahedra; 2 quadrilaterals (NEXT-2: nez = 1, Mz = 1, Kb0 = Kb1 = -1)
  int pdl_early = 0;       // set per launch: early programmatic-dependent triggers (small vectors)
};

// Device reduction scratch: partials[kRedBlocks][kRedSlots], scalars[32], counter.
struct RedScratch {
  double* partials;
  double* scalars;
  unsigned int* counter;
};

// 1-D tables of one order (host), sizes n, n*n.
struct Basis1D {
  int p = 0, n = 0;
  std::vector<double> x, w, D;   // D[i*n+m] = ell_m'(x_i)
};
Basis1D make_basis(int p);
// I[i*(pc+1)+a] = ell^{pc}_a(x^{pf}_i)
std::vector<double> make_interp(int pc, int pf);
// 1-D quadrature tables (k_gauss.cu): LGL nodes xn; B[i*n+a] = ell_a(q_i), DB = ell_a'(q_i), weights qw
// at the quadrature points q (quad 0: the LGL nodes themselves, quad 1: Gauss-Legendre)
void quad_tables_1d(int p, int quad, std::vector<double>& xn, std::vector<double>& B, std::vector<double>& DB,
                    std::vector<double>& qw);
// h-transfer at order p, child s in {0, 1}: H[i*(p+1)+a] = ell_a((xhat_i + 2 s - 1) / 2)
std::vector<double> make_h_interp(int p, int s);

}  // namespace sfmg

struct sfmg_level_s {
  sfmg_problem prob;
  sfmg::MeshDev m;
  int p, n;
  long long n3, E, N;
  // views into the caller's workspace
  double* G;       // [E][6][n3]
  double* dinv;    // [N] 1/diag(A_D)
  double* y;       // [N] operator output scratch
  double* t0;      // [N] scratch (Chebyshev previous iterate, host-variant staging)
  double* t1;      // [N] scratch (power iterate, host-variant staging)
  double* t2;      // [N] scratch (host-variant staging)
  sfmg::RedScratch red;
  int* bad;        // geometry check counter
  size_t ws_bytes;
  bool owned_by_hier;
  // benchmark timing of the element kernel (sfmg_profile_*): event pairs recorded around launches
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;   // [2 * launches]
  size_t prof_used = 0;
  // pipelined host-buffer apply (sfmg_apply_host): copy streams and per-chunk events, made lazily
  cudaStream_t hp_h2d = nullptr, hp_d2h = nullptr;
  int hp_slabs = 0;                 // 0: automatic slab count, else forced (sfmg_host_pipeline)
  std::vector<cudaEvent_t> hp_ev;   // [0] start, then [1 + 3c + {0,1,2}] = H2D / compute / D2H done
  // host-polled coarse CG (sfmg_api.cu coarse_cg_any): one batch of iterations captured as a CUDA graph
  // on the level's own stream, for one (x, r) pair
  cudaStream_t cgc_s = nullptr;
  cudaEvent_t cgc_ev[2] = {nullptr, nullptr};
  cudaGraphExec_t cgc_exec = nullptr;
  const double* cgc_x = nullptr;
  const double* cgc_r = nullptr;
  double cgc_rtol = 0.0;
  int cgc_maxit = 0;
};

struct sfmg_hier_s {
  sfmg_mg_params mg;
  std::vector<sfmg_level_s*> lv;
  std::vector<double> lam;
  std::vector<double*> b, x, r;  // per-level V-cycle vectors
  double *pr, *pz, *pp, *ph;     // PCG vectors on the finest level
  int64_t fine_applies;
  // V-cycle replayed as a CUDA graph (captured on a private stream, keyed on the b / x pointers)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t vc_exec = nullptr;
  const double* vc_b = nullptr;
  double* vc_x = nullptr;
  int64_t vc_fine_applies = 0;
  int vc_eager_runs = 0;
  bool host_coarse = false;   // coarsest order > 2: host-polled multi-kernel CG, V-cycle not captured
};

namespace sfmg {

// ---- launchers (k_operator.cu)
cudaError_t upload_order_tables(int p, cudaStream_t s);
cudaError_t launch_geometry(const MeshDev& m, double* G, int* bad, cudaStream_t s);
// v = bnd ? (u ? u[g] : bval) : 0  (bc 0);  v = 0  (bc 1)
cudaError_t launch_init(const MeshDev& m, int bc, const double* u, double bval, double* v, cudaStream_t s);
// v = 0 (one small block per SM, programmatic trigger at block start: the next apply overlaps it)
cudaError_t launch_zero(double* v, long long n, cudaStream_t s);
// v += A(M u) on interior rows (bc 0) or all rows (bc 1); v must be initialised.  Launched with
// programmatic dependent launch: wait_mode 1 = only v comes from the preceding kernel (wait before
// the first scatter), 2 = u does too (wait before the gather).  write_bnd (bc 0): the canonical
// element of each boundary node stores v = u there, so v only needs to be zero beforehand.
cudaError_t launch_apply(const MeshDev& m, int bc, const double* G, const double* u, double* v, int wait_mode,
                         int write_bnd, cudaStream_t s);
cudaError_t launch_diag(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s);
cudaError_t launch_load(const MeshDev& m, int rhs_id, double* f, cudaStream_t s);
// out = cur + c1 (cur - prev) + c2 dinv (b - y); then y = bnd ? out : 0 (ready for next apply)
cudaError_t launch_cheb_update(const MeshDev& m, const double* cur, const double* prev, double* out,
                               const double* b, double* y, const double* dinv, double c1, double c2,
                               cudaStream_t s);
// Fused step (k_apply_v4<.., FU>, 3 <= p <= 8, bc 0; opt-in with SFMG_FUSED=1): one persistent kernel forms
// y = A_D cur in an L2-resident ring of lattice planes and, one element layer behind, mode 0:
// out = cur + c1 (cur - prev) + c2 dinv (b - y) (prev unused when c1 == 0); mode 1: out = y.
// scratch: fused_scratch_doubles(m) doubles, ring part all zero on entry (fused_zero_ring) and on exit.
// Vectors 16-byte aligned; out may alias prev or cur.
bool fused_available(const MeshDev& m);
size_t fused_scratch_doubles(const MeshDev& m);
cudaError_t fused_zero_ring(const MeshDev& m, double* scratch, cudaStream_t s);
cudaError_t launch_fused_step(const MeshDev& m, const double* G, const double* cur, const double* prev, double* out,
                              const double* b, const double* dinv, double* scratch, double c1, double c2, int mode,
                              cudaStream_t s);
cudaError_t launch_export_geometry(const MeshDev& m, const double* G, double* out, cudaStream_t s);
// elements for which G storage is allocated (p <= 2: rounded up to 32 for the interleaved layout)
long long geometry_elems(int p, long long E);
cudaError_t launch_export_maps(const MeshDev& m, int32_t* l2g, uint8_t* mask, uint8_t* col, cudaStream_t s);
// single-CTA CG on a (small) level: x = A_D^{-1} b to rtol (R13)
cudaError_t launch_coarse_cg(const MeshDev& m, const double* G, const double* b, double* x, double* r,
                             double* p, double* q, double* scal, double rtol, int maxit, cudaStream_t s);

// ---- Gauss-Legendre quadrature variant (k_gauss.cu, NEXT-3); the launchers above dispatch to these
// when m.quad == 1
cudaError_t upload_gauss_tables(int p);
cudaError_t launch_geometry_gauss(const MeshDev& m, double* G, int* bad, cudaStream_t s);
cudaError_t launch_apply_gauss(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s);
cudaError_t launch_diag_gauss(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s);
cudaError_t launch_load_gauss(const MeshDev& m, double* f, cudaStream_t s);
cudaError_t launch_coarse_cg_gauss(const MeshDev& m, const double* G, const double* b, double* x, double* r,
                                   double* p, double* q, double* scal, double rtol, int maxit, cudaStream_t s);

// ---- 2-D quadrilateral variant (k_2d.cu, NEXT-2); the launchers above dispatch to these when m.dim == 2
cudaError_t upload_2d_tables(int p, int quad);
cudaError_t launch_geometry_2d(const MeshDev& m, double* G, int* bad, cudaStream_t s);
cudaError_t launch_apply_2d(const MeshDev& m, int bc, const double* G, const double* u, double* v, cudaStream_t s);
cudaError_t launch_diag_2d(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s);
cudaError_t launch_load_2d(const MeshDev& m, double* f, cudaStream_t s);
// 2-D transfer: kind 1 p pair, 2 h pair; dir 0 prolong (out = P0 in, += if add), 1 restrict (out = P0^T in)
cudaError_t launch_transfer_2d(const MeshDev& mc, const MeshDev& mf, int kind, int dir, const double* in, double* out,
                               int add, cudaStream_t s);

// ---- vector kernels (k_blas.cu)
cudaError_t launch_recip(const double* d, double* dinv, long long n, cudaStream_t s);
cudaError_t launch_fill(double* x, double v, long long n, cudaStream_t s);
cudaError_t launch_copy(const double* a, double* b, long long n, cudaStream_t s);
// scalars[slot] = sum a.b (deterministic two-level reduction)
cudaError_t launch_dot(const RedScratch& r, const double* a, const double* b, long long n, int slot, cudaStream_t s);
// power iteration: scalars[0] = x.y, scalars[1] = x.x/dinv, scalars[2] = |y dinv|^2; then
// x = y dinv / sqrt(scalars[2]); y = bnd ? x : 0; scalars[3] = scalars[0]/scalars[1]
cudaError_t launch_power_step(const MeshDev& m, const RedScratch& r, double* x, double* y, const double* dinv,
                              cudaStream_t s);
cudaError_t launch_power_start(const MeshDev& m, uint64_t seed, double* x, double* y, cudaStream_t s);
// r = b - y
cudaError_t launch_residual(const double* b, const double* y, double* r, long long n, cudaStream_t s);
// x += a p ; r -= a h with a = scal[ia] / scal[ib]; scalars[slot] = |r|^2
cudaError_t launch_pcg_xr(const RedScratch& red, double* x, double* r, const double* p, const double* h,
                          int ia, int ib, int slot, long long n, cudaStream_t s);
// p = z + (scal[ia] / scal[ib]) p
cudaError_t launch_pcg_p(const RedScratch& red, double* p, const double* z, int ia, int ib, long long n,
                         cudaStream_t s);
// general coarse CG (any order; R13): start (it = 0, rho = ||b||^2, flag), and the tail of one
// iteration after q = A p and (p, q) -> scalars[kCgcPQ]: x += a p, r -= a q, check, p = r + beta p
cudaError_t launch_cgc_start(const RedScratch& red, cudaStream_t s);
cudaError_t launch_cgc_iter_tail(const RedScratch& red, double* x, double* r, double* p, const double* q, long long n,
                                 double rtol, int maxit, cudaStream_t s);
// x += y
cudaError_t launch_axpy1(double* x, const double* y, long long n, cudaStream_t s);
// scalars[slot] = sum a b / dinv  (<a, b>_D, Arnoldi R26)
cudaError_t launch_dotw(const RedScratch& r, const double* a, const double* b, const double* dinv, long long n,
                        int slot, cudaStream_t s);
// y -= scalars[slot] x
cudaError_t launch_sub_scaled_dev(const RedScratch& r, int slot, const double* x, double* y, long long n,
                                  cudaStream_t s);
// y = a x (* d elementwise if d != null)
cudaError_t launch_scale_mul(double a, const double* x, const double* d, double* y, long long n, cudaStream_t s);

// ---- transfer (k_transfer.cu)
cudaError_t upload_interp_tables(int pc, cudaStream_t s);
// uf = P0 uc (add = 0) or uf += P0 uc (add = 1)
cudaError_t launch_prolong(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                           cudaStream_t s);
// rc = P0^T rf (rc zeroed inside)
cudaError_t launch_restrict(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s);
// h pair at p = 1 (fine ne = 2 coarse ne): uf = P0 uc (add: uf += P0 uc); rc = P0^T rf (gathers, no atomics)
cudaError_t launch_prolong_h(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                             cudaStream_t s);
cudaError_t launch_restrict_h(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s);
// h pair at any order p = 1..16 (NEXT-4): same contract, block per fine element, sum-factorised
cudaError_t upload_h_tables(int p);
cudaError_t launch_prolong_hp(const MeshDev& mc, const MeshDev& mf, const double* uc, double* uf, int add,
                              cudaStream_t s);
cudaError_t launch_restrict_hp(const MeshDev& mc, const MeshDev& mf, const double* rf, double* rc, cudaStream_t s);

void set_error(const std::string& s);

}  // namespace sfmg
