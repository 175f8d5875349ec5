/*
 * sfmg.h -- sum-factorised high-order p-multigrid on one NVIDIA B200 (sm_100a), fp64.
 *
 * C ABI of libsfmg.so, the B200-native hot path of Sundar, Stadler & Biros, "Comparison of
 * multigrid algorithms for high-order continuous finite element discretizations"
 * (arXiv 1402.5938).  Citations: "P:n" = PAPER.md line n; "R<k>" = DESIGN.md reading k.
 *
 * Problem (eq. (1)): -div(mu grad u) = f on the image of [0,1]^3, u = 0 on the
 * boundary, Galerkin discretisation a(u,v) = int mu grad u . grad v with order-p
 * tensor LGL nodal bases on a structured hex mesh, isoparametric
 * geometry and (p+1)^3-point LGL quadrature collocated with the nodes (R1, R2).
 *
 * Conventions for every call:
 *  - All arrays are fp64 (or the stated integer type), contiguous, and CALLER-OWNED.
 *    Pointers prefixed d_ are device pointers on the current CUDA device, h_ host pointers.
 *  - Global dof numbering: g = I + Mx (J + My K), I = ex p + a, ...  (lattice of
 *    Mx = nex p + 1 by My by Mz nodes, x fastest).  Elements e = ex + nex (ey + ney ez),
 *    local nodes l = a + (p+1)(b + (p+1) c).  Vectors have length N = Mx My Mz including the
 *    boundary (R17).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *    asynchronous on that stream unless documented "syncs".  One stream at a time per handle:
 *    handles own scratch inside the caller's workspace.
 *  - The library never allocates device memory.  A handle is built inside a caller-allocated
 *    device workspace whose size the *_query call returns; *_destroy frees host metadata only.
 *  - Every call returns sfmg_status; argument errors are detected synchronously and leave
 *    outputs untouched; asynchronous CUDA faults surface at the next synchronising call
 *    (SFMG_E_CUDA, text in sfmg_last_error()).  No C++ exception crosses the ABI.
 *  - Dirichlet treatment (R4): bc = 0 applies A_D = M A M + (I - M) with M the interior mask
 *    (identity rows and columns on the boundary); bc = 1 applies the unprojected A.
 */
#ifndef SFMG_H
#define SFMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SFMG_OK = 0,
  SFMG_E_ARG = 1,        /* null pointer, bad enum, vector length != N                       */
  SFMG_E_ORDER = 2,      /* p < 1 or p > 16                                                 */
  SFMG_E_MESH = 3,       /* an element count < 1 or a lattice too large for 32-bit indices  */
  SFMG_E_GEOMETRY = 4,   /* det J <= 0 at some quadrature point (folded element)            */
  SFMG_E_PCOARSEN = 5,   /* p odd where p/2 is required, or levels not (p, p/2) on one grid */
  SFMG_E_BREAKDOWN = 6,  /* (p, A p) <= 0 in CG                                             */
  SFMG_E_WORKSPACE = 7,  /* workspace smaller than the queried size, or misaligned          */
  SFMG_E_CUDA = 8        /* CUDA error; see sfmg_last_error()                                */
} sfmg_status;

/* What the paper's problem statement fixes (R3, R5, R6). */
typedef struct {
  int32_t nex, ney, nez;   /* elements per direction on [0,1]^3                             */
  int32_t order;           /* p = 1..16                                                     */
  int32_t warp;            /* 0 identity; 1: x_i += warp_amp sin(pi x) sin(pi y) sin(pi z)   */
  double warp_amp;         /*   (reference-cube point mapped per component; boundary fixed)  */
  int32_t coeff;           /* mu at the physical nodes: 0: c0; 1: exp(c1 S); 2: 10^(c1 S);   */
  double c0, c1;           /*   3: c0 + c1 sum_i cos^2(2 pi x_i); S = sin2pix sin2piy sin2piz */
  int32_t quadrature;      /* 0: (p+1)^3 LGL points collocated with the nodes (R1, BASELINE);  */
                           /* 1: (p+1)^3 Gauss-Legendre points, nodal LGL basis ("Gauss   */
                           /*    quadrature"): G is stored at the Gauss     */
                           /*    points and the apply adds interpolation passes               */
  int32_t dim;             /* 0 or 3: hexahedra (above); 2: quadrilaterals on [0,1]^2 (SURVEY 8(f)  */
                           /*    NEXT-2): nex x ney elements (nez must be 0 or 1),     */
                           /*    warp x_i += warp_amp sin(pi x) sin(pi y), mu kinds 0-2 with       */
                           /*    S = sin2pix sin2piy, 3: c0 + c1 (cos^2 2pi x + cos^2 2pi y)       */
                           /*    (2d-var), 4: c0 + c1 (cos^2 10pi x + cos^2 10pi y) (2d-var');    */
                           /*    every call below applies with (p+1)^2 per element.  Not for 2-D: */
                           /*    sfmg_export_l2g / _mask / _colors / _geometry (SFMG_E_ARG).      */
} sfmg_problem;

/* p-multigrid parameters (R7-R11, R13).  The last four fields select
 * the paper's own settings: zero-initialise the struct, or use the Python
 * MgParams defaults, to get the BASELINE configuration (Chebyshev, power iteration, no h levels). */
typedef struct {
  int32_t nu_pre, nu_post;   /* smoothing applications before / after the coarse correction */
  int32_t cheb_degree;       /* K: steps (= applies) per Chebyshev application               */
  double eig_lo_frac;        /* interval [lo_frac lambda, hi_frac lambda]; BASELINE 0.1, 1.1  */
  double eig_hi_frac;
  int32_t power_iters;       /* lambda_max: power iterations on D^{-1} A_D (R9); 10          */
  uint64_t power_seed;       /* splitmix64 seed of the power-iteration start vector; 12345   */
  double coarse_rtol;        /* p = 1 coarse CG: ||r|| <= coarse_rtol ||b||; 1e-10           */
  int32_t coarse_max_iter;   /* 10000                                                        */
  int32_t smoother;          /* 0: one smoothing application = a degree-cheb_degree Chebyshev- */
                             /*    Jacobi polynomial; 1: one damped point-Jacobi step         */
                             /*    x += jacobi_omega D^{-1} (b - A_D x)  */
  double jacobi_omega;       /* 2/3 in the paper; (0, 2)                                       */
  int32_t lambda_method;     /* 0: power_iters power iterations (R9); 1: power_iters Arnoldi    */
                             /*    steps in the D-inner product (R26)     */
  int32_t h_levels;          /* geometric coarsenings of the p = 1 mesh after p-coarsening     */
                             /*    (ne -> ne/2, trilinear h-transfer); */
                             /*    every ne must be divisible by 2^h_levels                   */
  int32_t coarsen;           /* 0: p-multigrid p, p/2, ..., 1, then h_levels at p = 1 (above); */
                             /* 1: high-order h-multigrid:    */
                             /*    order p (any 1..16) on meshes ne, ne/2, ..., ne/2^h_levels  */
                             /*    (h_levels >= 1), transfer = eq. (7) between nested meshes. */
                             /*    A coarsest order > 2 is solved by a host-polled CG, so that */
                             /*    V-cycle is not replayed as a CUDA graph                    */
} sfmg_mg_params;

/* Solve report.  history: caller-owned host buffer of history_cap doubles
 * receiving ||r_k||_2 for k = 0..iterations (truncated to history_cap), may be NULL. */
typedef struct {
  int32_t iterations;        /* outer iterations (MG-solver V-cycles or PCG iterations)      */
  int32_t converged;         /* 1 iff ||r|| <= rtol ||r0||                                   */
  double r0_norm, r_norm;
  int64_t fine_applies;      /* fine-level operator applications, cost model eq. (8)          */
  int64_t vcycles;           /* V-cycles performed                                            */
  double* history;
  int32_t history_cap;
} sfmg_report;

typedef struct sfmg_level_s* sfmg_level; /* one (mesh, p): G, diag, scratch                    */
typedef struct sfmg_hier_s* sfmg_hier;   /* levels p, p/2, ..., 1 on one element grid, then     */
                                         /* h_levels coarsenings of the p = 1 mesh            */

const char* sfmg_version(void);
/* Text of the last error in this thread ("" if none). */
const char* sfmg_last_error(void);

/* ---------------------------------------------------------------- level setup */
/* Sizes of a level: N (dofs incl. boundary), E (elements) and the device workspace bytes. */
sfmg_status sfmg_level_query(const sfmg_problem* prob, int64_t* n_dofs, int64_t* n_elem,
                             size_t* ws_bytes);
/* Build a level inside d_ws (>= ws_bytes, 256-byte aligned): 1-D LGL basis (host), geometric
 * factors G_q = w_i w_j w_k mu(x_q) detJ_q J_q^{-1} J_q^{-T} at every collocated quadrature
 * point (device), the diagonal of A_D and its inverse.  Syncs (checks det J > 0:
 * SFMG_E_GEOMETRY otherwise). */
sfmg_status sfmg_level_create(const sfmg_problem* prob, void* d_ws, size_t ws_bytes, void* stream,
                              sfmg_level* out);
sfmg_status sfmg_level_destroy(sfmg_level lv);
sfmg_status sfmg_level_info(sfmg_level lv, int64_t* n_dofs, int64_t* n_elem, int32_t* order);

/* Bit-exact exports of the index maps: l2g int32 [E][(p+1)^3];
 * mask uint8 [N] (1 = boundary); colors uint8 [E] = (ex&1) | (ey&1)<<1 | (ez&1)<<2. */
sfmg_status sfmg_export_l2g(sfmg_level lv, int32_t* d_l2g, void* stream);
sfmg_status sfmg_export_mask(sfmg_level lv, uint8_t* d_mask, void* stream);
sfmg_status sfmg_export_colors(sfmg_level lv, uint8_t* d_colors, void* stream);
/* Geometric factors as stored, fp64 [E][p+1][6][(p+1)^2]: element e, slice k (z index), component
 * (00,01,02,11,12,22), point (i + (p+1) j).  Slice-major so that one element (and one k-slice) is
 * one contiguous block for the TMA bulk copies of the apply kernel. */
sfmg_status sfmg_export_geometry(sfmg_level lv, double* d_G, void* stream);

/* ---------------------------------------------------------------- operator */
/* d_v = A_D d_u (bc = 0) or A d_u (bc = 1), matrix-free and sum-factorised.  n must be N;
 * d_u and d_v must not alias. */
sfmg_status sfmg_apply(sfmg_level lv, int32_t bc, const double* d_u, double* d_v, int64_t n,
                       void* stream);
/* diag(A_D) (bc = 0: boundary entries 1) or diag(A) (bc = 1). */
sfmg_status sfmg_diag(sfmg_level lv, int32_t bc, double* d_diag, int64_t n, void* stream);
/* lambda_max of D^{-1} A_D by `iters` power iterations with the D-Rayleigh quotient from a
 * splitmix64(seed) start vector, boundary zeroed (R9).  Syncs.
 * SFMG_E_ARG on a level without interior dofs (the start vector would be zero). */
sfmg_status sfmg_lambda_max(sfmg_level lv, int32_t iters, uint64_t seed, double* h_lambda,
                            void* stream);
/* lambda_max of D^{-1} A_D by `steps` Arnoldi iterations in the D-inner product <x,y>_D =
 * sum d x y (D^{-1} A_D is self-adjoint in it, so H is symmetric tridiagonal up to rounding;
 * Gram-Schmidt repeated once per step), from the same splitmix64(seed) start vector as
 * sfmg_lambda_max; the estimate is the largest eigenvalue of the k x k matrix H (k = steps, or
 * fewer if the Krylov space is exhausted) (R26).  d_work: caller-owned
 * device scratch of (steps + 2) * N doubles.  Syncs. */
sfmg_status sfmg_lambda_arnoldi(sfmg_level lv, int32_t steps, uint64_t seed, double* d_work,
                                double* h_lambda, void* stream);
/* `steps` damped point-Jacobi steps x += omega D^{-1} (b - A_D x), one
 * operator apply each; d_x in/out. */
sfmg_status sfmg_jacobi(sfmg_level lv, const double* d_b, double* d_x, int64_t n, int32_t steps,
                        double omega, void* stream);
/* One degree-`degree` Chebyshev-accelerated Jacobi application to A_D x = b on the interval
 * [lam_lo, lam_hi] of D^{-1} A_D (R7, R10): `degree` steps, each one
 * operator apply.  d_x is the initial guess on input and the smoothed iterate on output.  d_b and
 * d_x must not alias (the recurrence alternates its iterates through d_x): SFMG_E_ARG if equal. */
sfmg_status sfmg_cheb(sfmg_level lv, const double* d_b, double* d_x, int64_t n, int32_t degree,
                      double lam_lo, double lam_hi, void* stream);
/* Load vector of the manufactured solution u* = sin(pi x) sin(pi y) sin(pi z) (rhs_id 1):
 * b_g = (1 - bnd_g) sum_{(e,q) -> g} w_q detJ_q f(x_q), f = -div(mu grad u*). */
sfmg_status sfmg_load_vector(sfmg_level lv, int32_t rhs_id, double* d_f, int64_t n, void* stream);

/* Host-buffer variants (end-to-end path): copy h_u (pinned or pageable) to the level's
 * device scratch, run the call, copy the result back; syncs.  h_* have length N. */
sfmg_status sfmg_apply_host(sfmg_level lv, int32_t bc, const double* h_u, double* h_v, int64_t n,
                            void* stream);
/* sfmg_apply_host is pipelined over z-slabs of element layers: the host->device copy of slab c+1,
 * the kernels of slab c and the device->host copy of slab c-1 run concurrently (two internal copy
 * streams ordered after the caller's prior work on `stream`; the call syncs).  The result is the
 * same A_D u up to the summation order of the scatter.  slabs = 0 (default): automatic (<= 8
 * slabs of >= ~1 MB, 1 for Gauss quadrature); k > 0: min(k, 8, nez) slabs.  p <= 2 needs
 * nex*ney % 32 == 0 to split (else 1 slab). */
sfmg_status sfmg_host_pipeline(sfmg_level lv, int32_t slabs);
sfmg_status sfmg_cheb_host(sfmg_level lv, const double* h_b, double* h_x, int64_t n,
                           int32_t degree, double lam_lo, double lam_hi, void* stream);

/* Benchmark timing of the element (operator) kernel: while enabled, CUDA events are recorded on the
 * stream around every launch of this level's element kernel (apply and Chebyshev steps).  Recording
 * events between kernels removes the overlap of that kernel with its predecessor, so enable it only
 * for a separate measurement pass.  read: accumulated device milliseconds and launch count since the
 * last reset (syncs). */
sfmg_status sfmg_profile_enable(sfmg_level lv, int32_t enable);
sfmg_status sfmg_profile_read(sfmg_level lv, double* ms, int64_t* launches, int32_t reset);

/* ---------------------------------------------------------------- transfer */
/* p pair: fine.order == 2 coarse.order on the same element grid (coarse.order <= 8); or h pair:
 * one order (1..16), fine.ne == 2 coarse.ne in every direction (nesting in
 * reference-lattice coordinates, R25; fine element e is child (ex&1, ey&1, ez&1) of coarse element
 * (ex/2, ey/2, ez/2)).  Anything else: SFMG_E_PCOARSEN.
 * prolong: d_uf = P0 d_uc with P0 = M_f P M_c, P_gJ = phi^{coarse}_J(xi(g)) (eq. (7)).
 * restrict: d_rc = P0^T d_rf (R12).  Vectors sized N_coarse / N_fine. */
sfmg_status sfmg_prolong(sfmg_level coarse, sfmg_level fine, const double* d_uc, double* d_uf,
                         void* stream);
sfmg_status sfmg_restrict(sfmg_level coarse, sfmg_level fine, const double* d_rf, double* d_rc,
                          void* stream);

/* ---------------------------------------------------------------- hierarchy */
sfmg_status sfmg_hier_query(const sfmg_problem* fine, const sfmg_mg_params* mg, size_t* ws_bytes);
/* Build levels p, p/2, ..., 1 (geometry rediscretised per level, R20), then mg->h_levels p = 1
 * levels on meshes ne/2, ne/4, ..., their diagonals and lambda_max estimates (power iteration or
 * Arnoldi per mg->lambda_method).  Syncs.  SFMG_E_PCOARSEN if p is not a power of two or a mesh
 * size is not divisible by 2^h_levels. */
sfmg_status sfmg_hier_create(const sfmg_problem* fine, const sfmg_mg_params* mg, void* d_ws,
                             size_t ws_bytes, void* stream, sfmg_hier* out);
sfmg_status sfmg_hier_destroy(sfmg_hier h);
sfmg_status sfmg_hier_info(sfmg_hier h, int32_t* n_levels, int64_t* n_dofs_fine);
/* Level l (0 = finest) as a level handle owned by the hierarchy (do not destroy). */
sfmg_status sfmg_hier_level(sfmg_hier h, int32_t l, sfmg_level* out);
sfmg_status sfmg_hier_lambda(sfmg_hier h, int32_t l, double* h_lambda);
/* x = V(b) from x = 0: per level nu_pre smoothing applications (Chebyshev or Jacobi), residual,
 * restriction, recursion, prolongation + correction, nu_post applications; coarsest by CG
 * (R11, R13).  No host synchronisation when the coarsest level is a 3-D level of
 * order <= 2 (the single-CTA device CG; the whole V-cycle is replayed as a CUDA graph).  A 2-D
 * hierarchy, or a coarsest order > 2 (h-multigrid, NEXT-4), solves the coarsest level with the
 * host-polled CG, which synchronises the stream every 8 CG iterations. */
sfmg_status sfmg_vcycle(sfmg_hier h, const double* d_b, double* d_x, void* stream);
/* mode 0: MG as solver, x <- x + V(b - A x); mode 1: MG-preconditioned CG (Algorithm 1,
 * P:973-991).  x0 = 0 (the input content of d_x is ignored), stop at ||r||_2 <= rtol ||r0||_2
 * (P:1000-1003).  Non-convergence is not an error (converged = 0).  Syncs each iteration. */
sfmg_status sfmg_solve(sfmg_hier h, int32_t mode, const double* d_b, double* d_x, double rtol,
                       int32_t max_iter, sfmg_report* report, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFMG_H */
