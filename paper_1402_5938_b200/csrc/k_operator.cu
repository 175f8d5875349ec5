// Operator kernels for sm_100a: geometric factors, the matrix-free sum-factorised stiffness
// apply (the hot kernel), its diagonal, the Chebyshev update, the load vector, the index-map
// exports and the single-CTA coarse CG.  fp64 throughout (BASELINE north_star).
//
// Element operator, per element e with n = p+1 points/direction:
//   g0(i,j,k) = sum_m D[i][m] u(m,j,k), g1 = sum_m D[j][m] u(i,m,k), g2 = sum_m D[k][m] u(i,j,m)
//   w = G_q g                                 (G_q symmetric, 6 unique fp64 per point)
//   v(a,b,c) = sum_i D[i][a] w0(i,b,c) + sum_j D[j][b] w1(a,j,c) + sum_k D[k][c] w2(a,b,k)
//   v[l2g(e,.)] += v_e                        (fp64 RED into L2)
// D[i][m] = ell_m'(xhat_i) lives in __constant__ memory: with p a template parameter every loop
// is unrolled, every D index is a compile-time constant, and DFMA takes D as a constant-bank
// operand (no load instruction).
#include <cstdio>
#include <cstdlib>

#include "k_common.cuh"

namespace sfmg {

// Constant-memory tables (packed per order; 43 KB in total):
//  * c_Dc: D[i][m] = ell_m'(xhat_i) of every order; odd p <= 7 keep 5 identical copies, one per line
//    pass of the apply kernel, so each pass reads its own constant addresses and ptxas reloads D per
//    pass (LDCU into uniform registers feeding DFMA) instead of keeping all n^2 values live in the
//    register file across passes (which produced R2UR/IMAD juggling and spills).
//  * c_EO: even p >= 4, the even-odd split of D (and D^T), 6 copies (one per line-pass use).  LGL
//    nodes are symmetric, so D is centro-antisymmetric, D[n-1-i][n-1-m] = -D[i][m]; with
//    e_m = L_m + L_{n-1-m}, o_m = L_m - L_{n-1-m} (m < c = p/2):
//      (D L)_i       = S_i + T_i,   (D L)_{n-1-i} = S_i - T_i   (i < c),   (D L)_c = sum_m D[c][m] o_m
//      S_i = sum_m A[i][m] o_m,  A = (D[i][m] - D[i][n-1-m]) / 2
//      T_i = sum_m B[i][m] e_m + D[i][c] L_c,  B = (D[i][m] + D[i][n-1-m]) / 2
//    which is the same product with 2c^2 + 6c instead of n^2 fp64 operations (-31 % at p = 8,
//    -39 % at p = 16) and half the constants.
//  * c_xw: LGL nodes and weights of every order.
constexpr int kDCopies = 5;
// orders up to this share one even-odd table for D and one for D^T across the line passes (p = 8:
// Chebyshev step -2.4 %); above it every pass reads its own copy (p = 16 with shared tables: ptxas keeps
// the 144 coefficients live across passes and spills, 70 -> 105 us)
constexpr int kEoSharedMaxP = 8;
constexpr int dcopies(int P) { return (P % 2 == 1 && P <= 7) ? kDCopies : 1; }
constexpr int dOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += dcopies(q) * (q + 1) * (q + 1);
  return s;
}
constexpr int eoSize(int P) { return 2 * (P / 2) * (P / 2) + 2 * (P / 2); }
constexpr int eoOffset(int P) {
  int s = 0;
  for (int q = 4; q < P; q += 2) s += 6 * eoSize(q);
  return s;
}
constexpr int xOffset(int P) {
  int s = 0;
  for (int q = 1; q < P; ++q) s += q + 1;
  return s;
}
__constant__ double c_Dc[dOffset(kMaxOrder + 1)];
__constant__ double c_EO[eoOffset(kMaxOrder + 2)];
__constant__ double c_xw[2][xOffset(kMaxOrder + 1)];

static OncePerDevice g_uploaded[kMaxOrder + 1];
// shared-memory tables of the k-split apply (k_apply_ks.cuh), laid out on the host
static cudaError_t upload_ks_tables(int p, const std::vector<double>& D, const std::vector<double>& eo6);

static cudaError_t upload_order_tables_now(int p) {
  Basis1D B = make_basis(p);
  const int n = p + 1;
  cudaError_t e;
  for (int c = 0; c < dcopies(p); ++c) {
    e = cudaMemcpyToSymbol(c_Dc, B.D.data(), sizeof(double) * n * n, sizeof(double) * (dOffset(p) + c * n * n));
    if (e) return e;
  }
  if (p % 2 == 0 && p >= 4) {
    const int c = p / 2;
    std::vector<double> tab(6 * eoSize(p));
    for (int set = 0; set < 6; ++set) {
      auto M = [&](int i, int m) { return set < 3 ? B.D[i * n + m] : B.D[m * n + i]; };   // D or D^T
      double* t = tab.data() + set * eoSize(p);
      for (int i = 0; i < c; ++i)
        for (int m = 0; m < c; ++m) {
          t[i * c + m] = 0.5 * (M(i, m) - M(i, n - 1 - m));
          t[c * c + i * c + m] = 0.5 * (M(i, m) + M(i, n - 1 - m));
        }
      for (int i = 0; i < c; ++i) t[2 * c * c + i] = M(i, c);
      for (int m = 0; m < c; ++m) t[2 * c * c + c + m] = M(c, m);
    }
    e = cudaMemcpyToSymbol(c_EO, tab.data(), sizeof(double) * tab.size(), sizeof(double) * eoOffset(p));
    if (e) return e;
    if ((e = upload_ks_tables(p, B.D, tab))) return e;
  }
  e = cudaMemcpyToSymbol(c_xw, B.x.data(), sizeof(double) * n, sizeof(double) * xOffset(p));
  if (e) return e;
  return cudaMemcpyToSymbol(c_xw, B.w.data(), sizeof(double) * n, sizeof(double) * (xOffset(kMaxOrder + 1) + xOffset(p)));
}
cudaError_t upload_order_tables(int p, cudaStream_t s) {
  (void)s;
  if (p < 1 || p > kMaxOrder) return cudaErrorInvalidValue;
  return g_uploaded[p].run([p] { return upload_order_tables_now(p); });
}

// ------------------------------------------------------------------------------------------
// small device helpers

// D[i][m] of order P, copy `cp` (odd p <= 7 only; other orders keep one copy), idx = i (P+1) + m
template <int P>
__device__ __forceinline__ double dmat(int cp, int idx) {
  return c_Dc[dOffset(P) + (dcopies(P) > 1 ? cp : 0) * (P + 1) * (P + 1) + idx];
}

// out = M L for one 1-D line, M = D (SET 0..2) or D^T (SET 3..5), in the even-odd form above.
// zo: an offset that is always 0 but opaque to the compiler (k_apply_ks passes one derived from its
// element index), so the table loads stay inside the element loop as uniform loads feeding DFMA
// instead of being hoisted into (and spilled from) the per-thread register file
template <int P, int SET>
__device__ __forceinline__ void eo_line(const double (&L)[P + 1], double (&out)[P + 1], int zo = 0) {
  constexpr int N = P + 1, c = P / 2;
  constexpr int base = eoOffset(P) + (P <= kEoSharedMaxP ? (SET < 3 ? 0 : 3) : SET) * eoSize(P);
  double ev[c], od[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    ev[m] = L[m] + L[N - 1 - m];
    od[m] = L[m] - L[N - 1 - m];
  }
#pragma unroll
  for (int i = 0; i < c; ++i) {
    double S = 0.0, T = c_EO[base + 2 * c * c + i + zo] * L[c];
#pragma unroll
    for (int m = 0; m < c; ++m) {
      S = fma(c_EO[base + i * c + m + zo], od[m], S);
      T = fma(c_EO[base + c * c + i * c + m + zo], ev[m], T);
    }
    out[i] = S + T;
    out[N - 1 - i] = S - T;
  }
  double M = 0.0;
#pragma unroll
  for (int m = 0; m < c; ++m) M = fma(c_EO[base + 2 * c * c + c + m + zo], od[m], M);
  out[c] = M;
}

// Isoparametric Jacobian at collocated point (i,j,k): J[al][be] = d x_al / d xi_be
// = sum_m D[.][m] x_al along the be-line through the point (R2).
template <int P>
__device__ __forceinline__ void jacobian(const MeshDev& m, const double* sD, const double* xs, int ex,
                                         int ey, int ez, int i, int j, int k, double J[3][3]) {
  constexpr int N = P + 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) J[a][0] = J[a][1] = J[a][2] = 0.0;
  for (int mm = 0; mm < N; ++mm) {
    double X[3];
    node_pos<P>(m, xs, ex, ey, ez, mm, j, k, X);
    double d = sD[i * N + mm];
    J[0][0] += d * X[0]; J[1][0] += d * X[1]; J[2][0] += d * X[2];
    node_pos<P>(m, xs, ex, ey, ez, i, mm, k, X);
    d = sD[j * N + mm];
    J[0][1] += d * X[0]; J[1][1] += d * X[1]; J[2][1] += d * X[2];
    node_pos<P>(m, xs, ex, ey, ez, i, j, mm, X);
    d = sD[k * N + mm];
    J[0][2] += d * X[0]; J[1][2] += d * X[1]; J[2][2] += d * X[2];
  }
}

// ------------------------------------------------------------------------------------------
// K1 geometric factors: one thread per (element, point), G [E][k][6][n^2].

template <int P>
__global__ void __launch_bounds__(256) k_geometry(MeshDev m, double* __restrict__ G, int* bad) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  __shared__ double sD[N * N], sx[N], sw[N];
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) sD[t] = dmat<P>(0, t);
  for (int t = threadIdx.x; t < N; t += blockDim.x) { sx[t] = c_xw[0][xOffset(P) + t]; sw[t] = c_xw[1][xOffset(P) + t]; }
  __syncthreads();
  const long long total = m.E * N3;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long e = idx / N3;
    int q = (int)(idx - e * N3);
    int i = q % N, j = (q / N) % N, k = q / N2;
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    double J[3][3];
    jacobian<P>(m, sD, sx, ex, ey, ez, i, j, k, J);
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                 J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                 J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) atomicAdd(bad, 1);
    double id = 1.0 / det;
    double Ji[3][3];
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
    double X[3];
    node_pos<P>(m, sx, ex, ey, ez, i, j, k, X);
    double s = sw[i] * sw[j] * sw[k] * coeff_mu(m, X[0], X[1], X[2]) * det;
    const int comp[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      int a = comp[c][0], b = comp[c][1];
      G[GLayout<P>::off(e, c, i + N * j, k)] = s * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Programmatic dependent launch (PDL): a kernel launched with programmatic stream serialization
// may start while its predecessor is still running; griddepcontrol.wait blocks until the
// predecessor grid has completed and its memory is visible.  Kernels that feed an apply call
// launch_dependents at their start so the apply can issue its geometric-factor prefetches early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------------------------------
// K2 apply, v4 (p >= 3): persistent, software-pipelined across element groups.
// Block = EPB elements x (n x n) threads; thread t = (t0, t1) of an element owns one 1-D line per
// pass: P1 x-lines g0 = D u -> s0; P2 y-lines g1 = D u (in place); P3 z-lines in registers:
// g2 = D u, w = G g, w0 -> s0, w1 -> su, vz = D^T w2; P4 x-lines v0 = D^T w0 (in place);
// P5 y-lines su = D^T w1 + v0; P6 z-lines v = su + vz, fp64 RED into v.  Each line pass reads n
// values and does n^2 FMAs (D from __constant__ via uniform registers).
// Each block walks groups grp = blockIdx.x, + gridDim.x, ...:
//  * p <= 8 (GS): one TMA bulk copy (cp.async.bulk + mbarrier complete_tx) of the group's factors
//    into smem, issued for group g+1 as soon as P3 of group g has consumed the buffer;
//  * p >= 9: the factors are read in P3 straight from L2 with a 3-slice register ring;
//  * both: a TMA L2 prefetch (cp.async.bulk.prefetch.L2) of group g+2's factors, and the u column
//    of group g+1 loaded into registers during P4-P6 (group g+2's column prefetched to L2), so HBM
//    always has the next-but-one group of every resident block in flight.
// Smem per element: 2 n^3 doubles (+ 6 n^3 staged factors when GS).

__device__ __forceinline__ void cp_async8(double* dst, const double* src, unsigned src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// GS = true : the group's factors are staged in smem by one TMA bulk copy (p <= 8 fits).
// GS = false: P3 reads the factors straight from L2 into registers through a k-slice ring, with the
//             next element TMA-prefetched into L2 (p >= 9: G of one element is up to 236 KB and cannot
//             be staged).
//
// Tuning constants (measured choices; the rejected alternatives and their times are listed in
// profiles/r01_experiments.md).
constexpr int kRing = 5;           // !GS: register ring depth in k-slices (loads kRing - 1 slices ahead)
constexpr int kV4Smem = 52000;     // smem budget per block that sets the elements per block (p <= 8)
constexpr int kV4Thr = 256;        // thread budget per block that sets the elements per block
constexpr int kPfGS = 2;           // GS, long grids: L2 prefetch of group g+2
// Early programmatic-dependent triggers (v init, Chebyshev update, apply -> update) are used for
// vectors of at most this many dofs; SFMG_EARLY_MAXN in the environment overrides it (0: never; the
// tests run both paths).
constexpr long long kEarlyMaxN = 1ll << 24;
static bool early_pdl(const MeshDev& m) {
  static const long long thr = [] {
    const char* e = getenv("SFMG_EARLY_MAXN");
    return e ? atoll(e) : kEarlyMaxN;
  }();
  return m.N <= thr;
}

template <int P, bool GS>
struct V4Cfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr int PER_ELEM = (GS ? 8 : 2) * N3 * 8;   // smem bytes per element
  static constexpr int EPB_SMEM = kV4Smem / PER_ELEM > 0 ? kV4Smem / PER_ELEM : 1;
  static constexpr int EPB_THR = kV4Thr / N2 > 0 ? kV4Thr / N2 : 1;
  static constexpr int EPB = EPB_SMEM < EPB_THR ? EPB_SMEM : EPB_THR;
  static constexpr int THREADS = EPB * N2;
  static constexpr size_t SMEM = (size_t)EPB * PER_ELEM + 16;
  static constexpr int MINB_SMEM = (227 * 1024) / (SMEM + 1024) < 8 ? (227 * 1024) / (SMEM + 1024) : 8;
  static constexpr int MINB = GS ? MINB_SMEM : (P >= 12 ? 1 : 2);
};

// Developer timeline (-DSFMG_TIMELINE, tools/v4_timeline.py): %globaltimer marks per block of the
// v init and the persistent apply; compiled out of the library.
#ifdef SFMG_TIMELINE
__device__ unsigned long long g_tl_init[4096 * 2];
__device__ unsigned long long g_tl_v4[2048 * 4];
#define TLMARK(arr, stride, cap, s_)                                       \
  if (threadIdx.x == 0 && blockIdx.x < (cap)) {                            \
    unsigned long long t_;                                                 \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    arr[blockIdx.x * (stride) + (s_)] = t_;                                \
  }
#else
#define TLMARK(arr, stride, cap, s_)
#endif

// ------------------------------------------------------------------------------------------
// FU: the Chebyshev step (or the standalone apply) fused into one persistent kernel for vectors that
// do not fit in L2 (north_star: "fused with the operator apply so each step makes one pass over HBM";
// P:936-945 costs a smoother step as one matvec).  y = A x_k is never written to HBM: the blocks RED
// their element contributions into a ring of `rp` lattice planes (slot = K mod rp, L2 resident, all
// zero before and after the launch).  The lattice plane set L = planes [L p, (L+1) p) is final once the
// element layers L - 1 and L are complete; it is cut into gpl contiguous pieces, piece q attached to
// group slot (L+1) gpl + q + shift, and the block that owns a slot runs its piece right after the
// slot's scatter: it reads the finished y back from the ring, forms x_{k+1} = x_k + c1 (x_k - x_{k-1}) +
// c2 D^-1 (b - y) (boundary rows: y = x_k, R4), writes it and re-zeroes the ring entries.  Ordering:
//  * layer_done[L]: groups of element layer L whose scatter is complete; upd_done[L]: pieces of plane set
//    L complete.  Both are released by thread 0 (fence + atomic) after the block barrier that follows the
//    work, at the top of the block's next slot.
//  * before a slot's scatter, thread 0 acquires upd_done == gpl for every plane set whose ring slots the
//    element layer's planes reuse, and layer_done == gpl for the layers under the slot's piece.
// Every wait refers to strictly earlier slots (the launcher bounds shift accordingly) and every block
// of the persistent grid is resident, so the waits cannot deadlock; each spin still carries a clock
// timeout that raises *err.
struct FusedArgs {
  const double* prev = nullptr;
  double* out = nullptr;
  const double* b = nullptr;
  const double* dinv = nullptr;
  double c1 = 0.0, c2 = 0.0;
  unsigned int* layer_done = nullptr;
  unsigned int* upd_done = nullptr;
  int* err = nullptr;
  int rp = 0;      // ring planes
  int mode = 0;    // 0 Chebyshev / Jacobi update, 1 out = A_D x (ring copied out, boundary rows = x)
  long long gpl = 0, shift = 0;
  unsigned chunk = 0, chunk_last = 0;   // nodes per update piece (even), inner plane sets / the last one
  int color = 0;                        // COL: element colour of this launch
};

// Explicit reductions: in the fused kernel ptxas keeps atomicAdd as the value-returning ATOMG (the
// scatter then waits a full L2 round trip per node); red.* has no destination register.
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}
// Ring accesses carry an L2 evict-last policy: the ring is re-used every rp planes and must not be
// displaced by the streams that pass through L2 once (u, the factors in flight, x_{k-1}, b, D^-1).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void ring_red(double* p, double v, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol));
}
__device__ __forceinline__ double ring_ld(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void ring_st(double* p, double v, uint64_t pol) {
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_u32(unsigned int* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned int* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __noinline__ void spin_ge(const unsigned int* p, unsigned target, int* err) {
  if (ld_acquire_u32(p) >= target) return;
  const long long t0 = clock64();
  unsigned ns = 100;
  for (;;) {
    __nanosleep(ns);   // back-off: hundreds of pollers on one L2 line would stall the releasing atomics
    if (ns < 1600) ns *= 2;
    if (ld_acquire_u32(p) >= target) return;
    // ~2 s: never in a correct run; reported through *err (and every later wait gives up at once)
    if (clock64() - t0 > (1ll << 32) || *reinterpret_cast<volatile int*>(err)) {
      atomicExch(err, 86);
      return;
    }
  }
}

// Node range [lo, hi) of piece q of plane set L (see fused_piece).
template <int P>
__device__ __forceinline__ void fused_piece_range(const MeshDev& m, const FusedArgs& f, int L, unsigned q, unsigned& sL,
                                                  unsigned& eL, unsigned& lo, unsigned& hi) {
  const unsigned sxy = (unsigned)m.Mx * (unsigned)m.My;
  const bool last = (L == m.nez - 1);
  sL = (unsigned)L * P * sxy;
  eL = last ? (unsigned)m.N : sL + P * sxy;
  const unsigned chunk = last ? f.chunk_last : f.chunk;
  lo = (sL & ~1u) + q * chunk;
  hi = lo + chunk;
  if (hi > eL) hi = eL;
}
// L2 prefetch of the streams a piece reads from HBM (x_{k-1}, b, D^-1), issued by three threads at the top
// of the slot so that the piece, an element later, finds them in L2.
template <int P>
__device__ __forceinline__ void fused_piece_prefetch(const MeshDev& m, const FusedArgs& f, int L, unsigned q, int tid) {
  if (tid >= 3 || (f.mode & 3) != 0 || (f.mode & 4)) return;
  const double* src = tid == 0 ? f.b : (tid == 1 ? f.dinv : f.prev);
  if (tid == 2 && f.c1 == 0.0) return;
  unsigned sL, eL, lo, hi;
  fused_piece_range<P>(m, f, L, q, sL, eL, lo, hi);
  if (lo >= hi) return;
  lo &= ~1u;                           // 16-byte aligned start, size a multiple of 16 (may touch one node
  const unsigned n = (hi - lo + 1) & ~1u;   // past the piece; never past the vector's 16-byte padding)
  unsigned bytes = n * 8;
  if ((unsigned long long)lo + n > (unsigned long long)m.N) bytes -= 16;
  if (bytes) bulk_prefetch_l2(src + lo, bytes);
}

// One update piece of plane set L, by the NT threads of the block (tid = 0..NT-1): nodes
// [A + q chunk, A + (q+1) chunk) clipped to the set, A = the set's first node rounded down to even, chunk
// even, so every piece starts on a 16-byte boundary and is walked in double2 pairs (a lone first / last
// node of an odd-aligned set goes through the scalar path).  The ring already holds y = A_D x including
// the Dirichlet rows (their owner elements stored x there), so a node needs no lattice coordinates;
// only its plane (ring slot) is tracked, incrementally from one division per thread.
template <int P, int NT>
__device__ __forceinline__ void fused_piece(const MeshDev& m, const double* cur, double* ring, const FusedArgs& f,
                                            int L, unsigned q, int tid) {
  constexpr int U = 4;
  const unsigned sxy = (unsigned)m.Mx * (unsigned)m.My;
  const unsigned rp = (unsigned)f.rp;
  const bool cheb = ((f.mode & 3) == 0), use_prev = cheb && (f.c1 != 0.0);
  const double c1 = f.c1, c2 = f.c2;
  const uint64_t pol = l2_evict_last_policy();
  unsigned sL, eL, lo, hi;
  fused_piece_range<P>(m, f, L, q, sL, eL, lo, hi);
  if (lo >= hi || (f.mode & 4)) return;   // (mode & 4: developer ablation, no update traffic)
  auto value = [&](double xc, double xp, double bb, double dd, double y) -> double {
    return cheb ? xc + c1 * (xc - xp) + c2 * dd * (bb - y) : y;
  };
  auto one = [&](unsigned g) {
    const unsigned K = g / sxy, ri = (K % rp) * sxy + (g - K * sxy);
    const double y = ring_ld(ring + ri, pol);
    const double xc = cheb ? __ldcg(cur + g) : 0.0;
    const double xp = use_prev ? __ldcs(f.prev + g) : 0.0;
    const double bb = cheb ? __ldcs(f.b + g) : 0.0, dd = cheb ? __ldcs(f.dinv + g) : 0.0;
    __stcs(f.out + g, value(xc, xp, bb, dd, y));
    ring_st(ring + ri, 0.0, pol);
  };
  if (lo < sL) {   // odd-aligned set: its first node alone
    if (tid == 0) one(sL);
    lo += 2;
  }
  if (hi & 1) {    // (only hi == eL can be odd)
    --hi;
    if (tid == NT - 1) one(hi);
  }
  if (lo >= hi) return;
  const unsigned np = (hi - lo) >> 1;
  const unsigned K0 = lo / sxy, rr0 = lo - K0 * sxy, slot0 = K0 % rp;
  for (unsigned i0 = 0; i0 < np; i0 += NT * U) {
    double2 xc[U], xp[U], bb[U], dd[U];
    double y0[U], y1[U];
    unsigned a0[U], a1[U];
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const unsigned i = i0 + w * NT + tid;
      xc[w] = xp[w] = bb[w] = dd[w] = make_double2(0.0, 0.0);
      if (i < np) {
        const unsigned g = lo + 2 * i;
        unsigned r = rr0 + 2 * i, slot = slot0;
        while (r >= sxy) { r -= sxy; slot = (slot + 1 == rp) ? 0 : slot + 1; }
        a0[w] = slot * sxy + r;
        a1[w] = (r + 1 < sxy) ? a0[w] + 1 : ((slot + 1 == rp) ? 0 : slot + 1) * sxy;
        y0[w] = ring_ld(ring + a0[w], pol);
        y1[w] = ring_ld(ring + a1[w], pol);
        if (cheb) {
          xc[w] = __ldcg(reinterpret_cast<const double2*>(cur + g));
          if (use_prev) xp[w] = __ldcs(reinterpret_cast<const double2*>(f.prev + g));
          bb[w] = __ldcs(reinterpret_cast<const double2*>(f.b + g));
          dd[w] = __ldcs(reinterpret_cast<const double2*>(f.dinv + g));
        }
      }
    }
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const unsigned i = i0 + w * NT + tid;
      if (i < np) {
        double2 o;
        o.x = value(xc[w].x, xp[w].x, bb[w].x, dd[w].x, y0[w]);
        o.y = value(xc[w].y, xp[w].y, bb[w].y, dd[w].y, y1[w]);
        __stcs(reinterpret_cast<double2*>(f.out + lo + 2 * i), o);
        ring_st(ring + a0[w], 0.0, pol);
        ring_st(ring + a1[w], 0.0, pol);
      }
    }
  }
}

// IPS: element-interior nodes (one owner element) take a plain store instead of an fp64 RED (v must be
// zero there beforehand, as the init kernels leave it).  Used for vectors larger than L2 (N > 2^24)
// right after the v init, where a RED into a line that the init already evicted costs an HBM read; for
// L2-resident vectors the REDs are cheaper (config 2 measured slower with plain stores).
// COL (measurement variant, SFMG_COLOR=1; EPB = 1 orders only): one launch per element colour
// (ex & 1, ey & 1, ez & 1) -- elements of one colour share no node, so the scatter is a plain
// load-add-store instead of an fp64 RED (north_star: "element coloring or atomics, whichever ncu favours";
// measured in profiles/r02_experiments.md).
template <int P, bool DIR, bool GS, bool IPS = false, bool FU = false, bool COL = false>
__global__ void __launch_bounds__(V4Cfg<P, GS>::THREADS, V4Cfg<P, GS>::MINB)
    k_apply_v4(MeshDev m, const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ v,
               long long ngroups, int wait_mode, int write_bnd, FusedArgs f) {
  using C = V4Cfg<P, GS>;
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3;
  auto bsync = [&]() { __syncthreads(); };
  constexpr bool EO = (P % 2 == 0) && P >= 4;   // even-odd line products
  // the next group's u column is loaded right after this group's is staged, so it is in flight
  // during the whole element (measured: p = 16 -2.5 %, p <= 8 within noise)
  // (p >= 12: off; the u columns are L2-prefetched instead, which frees 2n registers: p = 16 -2 %)
  constexpr bool EARLY = P <= 11;
  // TR: the y-direction data live in a transposed array (index j + n i + n^2 k), so the y-line passes
  // read and write it with the x-lines' conflict-free stride; s0 holds u -> g0 -> w0 -> X (natural layout,
  // x-lines in place), su holds u -> g1 -> w1 -> Y (transposed, y-lines in place), and the z-line pass
  // adds X + Y + Z.  Removes the 2-way bank conflicts of natural-layout y-lines at p = 8.
  constexpr bool TR = GS && P == 8;   // measured: p = 8 step -2 %, p = 4 +1 %
  extern __shared__ __align__(128) double smem[];
  double* sG = smem;                                   // [EPB][k][6][n^2] (GS)
  const int le = threadIdx.x / N2;
  const int t = threadIdx.x - le * N2;
  const int t0 = t % N, t1 = t / N;
  double* s0 = smem + (GS ? C::EPB * 6 * N3 : 0) + le * 2 * N3;   // per element: s0, su
  double* su = s0 + N3;
  uint64_t* bar = (uint64_t*)(smem + C::EPB * (GS ? 8 : 2) * N3);
  if constexpr (FU) static_assert(DIR && GS && !IPS, "fused step: Dirichlet operator, staged factors");
  const double* gE = sG + le * 6 * N3;
  const long long sxy = (long long)m.Mx * m.My;
  const long long gstride = gridDim.x;
  if constexpr (COL) static_assert(C::EPB == 1 && !FU && !IPS, "coloured variant: one element per block");
  // first element of group g (COL: the g-th element of colour f.color, x fastest)
  auto gfirst = [&](long long g) -> long long {
    if constexpr (COL) {
      const int cx = f.color & 1, cy = (f.color >> 1) & 1, cz = (f.color >> 2) & 1;
      const unsigned nxc = (unsigned)(m.nex - cx + 1) >> 1, nyc = (unsigned)(m.ney - cy + 1) >> 1;
      const unsigned ug = (unsigned)g, tq = ug / nxc, ix = ug - tq * nxc, iz = tq / nyc, iy = tq - iz * nyc;
      (void)cz;
      return (long long)(2 * ix + cx) + (long long)m.nex * ((2 * iy + cy) + (long long)m.ney * (2 * iz + cz));
    } else {
      return g * C::EPB;
    }
  };
  auto group_bytes = [&](long long g) -> unsigned {
    long long nel = m.E - gfirst(g);
    if (nel > C::EPB) nel = C::EPB;
    return (unsigned)(nel * 6 * N3 * sizeof(double));
  };
  auto prefetch_group_l2 = [&](long long g) {   // TMA L2 prefetch in <= 64 KB pieces
    const char* src = (const char*)(G + gfirst(g) * 6 * N3);
    const unsigned total = group_bytes(g);
    for (unsigned o = 0; o < total; o += 65536u) bulk_prefetch_l2(src + o, total - o < 65536u ? total - o : 65536u);
  };
  // this thread's u column of group g (M u: zero outside the element / on Dirichlet nodes, R4)
  auto load_column = [&](long long g, double (&r)[N]) {
    const long long e = gfirst(g) + le;
    const bool act = e < m.E;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    const long long col = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + t0, J = ey * P + t1;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      bool ok = act;
      if (DIR) { const int K = ez * P + k; ok = ok && !(bxy || K == m.Kb0 || K == m.Kb1); }
      r[k] = ok ? __ldg(u + col + sxy * k) : 0.0;
    }
  };
  auto prefetch_column = [&](long long g) {
    const long long e = gfirst(g) + le;
    if (e >= m.E) return;
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const double* pu = u + (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
#pragma unroll
    for (int k = 0; k < N; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + sxy * k));
  };

  long long grp = blockIdx.x;
  // L2 prefetch distance of the factor stream in groups (GS: the TMA already holds group g+1 in smem)
  // L2 prefetch distance of the factor stream in groups.  GS: the TMA already holds group g+1 in smem;
  // an L2 prefetch of g+2 deepens the HBM pipeline, which pays in long runs (config 4: 2.68 -> 2.53 ms)
  // but delays the first TMA loads of short ones (config 2: 46.1 -> 48.1 us), so it is used only when
  // each block walks >= 16 groups.  !GS: g+1 (two generations of p >= 9 factors overflow L2).
  const int PF = GS ? (ngroups >= 16 * gstride ? kPfGS : 1) : 1;
  if (threadIdx.x == 0) {   // factor prefetches need nothing from the predecessor kernel
    if (GS) {
      mbar_init(bar, 1);
      if (grp < ngroups) bulk_load(sG, G + gfirst(grp) * 6 * N3, group_bytes(grp), bar);
    } else if (grp < ngroups) {
      prefetch_group_l2(grp);
    }
  }
  TLMARK(g_tl_v4, 4, 2048, 0);
  // wait_mode 2: u is produced by the predecessor; 1: only v is (wait before the first scatter)
  if (wait_mode == 2) pdl_wait();
  bool waited = (wait_mode != 1);
  double ru[N];
  if (grp < ngroups) load_column(grp, ru);
  if (grp + gstride < ngroups) prefetch_column(grp + gstride);
  unsigned phase = 0;
  // FU: this block's finished but unpublished work: acc_ln groups of element layer acc_layer and acc_sn
  // pieces of plane set acc_set.  They are released (one fence, then the counter REDs) when the block moves
  // on to another layer / set -- the counters only matter once a layer / set is complete, and a fence per
  // slot costs ~1 us of the block's critical path.
  int acc_layer = -1, acc_ln = 0, acc_set = -1, acc_sn = 0;
  int lay_chk = -1;     // FU: element layers <= lay_chk are known to be complete
  int chk_layer = -1;   // FU: plane sets <= chk_layer are known to be updated (their ring slots re-zeroed)
  for (; grp < ngroups; grp += gstride) {
    constexpr int zero = 0;
    if constexpr (FU) {   // this slot's update piece: start its HBM streams towards L2 now
      const long long pjp = grp - f.gpl - f.shift;
      if (pjp >= 0 && threadIdx.x < 3 && !(f.mode & 8)) {
        const int Lp = (int)((unsigned)pjp / (unsigned)f.gpl);
        fused_piece_prefetch<P>(m, f, Lp, (unsigned)pjp - (unsigned)Lp * (unsigned)f.gpl, threadIdx.x);
      }
    }
    // last group of this block: let a programmatic dependent (the Chebyshev update) launch now; it
    // waits (griddepcontrol.wait) for this grid's completion before reading v.  Small vectors only
    // (config 4 measured 2.51 -> 2.61 ms with it)
    if (m.pdl_early && grp + gstride >= ngroups) pdl_trigger();
    const long long e = gfirst(grp) + le;
    const bool act = e < m.E;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    const long long gcol = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + t0, J = ey * P + t1;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
    const double* Gg = G + (act ? e : 0) * 6 * N3 + t;   // GS == false: this thread's factor column
    constexpr int RG = kRing;                               // ring depth (loads RG - 1 slices ahead)
    double gb[RG][6];                                       // GS == false: k-slice ring in registers
    if (!GS) {
#pragma unroll
      for (int kk = 0; kk < RG - 1 && kk < N; ++kk)
#pragma unroll
        for (int c = 0; c < 6; ++c) gb[kk][c] = __ldcs(Gg + gofs<N>(c, 0, kk));
    }
    if (TR) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s0[t + N2 * k] = ru[k];
        su[t1 + N * t0 + N2 * k] = ru[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) su[t + N2 * k] = ru[k];
    }
    double rn[N];
    if (EARLY && grp + gstride < ngroups) {   // next group's u column, in flight during the whole element
      load_column(grp + gstride, rn);
      if (grp + 2 * gstride < ngroups) prefetch_column(grp + 2 * gstride);
    }
    bsync();
    {  // P1: g0 on x-line (j=t0, k=t1) -> s0 (TR: in place)
      double L[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = (TR ? s0 : su)[mm + N * t0 + N2 * t1];
      if constexpr (EO) {
        double o[N];
        eo_line<P, 0>(L, o);
#pragma unroll
        for (int i = 0; i < N; ++i) s0[i + N * t0 + N2 * t1] = o[i];
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) s = fma(dmat<P>(0, i * N + mm + zero), L[mm], s);
          s0[i + N * t0 + N2 * t1] = s;
        }
      }
    }
    bsync();
    {  // P2: g1 on y-line (i=t0, k=t1), in place in su
      // y-line element j of line (i, k): natural su[i + n j + n^2 k], transposed su[j + n i + n^2 k]
      const int yb = TR ? N * t0 + N2 * t1 : t0 + N2 * t1;
      constexpr int ys = TR ? 1 : N;
      double L[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = su[yb + ys * mm];
      if constexpr (EO) {
        double o[N];
        eo_line<P, 1>(L, o);
#pragma unroll
        for (int j = 0; j < N; ++j) su[yb + ys * j] = o[j];
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double s = 0.0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) s = fma(dmat<P>(1, j * N + mm + zero), L[mm], s);
          su[yb + ys * j] = s;
        }
      }
    }
    bsync();
    if (GS) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    double vz[N];
    {  // P3: g2 = D u on the z-line in registers, w = G g, vz = D^T w2
      double g2a[N];   // g2 for every k, then overwritten by w2
      if constexpr (EO) {
        eo_line<P, 2>(ru, g2a);
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double g2 = 0.0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) g2 = fma(dmat<P>(2, k * N + mm + zero), ru[mm], g2);
          g2a[k] = g2;
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double G00, G01, G02, G11, G12, G22;
        if (GS) {
          const double* Gk = gE + gofs<N>(0, t, k);
          G00 = Gk[0]; G01 = Gk[N2]; G02 = Gk[2 * N2]; G11 = Gk[3 * N2]; G12 = Gk[4 * N2]; G22 = Gk[5 * N2];
        } else {
          const int kr = k;   // ring slot index (compile-time after unrolling)
          if (k + RG - 1 < N) {
#pragma unroll
            for (int c = 0; c < 6; ++c) gb[(kr + RG - 1) % RG][c] = __ldcs(Gg + gofs<N>(c, 0, k + RG - 1));
          }
          G00 = gb[kr % RG][0]; G01 = gb[kr % RG][1]; G02 = gb[kr % RG][2];
          G11 = gb[kr % RG][3]; G12 = gb[kr % RG][4]; G22 = gb[kr % RG][5];
        }
        const int idx = t + N2 * k;
        const int idy = TR ? t1 + N * t0 + N2 * k : idx;   // (t0, t1, k) in su's layout
        const double g0 = s0[idx], g1 = su[idy], g2 = g2a[k];
        s0[idx] = G00 * g0 + G01 * g1 + G02 * g2;
        su[idy] = G01 * g0 + G11 * g1 + G12 * g2;
        g2a[k] = G02 * g0 + G12 * g1 + G22 * g2;
      }
      if constexpr (EO) {
        eo_line<P, 3>(g2a, vz);
      } else {
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(dmat<P>(2, k * N + c + zero), g2a[k], s);
          vz[c] = s;
        }
      }
    }
    bsync();
    {  // factors consumed: next group's G (TMA from L2) and the L2 prefetch of the group after
      const long long nx = grp + gstride;
      if (nx < ngroups && threadIdx.x == 0) {
        if (GS) {
          fence_proxy_async_smem();
          bulk_load(sG, G + gfirst(nx) * 6 * N3, group_bytes(nx), bar);
        }
        if (PF == 2 && nx + gstride < ngroups) prefetch_group_l2(nx + gstride);
        else if (!GS && nx < ngroups) prefetch_group_l2(nx);
      }
    }
    if (!EARLY && grp + gstride < ngroups) {   // next group's u column, in flight during P4-P6
      load_column(grp + gstride, rn);
      if (grp + 2 * gstride < ngroups) prefetch_column(grp + 2 * gstride);
    }
    {  // P4: v0 = D^T w0 on x-line (j=t0, k=t1), in place in s0
      double L[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = s0[mm + N * t0 + N2 * t1];
      if constexpr (EO) {
        double o[N];
        eo_line<P, 4>(L, o);
#pragma unroll
        for (int a = 0; a < N; ++a) s0[a + N * t0 + N2 * t1] = o[a];
      } else {
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double s = 0.0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) s = fma(dmat<P>(3, mm * N + a + zero), L[mm], s);
          s0[a + N * t0 + N2 * t1] = s;
        }
      }
    }
    bsync();
    {  // P5: su = D^T w1 + v0 on y-line (i=t0, k=t1) (TR: su = Y in place; v0 is added in P6)
      const int yb = TR ? N * t0 + N2 * t1 : t0 + N2 * t1;
      constexpr int ys = TR ? 1 : N;
      double L[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = su[yb + ys * mm];
      if constexpr (EO) {
        double o[N];
        eo_line<P, 5>(L, o);
#pragma unroll
        for (int b = 0; b < N; ++b) su[yb + ys * b] = TR ? o[b] : o[b] + s0[t0 + N * b + N2 * t1];
      } else {
#pragma unroll
        for (int b = 0; b < N; ++b) {
          double s = TR ? 0.0 : s0[t0 + N * b + N2 * t1];
#pragma unroll
          for (int mm = 0; mm < N; ++mm) s = fma(dmat<P>(4, mm * N + b + zero), L[mm], s);
          su[yb + ys * b] = s;
        }
      }
    }
    // FU: the update piece attached to this group slot (plane set one or more layers behind)
    const long long pj = FU ? grp - f.gpl - f.shift : -1;
    if constexpr (FU) {
      const int cur_set = pj >= 0 ? (int)((unsigned)pj / (unsigned)f.gpl) : -1;
      const bool fl = acc_ln > 0 && acc_layer != ez, fs = acc_sn > 0 && acc_set != cur_set;
      if (threadIdx.x == 0) {
        // release the finished layer / set of the earlier slots (every thread passed block barriers since
        // their last RED / store)
        if (fl || fs) {
          fence_acq_rel_gpu();
          if (fl) red_add_u32(f.layer_done + acc_layer, (unsigned)acc_ln);
          if (fs) red_add_u32(f.upd_done + acc_set, (unsigned)acc_sn);
        }
        // plane sets whose ring slots this element layer's planes [ez p, (ez+1) p] reuse must be updated
        const int need = (ez * P + P - f.rp >= 0) ? (ez * P + P - f.rp) / P : -1;
        for (; chk_layer < need; ++chk_layer) spin_ge(f.upd_done + chk_layer + 1, (unsigned)f.gpl, f.err);
        // the piece's plane set is final once the element layers up to it are complete
        for (; lay_chk < cur_set; ++lay_chk) spin_ge(f.layer_done + lay_chk + 1, (unsigned)f.gpl, f.err);
      }
      if (fl) acc_ln = 0;
      if (fs) acc_sn = 0;
    }
    bsync();
    if (!waited) {
      TLMARK(g_tl_v4, 4, 2048, 1);
      pdl_wait();
      TLMARK(g_tl_v4, 4, 2048, 2);
      waited = true;
    }
    if (act) {  // P6: z-line (i=t0, j=t1): v = su + vz, scatter (own column of su)
      const bool own_xy = (t0 > 0 || ex == 0) && (t1 > 0 || ey == 0);
      const long long gxy = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1);
      const int kz0 = FU ? (ez * P) % f.rp : 0;   // ring slot of the element's bottom plane
      const uint64_t rpol = FU ? l2_evict_last_policy() : 0;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        bool bnd = false;
        if (DIR) { const int K = ez * P + c; bnd = bxy || K == m.Kb0 || K == m.Kb1; }
        const double xy = TR ? s0[t + N2 * c] + su[t1 + N * t0 + N2 * c] : su[t + N2 * c];
        if constexpr (FU) {
          int slot = kz0 + c;
          if (slot >= f.rp) slot -= f.rp;
          if (!bnd) ring_red(v + gxy + sxy * slot, xy + vz[c], rpol);
          else if (own_xy && (c > 0 || ez == 0)) ring_st(v + gxy + sxy * slot, u[gcol + sxy * c], rpol);   // A_D x = x (R4)
        } else if (IPS && t0 > 0 && t0 < P && t1 > 0 && t1 < P && c > 0 && c < P) v[gcol + sxy * c] = xy + vz[c];
        else if (COL) { if (!bnd) v[gcol + sxy * c] += xy + vz[c]; }
        else if (!bnd) atomicAdd(v + gcol + sxy * c, xy + vz[c]);
        else if (write_bnd && own_xy && (c > 0 || ez == 0)) v[gcol + sxy * c] = u[gcol + sxy * c];  // (I-M) u
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) ru[k] = rn[k];
    if constexpr (FU) {
      acc_layer = ez;   // (all elements of a group lie in one layer: checked by the launcher)
      ++acc_ln;
      if (pj >= 0) {
        acc_set = (int)((unsigned)pj / (unsigned)f.gpl);
        ++acc_sn;
        fused_piece<P, C::THREADS>(m, u, v, f, acc_set, (unsigned)pj - (unsigned)acc_set * (unsigned)f.gpl, threadIdx.x);
      }
    }
  }
  if constexpr (FU) {   // the update pieces attached to the slots after the last element group
    const long long npieces = (long long)m.nez * f.gpl;
    for (;; grp += gstride) {
      const long long pj = grp - f.gpl - f.shift;
      const int cur_set = (pj >= 0 && pj < npieces) ? (int)((unsigned)pj / (unsigned)f.gpl) : -1;
      const bool fl = acc_ln > 0, fs = acc_sn > 0 && acc_set != cur_set;
      bsync();
      if (threadIdx.x == 0 && (fl || fs)) {
        fence_acq_rel_gpu();
        if (fl) red_add_u32(f.layer_done + acc_layer, (unsigned)acc_ln);
        if (fs) red_add_u32(f.upd_done + acc_set, (unsigned)acc_sn);
      }
      acc_ln = 0;
      if (fs) acc_sn = 0;
      if (pj >= npieces) break;
      if (pj < 0) continue;
      if (threadIdx.x == 0) {
        for (; lay_chk < cur_set; ++lay_chk) spin_ge(f.layer_done + lay_chk + 1, (unsigned)f.gpl, f.err);
      }
      bsync();
      acc_set = cur_set;
      ++acc_sn;
      fused_piece<P, C::THREADS>(m, u, v, f, cur_set, (unsigned)pj - (unsigned)cur_set * (unsigned)f.gpl, threadIdx.x);
    }
  }
  TLMARK(g_tl_v4, 4, 2048, 3);
}


#include "k_apply_ks.cuh"
#include "k_apply_v6.cuh"

template <int P>
static void build_ks_tables(const std::vector<double>& D, const std::vector<double>& eo6, double* out) {
  using C = KsCfg<P>;
  using HT = HalfTab<P>;
  constexpr int N = P + 1, c = HT::c, R = HT::R, EOS = C::EOS;
  const double* set0 = eo6.data();             // even-odd D
  const double* set3 = eo6.data() + 3 * EOS;   // even-odd D^T
  for (int q = 0; q < EOS; ++q) out[q] = set0[q];
  for (int mat = 0; mat < 2; ++mat)
    for (int hh = 0; hh < 2; ++hh) {
      const double* tab = mat ? set3 : set0;
      double* h = out + EOS + mat * C::HMS + hh * HT::HSTR;
      for (int r = 0; r < HT::HSTR; ++r) {
        double val = 0.0;   // rows past c (hh = 1, c odd) and the padding stay zero
        if (r < R * c) {
          const int i = hh * R + r / c;
          if (i < c) val = tab[i * c + r % c];
        } else if (r < 2 * R * c) {
          const int i = hh * R + (r - R * c) / c;
          if (i < c) val = tab[c * c + i * c + (r - R * c) % c];
        } else if (r < 2 * R * c + R) {
          const int i = hh * R + (r - 2 * R * c);
          if (i < c) val = tab[2 * c * c + i];
        } else if (r < 2 * R * c + R + c) {
          val = tab[2 * c * c + c + (r - 2 * R * c - R)];
        }
        h[r] = val;
      }
    }
  for (int q = 0; q < N * N; ++q) out[EOS + 2 * C::HMS + q] = D[q];
}

static cudaError_t upload_ks_tables(int p, const std::vector<double>& D, const std::vector<double>& eo6) {
  if (p < kKsMinP || p % 2) return cudaSuccess;
  std::vector<double> t(kKsTabMax, 0.0);
  switch (p) {
    case 12: build_ks_tables<12>(D, eo6, t.data()); break;
    case 14: build_ks_tables<14>(D, eo6, t.data()); break;
    case 16: build_ks_tables<16>(D, eo6, t.data()); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaMemcpyToSymbol(g_kstab, t.data(), sizeof(double) * kKsTabMax, sizeof(double) * kKsTabMax * ((p - 12) / 2));
}

// ------------------------------------------------------------------------------------------
// K2 apply, thread per element (p <= 2): the whole element (n^3 <= 27 nodes) lives in registers,
// so there is no shared memory and no barrier; G streams through coalesced element-interleaved
// loads (GLayout), the gather and the fp64 REDs of neighbouring lanes touch neighbouring nodes.

template <int P, bool DIR>
__global__ void __launch_bounds__(128) k_apply_tpe(MeshDev m, const double* __restrict__ G,
                                                   const double* __restrict__ u, double* __restrict__ v,
                                                   int wait_mode, int write_bnd) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  using GL = GLayout<P>;
  const long long sxy = (long long)m.Mx * m.My;
  if (wait_mode == 2) pdl_wait();
  bool waited = (wait_mode != 1);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m.E; e += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const long long g0 = (long long)(ex * P) + (long long)m.Mx * (ey * P) + sxy * (long long)(ez * P);
    double ue[N3], ve[N3];
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const int l = a + N * (b + N * c);
          bool bnd = false;
          if (DIR) {
            const int I = ex * P + a, J = ey * P + b, K = ez * P + c;
            bnd = I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == m.Kb0 || K == m.Kb1;
          }
          ue[l] = bnd ? 0.0 : __ldg(u + g0 + a + (long long)m.Mx * b + sxy * c);
          ve[l] = 0.0;
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double d0 = 0, d1 = 0, d2 = 0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            d0 = fma(dmat<P>(0, i * N + mm), ue[mm + N * (j + N * k)], d0);
            d1 = fma(dmat<P>(0, j * N + mm), ue[i + N * (mm + N * k)], d1);
            d2 = fma(dmat<P>(0, k * N + mm), ue[i + N * (j + N * mm)], d2);
          }
          const int ij = i + N * j;
          const double G00 = __ldcs(G + GL::off(e, 0, ij, k)), G01 = __ldcs(G + GL::off(e, 1, ij, k));
          const double G02 = __ldcs(G + GL::off(e, 2, ij, k)), G11 = __ldcs(G + GL::off(e, 3, ij, k));
          const double G12 = __ldcs(G + GL::off(e, 4, ij, k)), G22 = __ldcs(G + GL::off(e, 5, ij, k));
          const double w0 = G00 * d0 + G01 * d1 + G02 * d2;
          const double w1 = G01 * d0 + G11 * d1 + G12 * d2;
          const double w2 = G02 * d0 + G12 * d1 + G22 * d2;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            ve[mm + N * (j + N * k)] = fma(dmat<P>(0, i * N + mm), w0, ve[mm + N * (j + N * k)]);
            ve[i + N * (mm + N * k)] = fma(dmat<P>(0, j * N + mm), w1, ve[i + N * (mm + N * k)]);
            ve[i + N * (j + N * mm)] = fma(dmat<P>(0, k * N + mm), w2, ve[i + N * (j + N * mm)]);
          }
        }
    if (!waited) {
      pdl_wait();
      waited = true;
    }
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          bool bnd = false;
          if (DIR) {
            const int I = ex * P + a, J = ey * P + b, K = ez * P + c;
            bnd = I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == m.Kb0 || K == m.Kb1;
          }
          const long long g = g0 + a + (long long)m.Mx * b + sxy * c;
          if (!bnd) atomicAdd(v + g, ve[a + N * (b + N * c)]);
          else if (write_bnd && (a > 0 || ex == 0) && (b > 0 || ey == 0) && (c > 0 || ez == 0)) v[g] = u[g];
        }
  }
}

// Export of the factors in the canonical layout [E][k][6][n^2] whatever the internal layout.
template <int P>
__global__ void k_export_geometry(MeshDev m, const double* __restrict__ G, double* __restrict__ out) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < m.E * 6 * N3;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long e = idx / (6 * N3);
    const int r = (int)(idx - e * 6 * N3);
    const int k = r / (6 * N2), c = (r / N2) % 6, ij = r % N2;
    out[idx] = G[GLayout<P>::off(e, c, ij, k)];
  }
}

// ------------------------------------------------------------------------------------------
// K3 diagonal: for node (a,b,c) of element e
//   sum_i D[i][a]^2 G00(i,b,c) + sum_j D[j][b]^2 G11(a,j,c) + sum_k D[k][c]^2 G22(a,b,k)
//   + 2 D[a][a] D[b][b] G01(a,b,c) + 2 D[a][a] D[c][c] G02(a,b,c) + 2 D[b][b] D[c][c] G12(a,b,c)

template <int P>
__global__ void __launch_bounds__(256) k_diag(MeshDev m, int bc, const double* __restrict__ G, double* d) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  __shared__ double sD[N * N];
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) sD[t] = dmat<P>(0, t);
  __syncthreads();
  const long long total = m.E * N3;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long e = idx / N3;
    int l = (int)(idx - e * N3);
    int a = l % N, b = (l / N) % N, c = l / N2;
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    long long g = (long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c));
    if (bc == 0 && lattice_boundary(m, g)) continue;
    using GL = GLayout<P>;
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += sD[i * N + a] * sD[i * N + a] * G[GL::off(e, 0, i + N * b, c)];
    for (int j = 0; j < N; ++j) s += sD[j * N + b] * sD[j * N + b] * G[GL::off(e, 3, a + N * j, c)];
    for (int k = 0; k < N; ++k) s += sD[k * N + c] * sD[k * N + c] * G[GL::off(e, 5, a + N * b, k)];
    const double da = sD[a * N + a], db = sD[b * N + b], dc = sD[c * N + c];
    const int ab = a + N * b;
    s += 2.0 * da * db * G[GL::off(e, 1, ab, c)] + 2.0 * da * dc * G[GL::off(e, 2, ab, c)] +
         2.0 * db * dc * G[GL::off(e, 4, ab, c)];
    atomicAdd(d + g, s);
  }
}

// ------------------------------------------------------------------------------------------
// Load vector of u* = sin(pi x) sin(pi y) sin(pi z).

template <int P>
__global__ void __launch_bounds__(256) k_load(MeshDev m, double* f) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  __shared__ double sD[N * N], sx[N], sw[N];
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) sD[t] = dmat<P>(0, t);
  for (int t = threadIdx.x; t < N; t += blockDim.x) { sx[t] = c_xw[0][xOffset(P) + t]; sw[t] = c_xw[1][xOffset(P) + t]; }
  __syncthreads();
  const double pi = 3.14159265358979323846;
  const long long total = m.E * N3;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long e = idx / N3;
    int q = (int)(idx - e * N3);
    int i = q % N, j = (q / N) % N, k = q / N2;
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    long long g = (long long)(ex * P + i) + (long long)m.Mx * ((long long)(ey * P + j) + (long long)m.My * (ez * P + k));
    if (lattice_boundary(m, g)) continue;
    double J[3][3];
    jacobian<P>(m, sD, sx, ex, ey, ez, i, j, k, J);
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                 J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                 J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double X[3];
    node_pos<P>(m, sx, ex, ey, ez, i, j, k, X);
    double s0 = sinpi(X[0]), s1 = sinpi(X[1]), s2 = sinpi(X[2]);
    double c0 = cospi(X[0]), c1 = cospi(X[1]), c2 = cospi(X[2]);
    double us = s0 * s1 * s2;
    double gu[3] = {pi * c0 * s1 * s2, pi * s0 * c1 * s2, pi * s0 * s1 * c2};
    double mu = coeff_mu(m, X[0], X[1], X[2]);
    double gm[3];
    coeff_grad(m, X[0], X[1], X[2], mu, gm);
    double fx = 3.0 * pi * pi * mu * us - (gm[0] * gu[0] + gm[1] * gu[1] + gm[2] * gu[2]);
    atomicAdd(f + g, sw[i] * sw[j] * sw[k] * det * fx);
  }
}

// ------------------------------------------------------------------------------------------
// vector kernels that need the lattice

// v = (I - M) u (bc 0) or 0 (bc 1).  One warp per lattice row (J, K): the only integer divisions
// are per row, and each lane writes consecutive doubles of the row.
__global__ void __launch_bounds__(256) k_init(MeshDev m, int bc, const double* __restrict__ u, double bval,
                                              double* __restrict__ v, int early) {
  // early: the grid is one resident wave (8 blocks per SM) and triggers its programmatic dependent
  // (the persistent apply) at once, so the apply's launch overlaps this kernel; the apply waits
  // (griddepcontrol.wait) only before its first scatter.  Safe: every init block is already running
  // when the dependent launches, and an init block never waits on anything.
  TLMARK(g_tl_init, 2, 4096, 0);
  if (early) pdl_trigger();
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)m.My * m.Mz;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  auto row_bnd = [&](long long r) {
    const unsigned r32 = (unsigned)r;
    const int K = (int)(r32 / (unsigned)m.My), J = (int)(r32 - (unsigned)K * (unsigned)m.My);
    return (bc == 0) && (J == 0 || J == m.My - 1 || K == m.Kb0 || K == m.Kb1);
  };
  // rows, one warp each: Dirichlet rows copied (bnd value), the others zeroed between their two x-face
  // nodes -- stores only, so a warp never waits on a load in a row it does not own a boundary in
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wstride) {
    double* vr = v + r * m.Mx;
    if (row_bnd(r)) {
      const double* ur = u ? u + r * m.Mx : nullptr;
#pragma unroll 4
      for (int I = lane; I < m.Mx; I += 32) vr[I] = ur ? ur[I] : bval;
    } else {
      const int lo = (bc == 0) ? 1 : 0;
      for (int I = lo + lane; I < m.Mx - lo; I += 32) vr[I] = 0.0;
    }
  }
  // the x-face nodes (I = 0, Mx - 1) of the other rows, one thread per row: the boundary loads of
  // different rows are independent and overlap
  if (bc == 0) {
    const long long tstride = (long long)gridDim.x * blockDim.x;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += tstride) {
      if (row_bnd(r)) continue;
      const long long g0 = r * m.Mx, g1 = g0 + m.Mx - 1;
      const double a = u ? u[g0] : bval, b = u ? u[g1] : bval;
      v[g0] = a;
      v[g1] = b;
    }
  }
  if (!early) pdl_trigger();   // after this block's work (see k_cheb_update)
#ifdef SFMG_TIMELINE
  __syncthreads();
  TLMARK(g_tl_init, 2, 4096, 1);
#endif
}

// v = 0 before a p <= 2 standalone apply, whose canonical owner elements store the boundary values
// (write_bnd).  Pure 16-byte stores, one small block per SM that triggers its programmatic dependent at
// once, so the apply's blocks start during the zeroing and only their first scatter waits
// (griddepcontrol.wait).  (For p >= 3 the row-wise k_init + owner-free scatter measured faster; the
// fused in-kernel init with a grid barrier and this kernel in front of k_apply_v4 were both slower,
// profiles/r02_experiments.md.)
constexpr int kZeroThreads = 64;
__global__ void __launch_bounds__(kZeroThreads) k_zero(double* __restrict__ v, long long n) {
  pdl_trigger();
  const long long n2 = n >> 1;   // v is 16-byte aligned (checked by the launcher)
  const long long q0 = n2 * blockIdx.x / gridDim.x, q1 = n2 * (blockIdx.x + 1) / gridDim.x;
  double2* v2 = reinterpret_cast<double2*>(v);
  for (long long q = q0 + threadIdx.x; q < q1; q += blockDim.x) v2[q] = make_double2(0.0, 0.0);
  if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) v[n - 1] = 0.0;
}

__global__ void k_cheb_update(MeshDev m, const double* cur, const double* prev, double* out,
                              const double* __restrict__ b, double* y, const double* __restrict__ dinv,
                              double c1, double c2, int early) {
  if (early) pdl_trigger();   // one resident wave: see k_init
  pdl_wait();   // launched as the apply's programmatic dependent
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < m.N; g += (long long)gridDim.x * blockDim.x) {
    const double xc = cur[g];
    const double xp = (c1 != 0.0) ? prev[g] : 0.0;
    const double xn = xc + c1 * (xc - xp) + c2 * dinv[g] * (b[g] - y[g]);
    out[g] = xn;
    y[g] = lattice_boundary(m, g) ? xn : 0.0;
  }
  if (!early) pdl_trigger();   // after this block's work: every block of this grid is then resident or
                               // done, so the dependent persistent apply can never starve it of SM resources
}

__global__ void k_export_maps(MeshDev m, int32_t* l2g, uint8_t* mask, uint8_t* col) {
  const int P = m.p, N = P + 1;
  const long long N3 = (long long)N * N * N;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l2g)
    for (long long idx = t0; idx < m.E * N3; idx += stride) {
      long long e = idx / N3;
      int l = (int)(idx - e * N3);
      int a = l % N, b = (l / N) % N, c = l / (N * N);
      int ex, ey, ez;
      elem_coords(m, e, ex, ey, ez);
      l2g[idx] = (int32_t)((long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c)));
    }
  if (mask)
    for (long long g = t0; g < m.N; g += stride) mask[g] = lattice_boundary(m, g) ? 1 : 0;
  if (col)
    for (long long e = t0; e < m.E; e += stride) {
      int ex, ey, ez;
      elem_coords(m, e, ex, ey, ez);
      col[e] = (uint8_t)((ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2));
    }
}

// ------------------------------------------------------------------------------------------
// K8 coarse CG (R13): one CTA runs the whole unpreconditioned CG loop on the p = 1 level, so a
// V-cycle needs no host synchronisation.  Vectors live in global memory (L2-resident at these
// sizes) and are re-read with ld.global.cg, bypassing the incoherent L1.


template <int P>
__device__ void cta_apply(const MeshDev& m, const double* __restrict__ G, const double* x, double* y) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  for (long long g = threadIdx.x; g < m.N; g += blockDim.x) y[g] = lattice_boundary(m, g) ? __ldcg(x + g) : 0.0;
  __syncthreads();
  for (long long e = threadIdx.x; e < m.E; e += blockDim.x) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    double ue[N3], ve[N3];
    long long gl[N3];
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const int l = a + N * (b + N * c);
          long long g = (long long)(ex * P + a) + (long long)m.Mx * ((long long)(ey * P + b) + (long long)m.My * (ez * P + c));
          const bool bnd = lattice_boundary(m, g);
          gl[l] = bnd ? -1 : g;
          ue[l] = bnd ? 0.0 : __ldcg(x + g);
          ve[l] = 0.0;
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double g0 = 0, g1 = 0, g2 = 0;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            g0 = fma(dmat<P>(0, i * N + mm), ue[mm + N * (j + N * k)], g0);
            g1 = fma(dmat<P>(0, j * N + mm), ue[i + N * (mm + N * k)], g1);
            g2 = fma(dmat<P>(0, k * N + mm), ue[i + N * (j + N * mm)], g2);
          }
          const int ij = i + N * j;
          using GL = GLayout<P>;
          const double G00 = G[GL::off(e, 0, ij, k)], G01 = G[GL::off(e, 1, ij, k)], G02 = G[GL::off(e, 2, ij, k)];
          const double G11 = G[GL::off(e, 3, ij, k)], G12 = G[GL::off(e, 4, ij, k)], G22 = G[GL::off(e, 5, ij, k)];
          const double w0 = G00 * g0 + G01 * g1 + G02 * g2;
          const double w1 = G01 * g0 + G11 * g1 + G12 * g2;
          const double w2 = G02 * g0 + G12 * g1 + G22 * g2;
#pragma unroll
          for (int mm = 0; mm < N; ++mm) {
            ve[mm + N * (j + N * k)] = fma(dmat<P>(0, i * N + mm), w0, ve[mm + N * (j + N * k)]);
            ve[i + N * (mm + N * k)] = fma(dmat<P>(0, j * N + mm), w1, ve[i + N * (mm + N * k)]);
            ve[i + N * (j + N * mm)] = fma(dmat<P>(0, k * N + mm), w2, ve[i + N * (j + N * mm)]);
          }
        }
#pragma unroll
    for (int l = 0; l < N3; ++l)
      if (gl[l] >= 0) atomicAdd(y + gl[l], ve[l]);
  }
  __threadfence_block();
  __syncthreads();
}

// Shared-memory variant (N <= kCoarseSmemN): x, r, p, q live in smem (the operator scatter uses
// shared-memory fp64 atomics), the geometric factors are read through the L1-cached read-only path.
template <int P>
__global__ void __launch_bounds__(512) k_coarse_cg_smem(MeshDev m, const double* __restrict__ G,
                                                        const double* __restrict__ b, double* __restrict__ xout,
                                                        double* scal, double rtol, int maxit) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  using GL = GLayout<P>;
  extern __shared__ double cg_sm[];
  __shared__ double red[32];
  const long long n = m.N;
  double* x = cg_sm;
  double* r = x + n;
  double* p = r + n;
  double* q = p + n;
  double rr = 0.0;
  for (long long g = threadIdx.x; g < n; g += blockDim.x) {
    const double bg = b[g];
    x[g] = 0.0; r[g] = bg; p[g] = bg;
    rr += bg * bg;
  }
  rr = block_sum(rr, red);
  const double bn = sqrt(rr);
  int it = 0, status = 0;
  if (bn > 0.0) {
    for (; it < maxit; ++it) {
      if (sqrt(rr) <= rtol * bn) break;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) q[g] = 0.0;
      __syncthreads();
      for (long long e = threadIdx.x; e < m.E; e += blockDim.x) {   // q = A_D p on interior rows
        int ex, ey, ez;
        elem_coords(m, e, ex, ey, ez);
        double ue[N3], ve[N3];
        int gl[N3];
#pragma unroll
        for (int c = 0; c < N; ++c)
#pragma unroll
          for (int bb = 0; bb < N; ++bb)
#pragma unroll
            for (int a = 0; a < N; ++a) {
              const int l = a + N * (bb + N * c);
              const int I = ex * P + a, J = ey * P + bb, K = ez * P + c;
              const bool bnd = I == 0 || I == m.Mx - 1 || J == 0 || J == m.My - 1 || K == 0 || K == m.Mz - 1;
              const int g = I + m.Mx * (J + m.My * K);
              gl[l] = bnd ? -1 : g;
              ue[l] = bnd ? 0.0 : p[g];
              ve[l] = 0.0;
            }
#pragma unroll
        for (int k = 0; k < N; ++k)
#pragma unroll
          for (int j = 0; j < N; ++j)
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double d0 = 0, d1 = 0, d2 = 0;
#pragma unroll
              for (int mm = 0; mm < N; ++mm) {
                d0 = fma(dmat<P>(0, i * N + mm), ue[mm + N * (j + N * k)], d0);
                d1 = fma(dmat<P>(0, j * N + mm), ue[i + N * (mm + N * k)], d1);
                d2 = fma(dmat<P>(0, k * N + mm), ue[i + N * (j + N * mm)], d2);
              }
              const int ij = i + N * j;
              const double G00 = __ldg(G + GL::off(e, 0, ij, k)), G01 = __ldg(G + GL::off(e, 1, ij, k));
              const double G02 = __ldg(G + GL::off(e, 2, ij, k)), G11 = __ldg(G + GL::off(e, 3, ij, k));
              const double G12 = __ldg(G + GL::off(e, 4, ij, k)), G22 = __ldg(G + GL::off(e, 5, ij, k));
              const double w0 = G00 * d0 + G01 * d1 + G02 * d2;
              const double w1 = G01 * d0 + G11 * d1 + G12 * d2;
              const double w2 = G02 * d0 + G12 * d1 + G22 * d2;
#pragma unroll
              for (int mm = 0; mm < N; ++mm) {
                ve[mm + N * (j + N * k)] = fma(dmat<P>(0, i * N + mm), w0, ve[mm + N * (j + N * k)]);
                ve[i + N * (mm + N * k)] = fma(dmat<P>(0, j * N + mm), w1, ve[i + N * (mm + N * k)]);
                ve[i + N * (j + N * mm)] = fma(dmat<P>(0, k * N + mm), w2, ve[i + N * (j + N * mm)]);
              }
            }
#pragma unroll
        for (int l = 0; l < N3; ++l)
          if (gl[l] >= 0) atomicAdd(q + gl[l], ve[l]);
      }
      __syncthreads();
      double pq = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) pq += p[g] * q[g];
      pq = block_sum(pq, red);
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rr / pq;
      double rn = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) {
        x[g] += alpha * p[g];
        const double rg = r[g] - alpha * q[g];
        r[g] = rg;
        rn += rg * rg;
      }
      rn = block_sum(rn, red);
      const double beta = rn / rr;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) p[g] = r[g] + beta * p[g];
      rr = rn;
      __syncthreads();
    }
  }
  __syncthreads();
  for (long long g = threadIdx.x; g < n; g += blockDim.x) xout[g] = x[g];
  if (threadIdx.x == 0) { scal[8] = (double)it; scal[9] = sqrt(rr); scal[10] = (double)status; }
}

template <int P>
__global__ void __launch_bounds__(256) k_coarse_cg(MeshDev m, const double* __restrict__ G, const double* b,
                                                    double* x, double* r, double* p, double* q, double* scal,
                                                    double rtol, int maxit) {
  __shared__ double red[32];
  const long long n = m.N;
  double rr = 0.0;
  for (long long g = threadIdx.x; g < n; g += blockDim.x) {
    const double bg = b[g];
    x[g] = 0.0; r[g] = bg; p[g] = bg;
    rr += bg * bg;
  }
  rr = block_sum(rr, red);
  const double bn = sqrt(rr);
  int it = 0, status = 0;
  if (bn > 0.0) {
    for (; it < maxit; ++it) {
      if (sqrt(rr) <= rtol * bn) break;
      __syncthreads();
      cta_apply<P>(m, G, p, q);
      double pq = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) pq += __ldcg(p + g) * __ldcg(q + g);
      pq = block_sum(pq, red);
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rr / pq;
      double rn = 0.0;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) {
        x[g] = __ldcg(x + g) + alpha * __ldcg(p + g);
        const double rg = __ldcg(r + g) - alpha * __ldcg(q + g);
        r[g] = rg;
        rn += rg * rg;
      }
      rn = block_sum(rn, red);
      const double beta = rn / rr;
      for (long long g = threadIdx.x; g < n; g += blockDim.x) p[g] = __ldcg(r + g) + beta * __ldcg(p + g);
      rr = rn;
      __threadfence_block();
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) { scal[8] = (double)it; scal[9] = sqrt(rr); scal[10] = (double)status; }
}

// ------------------------------------------------------------------------------------------
// launchers

static int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  if (b > 148LL * 16) b = 148LL * 16;
  if (b < 1) b = 1;
  return (int)b;
}

#define SFMG_DISPATCH_P(p, F, ...)  \
  switch (p) {                      \
    case 1: F<1>(__VA_ARGS__); break;   \
    case 2: F<2>(__VA_ARGS__); break;   \
    case 3: F<3>(__VA_ARGS__); break;   \
    case 4: F<4>(__VA_ARGS__); break;   \
    case 5: F<5>(__VA_ARGS__); break;   \
    case 6: F<6>(__VA_ARGS__); break;   \
    case 7: F<7>(__VA_ARGS__); break;   \
    case 8: F<8>(__VA_ARGS__); break;   \
    case 9: F<9>(__VA_ARGS__); break;   \
    case 10: F<10>(__VA_ARGS__); break; \
    case 11: F<11>(__VA_ARGS__); break; \
    case 12: F<12>(__VA_ARGS__); break; \
    case 13: F<13>(__VA_ARGS__); break; \
    case 14: F<14>(__VA_ARGS__); break; \
    case 15: F<15>(__VA_ARGS__); break; \
    case 16: F<16>(__VA_ARGS__); break; \
    default: return cudaErrorInvalidValue; \
  }

template <int P>
static void geometry_p(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
  k_geometry<P><<<grid_for(m.E * N3, 256), 256, 0, s>>>(m, G, bad);
}
cudaError_t launch_geometry(const MeshDev& m, double* G, int* bad, cudaStream_t s) {
  if (m.dim == 2) return launch_geometry_2d(m, G, bad, s);
  if (m.quad) return launch_geometry_gauss(m, G, bad, s);
  SFMG_DISPATCH_P(m.p, geometry_p, m, G, bad, s);
  return cudaGetLastError();
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// sets the dynamic smem limit of kernel k once per device and returns its resident blocks per SM
template <typename K>
static cudaError_t persistent_blocks(IntPerDevice& cache, K k, int threads, size_t smem, int& per_sm) {
  return cache.get(per_sm, [&](int& v) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, threads, smem);
  });
}

// The k-split cluster kernel is correct (parity-tested) but measured slower than k_apply_v4 at p = 16
// (config 3: 76 vs 59.5 us per element-kernel launch; profiles/r02_experiments.md), so it is opt-in:
// SFMG_KSPLIT=1.
static bool ks_enabled() {
  static const bool on = [] {
    const char* e = getenv("SFMG_KSPLIT");
    return e && e[0] == '1';
  }();
  return on;
}

static bool color_enabled() {
  static const bool on = [] {
    const char* e = getenv("SFMG_COLOR");
    return e && e[0] == '1';
  }();
  return on;
}

// SFMG_V6=1: the two-blocks-per-SM kernel for even p >= 12 (k_apply_v6.cuh; measured in
// profiles/r02_experiments.md)
static bool v6_enabled() {
  static const bool on = [] {
    const char* e = getenv("SFMG_V6");
    return e && e[0] == '1';
  }();
  return on;
}
template <int P, bool DIR>
static cudaError_t launch_v6(const MeshDev& m, const double* G, const double* u, double* v, int wait_mode,
                             int write_bnd, cudaStream_t s) {
  using C = V6Cfg<P>;
  static IntPerDevice occ;
  int resident = 0;
  cudaError_t e = persistent_blocks(occ, k_apply_v6<P, DIR>, C::THREADS, C::SMEM, resident);
  if (e) return e;
  long long grid = (long long)resident * num_sms();
  if (grid > m.E) grid = m.E;
  MeshDev mm = m;
  mm.pdl_early = early_pdl(m) ? 1 : 0;
  return launch_pdl(k_apply_v6<P, DIR>, (unsigned)grid, (unsigned)C::THREADS, C::SMEM, s, mm, G, u, v, wait_mode,
                    write_bnd);
}

template <int P, bool DIR, bool IPS>
static cudaError_t launch_ks(const MeshDev& m, const double* G, const double* u, double* v, int wait_mode,
                             int write_bnd, cudaStream_t s) {
  using C = KsCfg<P>;
  static IntPerDevice clusters;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int ncl = 0;
  cudaError_t e = clusters.get(ncl, [&](int& n) {
    cudaError_t r = cudaFuncSetAttribute(k_apply_ks<P, DIR, IPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (r) return r;
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(2 * num_sms());
    q.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(&n, k_apply_ks<P, DIR, IPS>, &q);
  });
  if (e) return e;
  long long grid = ncl < m.E ? ncl : m.E;
  cfg.gridDim = dim3((unsigned)(2 * grid));
  return cudaLaunchKernelEx(&cfg, k_apply_ks<P, DIR, IPS>, m, G, u, v, wait_mode, write_bnd);
}

template <int P, bool DIR>
static cudaError_t apply_pd(const MeshDev& m, const double* G, const double* u, double* v, int wait_mode,
                            int write_bnd, cudaStream_t s) {
  if constexpr (P <= 2) {
    static IntPerDevice occ;
    int per_sm = 0;
    cudaError_t e = persistent_blocks(occ, k_apply_tpe<P, DIR>, 128, 0, per_sm);
    if (e) return e;
    long long blocks = (m.E + 127) / 128;
    if (blocks > (long long)per_sm * num_sms()) blocks = (long long)per_sm * num_sms();
    return launch_pdl(k_apply_tpe<P, DIR>, (unsigned)blocks, 128, 0, s, m, G, u, v, wait_mode, write_bnd);
  } else {
    if constexpr (P >= kKsMinP && P % 2 == 0) {   // even orders: the even-odd line products keep the
                                                   // kernel within the register file (odd p spills)
      if (v6_enabled()) return launch_v6<P, DIR>(m, G, u, v, wait_mode, write_bnd, s);
      if (ks_enabled()) {
        MeshDev mm = m;
        mm.pdl_early = early_pdl(m) ? 1 : 0;
        if (!mm.pdl_early && wait_mode == 1) return launch_ks<P, DIR, true>(mm, G, u, v, wait_mode, write_bnd, s);
        return launch_ks<P, DIR, false>(mm, G, u, v, wait_mode, write_bnd, s);
      }
    }
    constexpr bool GS = (P <= 8);
    using C = V4Cfg<P, GS>;
    static IntPerDevice occ, occ_ips;
    int resident = 0;
    cudaError_t e;
    if constexpr (GS && C::EPB == 1) {
      if (color_enabled()) {   // measurement variant: eight coloured launches with plain load-add-stores
        static IntPerDevice occ_col;
        auto kc = k_apply_v4<P, DIR, GS, false, false, true>;
        if ((e = persistent_blocks(occ_col, kc, C::THREADS, C::SMEM, resident))) return e;
        MeshDev mm = m;
        mm.pdl_early = 0;
        for (int c = 0; c < 8; ++c) {
          const long long nc = (long long)((m.nex - (c & 1) + 1) / 2) * ((m.ney - ((c >> 1) & 1) + 1) / 2) *
                               ((m.nez - ((c >> 2) & 1) + 1) / 2);
          if (nc == 0) continue;
          long long grid = (long long)resident * num_sms();
          if (grid > nc) grid = nc;
          FusedArgs fa;
          fa.color = c;
          // (programmatic launch: a coloured launch starts its factor prefetch during the previous one's
          // tail and waits for its completion before the gather)
          if ((e = launch_pdl(kc, (unsigned)grid, (unsigned)C::THREADS, C::SMEM, s, mm, G, u, v, nc,
                              c == 0 ? wait_mode : 2, write_bnd, fa)))
            return e;
        }
        return cudaSuccess;
      }
    }
    e = persistent_blocks(occ, k_apply_v4<P, DIR, GS>, C::THREADS, C::SMEM, resident);
    if (e) return e;
    const long long groups = (m.E + C::EPB - 1) / C::EPB;
    long long grid = (long long)resident * num_sms();
    if (grid > groups) grid = groups;
    MeshDev mm = m;
    mm.pdl_early = early_pdl(m) ? 1 : 0;
    if (!mm.pdl_early && wait_mode == 1) {   // right after the v init (measured: config 4 apply -5 %; after a
                                             // Chebyshev update +2 %)
      int r2 = 0;
      if ((e = persistent_blocks(occ_ips, k_apply_v4<P, DIR, GS, true>, C::THREADS, C::SMEM, r2))) return e;
      return launch_pdl(k_apply_v4<P, DIR, GS, true>, (unsigned)grid, (unsigned)C::THREADS, C::SMEM, s, mm, G, u, v,
                        groups, wait_mode, write_bnd, FusedArgs{});
    }
    return launch_pdl(k_apply_v4<P, DIR, GS>, (unsigned)grid, (unsigned)C::THREADS, C::SMEM, s, mm, G, u, v, groups,
                      wait_mode, write_bnd, FusedArgs{});
  }
}
template <int P>
static void apply_p(const MeshDev& m, int bc, const double* G, const double* u, double* v, int wait_mode,
                    int write_bnd, cudaStream_t s, cudaError_t* err) {
  *err = (bc == 0) ? apply_pd<P, true>(m, G, u, v, wait_mode, write_bnd, s)
                   : apply_pd<P, false>(m, G, u, v, wait_mode, write_bnd, s);
}
cudaError_t launch_apply(const MeshDev& m, int bc, const double* G, const double* u, double* v, int wait_mode,
                         int write_bnd, cudaStream_t s) {
  if (m.dim == 2) return launch_apply_2d(m, bc, G, u, v, s);   // v initialised by the caller (no PDL)
  if (m.quad) return launch_apply_gauss(m, bc, G, u, v, s);   // v initialised by the caller (no PDL)
  cudaError_t err = cudaSuccess;
  SFMG_DISPATCH_P(m.p, apply_p, m, bc, G, u, v, wait_mode, write_bnd, s, &err);
  if (err) return err;
  return cudaGetLastError();
}

// ---- fused Chebyshev step / apply for vectors beyond L2 (k_apply_v4<.., FU>)

// SFMG_FUSED=1: the fused kernel wherever it applies (tests, measurements); otherwise never
static int fused_env() {
  static const int v = [] {
    const char* e = getenv("SFMG_FUSED");
    return e ? atoi(e) : -1;
  }();
  return v;
}
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
template <int P>
static constexpr int fused_epb() {
  if constexpr (P >= 3 && P <= 8) return V4Cfg<P, true>::EPB;
  return 0;
}
static int fused_epb_of(int p) {
  switch (p) {
    case 3: return fused_epb<3>();
    case 4: return fused_epb<4>();
    case 5: return fused_epb<5>();
    case 6: return fused_epb<6>();
    case 7: return fused_epb<7>();
    case 8: return fused_epb<8>();
  }
  return 0;
}
static int fused_ring_planes(const MeshDev& m) {
  static const int extra = env_int("SFMG_FUSED_RING_EXTRA", 0);
  int rp = 3 * m.p + 1 + extra;   // >= 3 p + 1: the pieces may lag their layer by a grid round (launcher)
  if (rp < 2 * m.p + 1) rp = 2 * m.p + 1;
  return rp > m.Mz ? m.Mz : rp;
}
size_t fused_scratch_doubles(const MeshDev& m) {
  return (size_t)fused_ring_planes(m) * m.Mx * m.My + (size_t)m.nez + 8;   // ring, counters (2 nez + 1 ints)
}
bool fused_available(const MeshDev& m) {
  const int mode = fused_env();
  if (mode == 0 || m.dim != 3 || m.quad) return false;
  const int epb = fused_epb_of(m.p);
  if (epb == 0 || m.nez < 3) return false;
  if (((long long)m.nex * m.ney) % epb) return false;       // every group inside one element layer
  if (m.N >= (1ll << 32)) return false;                      // 32-bit lattice arithmetic in the updater
  if (fused_scratch_doubles(m) > (size_t)m.N) return false;  // the ring lives in the level's y vector
  if (2 * m.p + 1 > m.Mz) return false;
  // opt-in: measured slower than the unfused step (config 4: 4.0-4.1 vs 3.6 ms; DESIGN.md section 6,
  // profiles/r02_experiments.md) although its DRAM traffic is the algorithmic 1.04x with
  // SFMG_L2_PERSIST_MB=64
  return mode == 1;
}

template <int P>
static void fused_p(const MeshDev& m, const double* G, const double* cur, double* scratch, FusedArgs f,
                    cudaStream_t s, cudaError_t* err) {
  if constexpr (P >= 3 && P <= 8) {
    using C = V4Cfg<P, true>;
    auto kern = k_apply_v4<P, true, true, false, true>;
    static IntPerDevice occ;
    int resident = 0;
    constexpr int threads = C::THREADS;
    if ((*err = persistent_blocks(occ, kern, threads, C::SMEM, resident))) return;
    const long long groups = m.E / C::EPB;
    long long grid = (long long)resident * num_sms();
    if (grid > groups) grid = groups;
    f.gpl = ((long long)m.nex * m.ney) / C::EPB;
    auto even_chunk = [&](long long nodes) {   // ceil((nodes + 1) / gpl), rounded up to even
      long long c = (nodes + 1 + f.gpl - 1) / f.gpl;
      return (unsigned)((c + 1) & ~1ll);
    };
    const long long sxy = (long long)m.Mx * m.My;
    f.chunk = even_chunk((long long)P * sxy);
    f.chunk_last = even_chunk((long long)(P + 1) * sxy);
    // A piece runs after its slot's scatter, and a scatter waits for the plane sets whose ring slots it
    // reuses (sets <= M + 1 - ceil(rp / p) for element layer M); those must be attached to earlier
    // slots: shift <= (ceil(rp / p) - 3) gpl.  rp = 2 p + 1 allows no shift, rp >= 3 p + 1 one grid round.
    static const int shift_rounds = env_int("SFMG_FUSED_SHIFT", 1);
    const long long max_shift = (long long)((f.rp + P - 1) / P - 3) * f.gpl;
    f.shift = grid * shift_rounds;
    if (f.shift > max_shift) f.shift = max_shift;
    if (f.shift < 0) f.shift = 0;
    MeshDev mm = m;
    mm.pdl_early = 0;
    // plain launch (no programmatic overlap): every block is resident and nothing of the previous step
    // is still running when the first spin-wait starts
    kern<<<(unsigned)grid, threads, C::SMEM, s>>>(mm, G, cur, scratch, groups, 0, 0, f);
    *err = cudaGetLastError();
  } else {
    *err = cudaErrorInvalidValue;
  }
}

// One fused step on the whole lattice: mode 0 out = cur + c1 (cur - prev) + c2 dinv (b - A_D cur);
// mode 1 out = A_D cur.  scratch: fused_scratch_doubles(m) doubles whose ring part is all zero (it is
// left all zero).  All vectors 16-byte aligned; out may alias prev or cur.
cudaError_t launch_fused_step(const MeshDev& m, const double* G, const double* cur, const double* prev, double* out,
                              const double* b, const double* dinv, double* scratch, double c1, double c2, int mode,
                              cudaStream_t s) {
  FusedArgs f;
  f.prev = prev; f.out = out; f.b = b; f.dinv = dinv; f.c1 = c1; f.c2 = c2; f.mode = mode;
  f.rp = fused_ring_planes(m);
  const size_t ring = (size_t)f.rp * m.Mx * m.My;
  static const int dbg = env_int("SFMG_FUSED_DBG", 0);
  f.mode |= dbg;
  static const int persist_mb = env_int("SFMG_L2_PERSIST_MB", 0);   // developer experiment
  if (persist_mb > 0) {
    static bool done = false;
    if (!done) {
      cudaError_t pe = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_mb << 20);
      fprintf(stderr, "persisting L2 limit %d MB: %s\n", persist_mb, cudaGetErrorString(pe));
      done = true;
    }
  }
  unsigned int* cnt = reinterpret_cast<unsigned int*>(scratch + ring);
  f.layer_done = cnt;
  f.upd_done = cnt + m.nez;
  f.err = reinterpret_cast<int*>(cnt + 2 * m.nez);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned int) * (2 * (size_t)m.nez + 1), s);
  if (e) return e;
  cudaError_t err = cudaSuccess;
  SFMG_DISPATCH_P(m.p, fused_p, m, G, cur, scratch, f, s, &err);
  return err;
}
cudaError_t fused_zero_ring(const MeshDev& m, double* scratch, cudaStream_t s) {
  return cudaMemsetAsync(scratch, 0, sizeof(double) * fused_scratch_doubles(m), s);
}

template <int P>
static void diag_p(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
  k_diag<P><<<grid_for(m.E * N3, 256), 256, 0, s>>>(m, bc, G, d);
}
cudaError_t launch_diag(const MeshDev& m, int bc, const double* G, double* d, cudaStream_t s) {
  cudaError_t e = launch_init(m, bc, nullptr, 1.0, d, s);
  if (e) return e;
  if (m.dim == 2) return launch_diag_2d(m, bc, G, d, s);
  if (m.quad) return launch_diag_gauss(m, bc, G, d, s);
  SFMG_DISPATCH_P(m.p, diag_p, m, bc, G, d, s);
  return cudaGetLastError();
}

template <int P>
static void load_p(const MeshDev& m, double* f, cudaStream_t s) {
  constexpr int N3 = (P + 1) * (P + 1) * (P + 1);
  k_load<P><<<grid_for(m.E * N3, 256), 256, 0, s>>>(m, f);
}
cudaError_t launch_load(const MeshDev& m, int rhs_id, double* f, cudaStream_t s) {
  if (rhs_id != 1) return cudaErrorInvalidValue;
  cudaError_t e = launch_init(m, 1, nullptr, 0.0, f, s);
  if (e) return e;
  if (m.dim == 2) return launch_load_2d(m, f, s);
  if (m.quad) return launch_load_gauss(m, f, s);
  SFMG_DISPATCH_P(m.p, load_p, m, f, s);
  return cudaGetLastError();
}

cudaError_t launch_init(const MeshDev& m, int bc, const double* u, double bval, double* v, cudaStream_t s) {
  int grid = grid_for((long long)m.My * m.Mz * 32, 256);
  // early trigger only for small vectors: for large ones the init outlasts the apply's first element and
  // the early-started apply blocks slow it down (config 2 46.3 -> 44.0 us; config 4 2.51 -> 3.21 ms)
  const int early = early_pdl(m) ? 1 : 0;
  if (early && grid > 8 * num_sms()) grid = 8 * num_sms();
  k_init<<<grid, 256, 0, s>>>(m, bc, u, bval, v, early);
  return cudaGetLastError();
}

cudaError_t launch_zero(double* v, long long n, cudaStream_t s) {
  if ((uintptr_t)v & 15) return cudaMemsetAsync(v, 0, sizeof(double) * n, s);
  k_zero<<<num_sms(), kZeroThreads, 0, s>>>(v, n);
  return cudaGetLastError();
}

cudaError_t launch_cheb_update(const MeshDev& m, const double* cur, const double* prev, double* out,
                               const double* b, double* y, const double* dinv, double c1, double c2,
                               cudaStream_t s) {
  int grid = grid_for(m.N, 256);
  static IntPerDevice occ;
  int per = 0;
  cudaError_t e = occ.get(per, [](int& v) { return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_cheb_update, 256, 0); });
  if (e) return e;
  const int early = early_pdl(m) ? 1 : 0;
  if (early && grid > per * num_sms()) grid = per * num_sms();
  return launch_pdl(k_cheb_update, (unsigned)grid, 256u, 0, s, m, cur, prev, out, b, y, dinv, c1, c2, early);
}

template <int P>
static void export_geometry_p(const MeshDev& m, const double* G, double* out, cudaStream_t s) {
  k_export_geometry<P><<<grid_for(m.E * 6 * (P + 1) * (P + 1) * (P + 1), 256), 256, 0, s>>>(m, G, out);
}
cudaError_t launch_export_geometry(const MeshDev& m, const double* G, double* out, cudaStream_t s) {
  SFMG_DISPATCH_P(m.p, export_geometry_p, m, G, out, s);
  return cudaGetLastError();
}

long long geometry_elems(int p, long long E) { return p <= 2 ? ((E + 31) / 32) * 32 : E; }

cudaError_t launch_export_maps(const MeshDev& m, int32_t* l2g, uint8_t* mask, uint8_t* col, cudaStream_t s) {
  long long work = m.E * (long long)(m.p + 1) * (m.p + 1) * (m.p + 1);
  k_export_maps<<<grid_for(work, 256), 256, 0, s>>>(m, l2g, mask, col);
  return cudaGetLastError();
}

constexpr int kCoarseThreads = 512;
// Coarse p = 1 CG with the operator as a 27-point stencil in registers (N <= 768 lattice nodes, one
// thread per node).  Each thread first assembles its row of A_D = M A M + (I - M) from the <= 8
// elements around its node: K_e[l][m] = sum_q (grad phi_l)(q)^T G_q (grad phi_m)(q) with the collocated
// p = 1 gradients (D from __constant__, G in the element-interleaved p <= 2 layout), columns of
// boundary nodes dropped (R4).  The CG iteration is then one 27-term register x shared-memory product
// per row and two block reductions -- the same unpreconditioned CG, x0 = 0, ||r|| <= rtol ||b|| (R13),
// as k_coarse_cg_smem, which re-ran the element apply (48 factor loads per element) every iteration.
constexpr int kStencilThreads = 768;
// block-wide sum with a single barrier: the caller alternates partial buffers so that no thread can
// still be reading a buffer when it is written again (k_coarse_cg_stencil: pq -> red0, ||r||^2 -> red1)
__device__ __forceinline__ double block_sum_1bar(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) red[w] = v;
  __syncthreads();
  double s = ln < (int)((blockDim.x + 31) >> 5) ? red[ln] : 0.0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
// block-wide sum for the single-CTA CG: warp shuffles, one partial per warp in smem, then every warp
// reduces the <= 32 partials with shuffles (no serial chain over the partials)
__device__ __forceinline__ double block_sum_fast(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  __syncthreads();
  if (ln == 0) red[w] = v;
  __syncthreads();
  double s = ln < (int)((blockDim.x + 31) >> 5) ? red[ln] : 0.0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
__global__ void __launch_bounds__(kStencilThreads) k_coarse_cg_stencil(MeshDev m, const double* __restrict__ G,
                                                                        const double* __restrict__ b,
                                                                        double* __restrict__ xout, double* scal,
                                                                        double rtol, int maxit) {
  using GL = GLayout<1>;
  __shared__ double sp[kStencilThreads];
  __shared__ double red[32], red1[32];
  const int g = threadIdx.x;
  const bool live = g < m.N;
  const int Mx = m.Mx, My = m.My, Mz = m.Mz;
  int I = 0, J = 0, K = 0;
  if (live) {
    I = g % Mx;
    J = (g / Mx) % My;
    K = g / (Mx * My);
  }
  auto interior = [&](int i, int j, int k) { return i > 0 && i < Mx - 1 && j > 0 && j < My - 1 && k > 0 && k < Mz - 1; };
  const bool inner = live && interior(I, J, K);
  double S[27];
#pragma unroll
  for (int d = 0; d < 27; ++d) S[d] = 0.0;
  if (inner) {
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int ex = I - 1 + dx, ey = J - 1 + dy, ez = K - 1 + dz;   // element; node is its local (a, b, c)
          constexpr int zero = 0;
          const int a = 1 - dx + zero, bb = 1 - dy + zero, c = 1 - dz + zero;
          const long long e = ex + (long long)m.nex * (ey + (long long)m.ney * ez);
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int ij = i + 2 * j;
                const double G00 = __ldg(G + GL::off(e, 0, ij, k)), G01 = __ldg(G + GL::off(e, 1, ij, k));
                const double G02 = __ldg(G + GL::off(e, 2, ij, k)), G11 = __ldg(G + GL::off(e, 3, ij, k));
                const double G12 = __ldg(G + GL::off(e, 4, ij, k)), G22 = __ldg(G + GL::off(e, 5, ij, k));
                // grad phi_l at q = (i, j, k) for l = (a, bb, c)
                const double l0 = (j == bb && k == c) ? dmat<1>(0, i * 2 + a) : 0.0;
                const double l1 = (i == a && k == c) ? dmat<1>(0, j * 2 + bb) : 0.0;
                const double l2 = (i == a && j == bb) ? dmat<1>(0, k * 2 + c) : 0.0;
                const double w0 = G00 * l0 + G01 * l1 + G02 * l2;
                const double w1 = G01 * l0 + G11 * l1 + G12 * l2;
                const double w2 = G02 * l0 + G12 * l1 + G22 * l2;
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
                  for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
                    for (int a2 = 0; a2 < 2; ++a2) {
                      const double m0 = (j == b2 && k == c2) ? dmat<1>(0, i * 2 + a2) : 0.0;
                      const double m1 = (i == a2 && k == c2) ? dmat<1>(0, j * 2 + b2) : 0.0;
                      const double m2 = (i == a2 && j == b2) ? dmat<1>(0, k * 2 + c2) : 0.0;
                      const int d = (a2 - a + 1) + 3 * (b2 - bb + 1) + 9 * (c2 - c + 1);
                      const bool col = interior(ex + a2, ey + b2, ez + c2);
                      S[d] += col ? (w0 * m0 + w1 * m1 + w2 * m2) : 0.0;
                    }
              }
        }
  }
  double x = 0.0, r = live ? b[g] : 0.0, p = r;
  sp[g] = p;
  double rr = block_sum_fast(r * r, red);
  const double bn = sqrt(rr);
  int it = 0, status = 0;
  if (bn > 0.0) {
    for (; it < maxit; ++it) {
      if (sqrt(rr) <= rtol * bn) break;
      __syncthreads();
      double q = p;   // boundary rows: identity
      if (inner) {
        double q3[3] = {0.0, 0.0, 0.0};   // one partial sum per z offset (three short FMA chains)
#pragma unroll
        for (int d = 0; d < 27; ++d) {
          const int ox = d % 3 - 1, oy = (d / 3) % 3 - 1, oz = d / 9 - 1;
          q3[d / 9] = fma(S[d], sp[g + ox + Mx * (oy + My * oz)], q3[d / 9]);
        }
        q = (q3[0] + q3[1]) + q3[2];
      } else if (!live) {
        q = 0.0;
      }
      const double pq = block_sum_1bar(p * q, red);    // 1 barrier (buffers alternate; the rn
                                                       // barrier and the loop-top one separate reuses)
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rr / pq;
      x += alpha * p;
      r -= alpha * q;
      const double rn = block_sum_1bar(r * r, red1);
      p = r + (rn / rr) * p;
      sp[g] = p;   // every read of the old p is before the reductions' barriers
      rr = rn;
    }
  }
  if (live) xout[g] = x;
  if (threadIdx.x == 0) { scal[8] = (double)it; scal[9] = sqrt(rr); scal[10] = (double)status; }
}

constexpr long long kCoarseSmemN = 6400;   // x, r, p, q of up to this many dofs live in shared memory

cudaError_t launch_coarse_cg(const MeshDev& m, const double* G, const double* b, double* x, double* r,
                             double* p, double* q, double* scal, double rtol, int maxit, cudaStream_t s) {
  if (m.quad) return launch_coarse_cg_gauss(m, G, b, x, r, p, q, scal, rtol, maxit, s);
  if (m.p != 1 && m.p != 2) return cudaErrorInvalidValue;
  if (m.p == 1 && m.dim == 3 && m.N <= kStencilThreads) {
    k_coarse_cg_stencil<<<1, kStencilThreads, 0, s>>>(m, G, b, x, scal, rtol, maxit);
    return cudaGetLastError();
  }
  if (m.N <= kCoarseSmemN) {
    const size_t smem = sizeof(double) * 4 * (size_t)m.N;
    static OncePerDevice attr1, attr2;
    const int lim = (int)(sizeof(double) * 4 * kCoarseSmemN);
    if (m.p == 1) {
      cudaError_t e = attr1.run([&] {
        return cudaFuncSetAttribute(k_coarse_cg_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
      });
      if (e) return e;
      k_coarse_cg_smem<1><<<1, kCoarseThreads, smem, s>>>(m, G, b, x, scal, rtol, maxit);
    } else {
      cudaError_t e = attr2.run([&] {
        return cudaFuncSetAttribute(k_coarse_cg_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
      });
      if (e) return e;
      k_coarse_cg_smem<2><<<1, kCoarseThreads, smem, s>>>(m, G, b, x, scal, rtol, maxit);
    }
    return cudaGetLastError();
  }
  if (m.p == 1)
    k_coarse_cg<1><<<1, 256, 0, s>>>(m, G, b, x, r, p, q, scal, rtol, maxit);
  else
    k_coarse_cg<2><<<1, 256, 0, s>>>(m, G, b, x, r, p, q, scal, rtol, maxit);
  return cudaGetLastError();
}

}  // namespace sfmg


#ifdef SFMG_KS_DBG
extern "C" int sfmg_ksdbg_read(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, sfmg::g_ksdbg, sizeof(unsigned long long) * n);
}
#endif

#ifdef SFMG_TIMELINE
extern "C" int sfmg_tl_read(unsigned long long* init, int ni, unsigned long long* v4, int nv) {
  cudaError_t e = cudaMemcpyFromSymbol(init, sfmg::g_tl_init, sizeof(unsigned long long) * ni);
  if (e) return (int)e;
  return (int)cudaMemcpyFromSymbol(v4, sfmg::g_tl_v4, sizeof(unsigned long long) * nv);
}
#endif
