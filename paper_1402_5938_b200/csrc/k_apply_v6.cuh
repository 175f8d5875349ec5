// K2 apply, v6 (even p >= 12; opt-in, SFMG_V6=1): two elements in flight per SM.
//
// k_apply_v4 at p = 16 holds one block (289 threads, 168 registers) per SM: the thread that owns a
// z-column keeps the u column, its z-derivative and the transposed z-product in registers across the
// x / y passes, which caps the SM at 10 warps.  v6 keeps that per-column data in a third shared-memory
// array that only the owner thread ever touches (so its last two k-planes can live in two registers:
// 3 n^3 doubles would miss the two-block shared-memory budget by 4 KB, 3 n^3 - 2 n^2 fit), never holds
// more than one line in registers, and is compiled for two blocks per SM (<= 96 registers):
//   gather: u column -> su, g2 = D u (z) -> sz;  P1: g0 = D u (x) -> s0;  P2: g1 = D u (y) -> su in place;
//   P3 (column): w = G g with the factors read from L2 (streaming, the element was L2-prefetched),
//       w0 -> s0, w1 -> su, w2 -> sz, then sz = D^T w2 (z) in place;
//   P4: s0 = D^T w0 (x) in place;  P5: su = D^T w1 (y) + s0;  P6: v += su + sz (fp64 RED).
// Same launch contract as k_apply_v4 (wait_mode, write_bnd, early programmatic triggers).
// Measured (config 3, p = 16): 71 us per apply against k_apply_v4's 62.5 us -- two elements in flight, but
// each takes 2.2x as long (96-register cap, three times the shared-memory wavefronts); kept opt-in as the
// record of the experiment (profiles/r02_experiments.md).
// (included inside namespace sfmg by k_operator.cu, after the helpers it uses)

// out = M L for one line with the even-odd tables in shared memory (tab: eoSize(P) doubles of D (set 0) or
// D^T (set 3)): as __constant__ operands ptxas hoists the p = 16 tables into registers and spills them
// at the 96-register cap; shared-memory broadcast loads stay in the loop.
template <int P>
__device__ __forceinline__ void eo_line_s(const double* __restrict__ tab, const double (&L)[P + 1], double (&out)[P + 1]) {
  constexpr int N = P + 1, c = P / 2;
  double ev[c], od[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    ev[m] = L[m] + L[N - 1 - m];
    od[m] = L[m] - L[N - 1 - m];
  }
  if constexpr (c % 2 == 0) {   // 16-byte table loads (tab is 16-byte aligned)
    const double2* t2 = reinterpret_cast<const double2*>(tab);
#pragma unroll
    for (int i = 0; i < c; ++i) {
      double S = 0.0, T = tab[2 * c * c + i] * L[c];
#pragma unroll
      for (int m = 0; m < c; m += 2) {
        const double2 a = t2[(i * c + m) / 2], b = t2[(c * c + i * c + m) / 2];
        S = fma(a.x, od[m], S);
        S = fma(a.y, od[m + 1], S);
        T = fma(b.x, ev[m], T);
        T = fma(b.y, ev[m + 1], T);
      }
      out[i] = S + T;
      out[N - 1 - i] = S - T;
    }
    double M = 0.0;
#pragma unroll
    for (int m = 0; m < c; m += 2) {
      const double2 a = t2[(2 * c * c + c + m) / 2];
      M = fma(a.x, od[m], M);
      M = fma(a.y, od[m + 1], M);
    }
    out[c] = M;
  } else {
#pragma unroll
    for (int i = 0; i < c; ++i) {
      double S = 0.0, T = tab[2 * c * c + i] * L[c];
#pragma unroll
      for (int m = 0; m < c; ++m) {
        S = fma(tab[i * c + m], od[m], S);
        T = fma(tab[c * c + i * c + m], ev[m], T);
      }
      out[i] = S + T;
      out[N - 1 - i] = S - T;
    }
    double M = 0.0;
#pragma unroll
    for (int m = 0; m < c; ++m) M = fma(tab[2 * c * c + c + m], od[m], M);
    out[c] = M;
  }
}

template <int P>
struct V6Cfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr int ZP = N - 2;                       // k-planes of the owner-private array in smem
  static constexpr int THREADS = N2;
  static constexpr int TAB = 2 * eoSize(P);             // even-odd D and D^T tables
  static constexpr size_t SMEM = sizeof(double) * (2 * N3 + ZP * N2 + TAB) + 16;
  static constexpr int MINB = 2;
};

template <int P, bool DIR>
__global__ void __launch_bounds__(V6Cfg<P>::THREADS, V6Cfg<P>::MINB)
    k_apply_v6(MeshDev m, const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ v,
               int wait_mode, int write_bnd) {
  using C = V6Cfg<P>;
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3, ZP = C::ZP;
  static_assert(P % 2 == 0 && P >= 4, "even-odd line products");
  extern __shared__ __align__(128) double smem6[];
  double* tD = smem6;                   // even-odd D (16-byte aligned: eoSize is even)
  double* tT = tD + eoSize(P);          // even-odd D^T
  double* s0 = tT + eoSize(P);
  double* su = s0 + N3;
  double* sz = su + N3;   // [ZP][n^2], owner-private columns; planes ZP, ZP + 1 in zr0, zr1
  for (int q = threadIdx.x; q < eoSize(P); q += blockDim.x) {
    tD[q] = c_EO[eoOffset(P) + (P <= kEoSharedMaxP ? 0 : 0) * eoSize(P) + q];
    tT[q] = c_EO[eoOffset(P) + 3 * eoSize(P) + q];
  }
  __syncthreads();
  const int t = threadIdx.x, t0 = t % N, t1 = t / N;
  const long long sxy = (long long)m.Mx * m.My;
  const long long gstride = gridDim.x;
  auto prefetch_elem_l2 = [&](long long e) {
    const char* src = (const char*)(G + e * 6 * N3);
    const unsigned total = (unsigned)(6 * N3 * sizeof(double));
    for (unsigned o = 0; o < total; o += 65536u) bulk_prefetch_l2(src + o, total - o < 65536u ? total - o : 65536u);
  };
  auto prefetch_column = [&](long long e) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const double* pu = u + (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
#pragma unroll
    for (int k = 0; k < N; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + sxy * k));
  };
  long long e = blockIdx.x;
  if (t == 0 && e < m.E) prefetch_elem_l2(e);
  if (wait_mode == 2) pdl_wait();
  bool waited = (wait_mode != 1);
  for (; e < m.E; e += gstride) {
    if (m.pdl_early && e + gstride >= m.E) pdl_trigger();
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const long long gcol = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + t0, J = ey * P + t1;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
    double zr0, zr1;
    {  // gather (M u, R4) and the z-derivative of the thread's own column
      double L[N], o[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        bool ok = true;
        if (DIR) { const int K = ez * P + k; ok = !(bxy || K == m.Kb0 || K == m.Kb1); }
        L[k] = ok ? __ldg(u + gcol + sxy * k) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < N; ++k) su[t + N2 * k] = L[k];
      eo_line_s<P>(tD, L, o);
#pragma unroll
      for (int k = 0; k < ZP; ++k) sz[t + N2 * k] = o[k];
      zr0 = o[ZP];
      zr1 = o[ZP + 1];
    }
    if (e + gstride < m.E) prefetch_column(e + gstride);
    __syncthreads();
    {  // P1: g0 on x-line (j = t0, k = t1) -> s0
      double L[N], o[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = su[mm + N * t0 + N2 * t1];
      eo_line_s<P>(tD, L, o);
#pragma unroll
      for (int i = 0; i < N; ++i) s0[i + N * t0 + N2 * t1] = o[i];
    }
    __syncthreads();
    {  // P2: g1 on y-line (i = t0, k = t1), in place in su
      double L[N], o[N];
      const int yb = t0 + N2 * t1;
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = su[yb + N * mm];
      eo_line_s<P>(tD, L, o);
#pragma unroll
      for (int j = 0; j < N; ++j) su[yb + N * j] = o[j];
    }
    __syncthreads();
    {  // P3: column (i = t0, j = t1): w = G g (factors from L2), then D^T w2 along z in place
      const double* Gg = G + e * 6 * N3 + t;
      double w2[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double G00 = __ldcs(Gg + gofs<N>(0, 0, k)), G01 = __ldcs(Gg + gofs<N>(1, 0, k));
        const double G02 = __ldcs(Gg + gofs<N>(2, 0, k)), G11 = __ldcs(Gg + gofs<N>(3, 0, k));
        const double G12 = __ldcs(Gg + gofs<N>(4, 0, k)), G22 = __ldcs(Gg + gofs<N>(5, 0, k));
        const int idx = t + N2 * k;
        const double g0 = s0[idx], g1 = su[idx];
        const double g2 = (k < ZP) ? sz[idx] : (k == ZP ? zr0 : zr1);
        s0[idx] = G00 * g0 + G01 * g1 + G02 * g2;
        su[idx] = G01 * g0 + G11 * g1 + G12 * g2;
        w2[k] = G02 * g0 + G12 * g1 + G22 * g2;
      }
      double o[N];
      eo_line_s<P>(tT, w2, o);
#pragma unroll
      for (int k = 0; k < ZP; ++k) sz[t + N2 * k] = o[k];
      zr0 = o[ZP];
      zr1 = o[ZP + 1];
    }
    __syncthreads();
    if (t == 0 && e + gstride < m.E) prefetch_elem_l2(e + gstride);
    {  // P4: v0 = D^T w0 on x-line, in place in s0
      double L[N], o[N];
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = s0[mm + N * t0 + N2 * t1];
      eo_line_s<P>(tT, L, o);
#pragma unroll
      for (int a = 0; a < N; ++a) s0[a + N * t0 + N2 * t1] = o[a];
    }
    __syncthreads();
    {  // P5: su = D^T w1 + v0 on y-line (i = t0, k = t1)
      double L[N], o[N];
      const int yb = t0 + N2 * t1;
#pragma unroll
      for (int mm = 0; mm < N; ++mm) L[mm] = su[yb + N * mm];
      eo_line_s<P>(tT, L, o);
#pragma unroll
      for (int b = 0; b < N; ++b) su[yb + N * b] = o[b] + s0[yb + N * b];
    }
    __syncthreads();
    if (!waited) {
      pdl_wait();
      waited = true;
    }
    {  // P6: column (i = t0, j = t1): v = su + sz, scatter
      const bool own_xy = (t0 > 0 || ex == 0) && (t1 > 0 || ey == 0);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        bool bnd = false;
        if (DIR) { const int K = ez * P + c; bnd = bxy || K == m.Kb0 || K == m.Kb1; }
        const double z = (c < ZP) ? sz[t + N2 * c] : (c == ZP ? zr0 : zr1);
        if (!bnd) atomicAdd(v + gcol + sxy * c, su[t + N2 * c] + z);
        else if (write_bnd && own_xy && (c > 0 || ez == 0)) v[gcol + sxy * c] = u[gcol + sxy * c];   // (I - M) u
      }
    }
    // (the next gather writes only the su / sz column this thread just read; s0 is rewritten two
    //  barriers later)
  }
}

