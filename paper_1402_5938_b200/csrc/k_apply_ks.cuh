// K2 apply for high orders, "k-split" (included by k_operator.cu; uses its constant tables and
// helpers).  The element operator is the same as k_apply_v4's:
//   g = (D x I x I, I x D x I, I x I x D) u_e,  w = G_q g,  v_e = sum of the transposed contractions.
//
// Why a different kernel at p >= 12: one element's factors (48 n^3 bytes, 236 KB at p = 16) do not
// fit one SM's shared memory, so k_apply_v4 reads them from L2 through a register ring in its z-line
// pass, holds one element (10 warps) per SM and walks 512 elements over 148 SMs in 4 rounds (3.46 ->
// 86 % wave efficiency): 0.41 of the HBM roofline at p = 16.
//
// Here each element is split by k-slices across the two CTAs of a thread-block cluster (one per SM):
// CTA h owns slices [k0, k0 + KH) (k0 = 0, KH = ceil(n/2) for h = 0; the rest for h = 1).
//  * Its factors G[e][k0 .. k0+KH) are ONE contiguous block of the slice-major layout: TMA bulk copies
//    (in chunks of kChunk slices, one mbarrier each, so the z-pass starts on the first chunk) land
//    them in shared memory; the next element's copy is issued as soon as the z-pass consumed the
//    buffer, and an L2 prefetch of the element after that keeps HBM busy one element further ahead.
//  * The x- and y-line passes (P1/P2 with D, P4/P5 with D^T) touch only the CTA's own slices: one
//    line per lane pair (each lane half of the output pairs), x and y in the same barrier phase
//    (different arrays); the z-pass has one thread per (i, j) column (10 warps at p = 16).
//  * The z-direction couples the halves.  g2(k) = sum_m D[k][m] u(m) needs the whole u column, which
//    each CTA gathers itself (8 B per node, against 48 B per node of factors).  The transposed
//    contraction Z(c) = sum_k D[k][c] w2(k) gets a partial sum from each half:
//    Z_h(c) = sum_{k in own} D[k][c] w2(k) for all c.  The partial for the partner's slices goes
//    straight into the partner's receive buffer by asynchronous DSMEM stores (st.async) that complete
//    transaction bytes on the partner's receive mbarrier, which the partner waits on before its scatter
//    (no fence: a release-ordered cluster barrier here emitted a GPU-scope MEMBAR behind the previous
//    element's outstanding REDs).  Reuse of the receive buffer: a relaxed cluster-barrier arrive after
//    each CTA's scatter, waited for before the partner's next remote stores.
//  * P6 scatters X + Y + Z_own + Z_partner of its own slices: fp64 RED (or the IPS plain store).
// 512 elements become 1024 half-elements over 148 SMs: 7 rounds of 74 clusters (98.8 % waves).
// even orders from this one up take the k-split cluster kernel; their shared-memory tables (even-odd D,
// two-lane half tables of D and D^T, D) are laid out on the host (upload_ks_tables) in g_kstab
constexpr int kKsMinP = 12;
constexpr int kKsTabMax = 1024;
__device__ double g_kstab[3][kKsTabMax];   // p = 12, 14, 16

template <int P>
struct KsCfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr int KH0 = (N + 1) / 2, KH1 = N - KH0, KMAX = KH0;
  // one thread per z-column (i, j) in the z-pass; two lanes per own x-line / y-line in P1/P2, P4/P5
  static constexpr int TMAX = (N2 > 2 * N * KMAX) ? N2 : 2 * N * KMAX;
  static constexpr int THREADS = ((TMAX + 31) / 32) * 32;
  static constexpr int kChunk = 3;                               // slices per TMA chunk / mbarrier
  static constexpr int NCH = (KMAX + kChunk - 1) / kChunk;
  static constexpr int SLICE = 6 * N2;                           // doubles per factor slice
  // smem (doubles): G [KMAX][6][n^2], s0, su, sz, rx [KMAX][n^2]; mbarriers (NCH factor chunks, receive)
  static constexpr size_t OFF_S0 = (size_t)KMAX * SLICE;
  static constexpr size_t OFF_SU = OFF_S0 + (size_t)KMAX * N2;
  static constexpr size_t OFF_SZ = OFF_SU + (size_t)KMAX * N2;
  static constexpr size_t OFF_RX = OFF_SZ + (size_t)KMAX * N2;
  // 1-D tables in smem: even-odd D (z-line g2), two-lane half tables of D and D^T (x/y passes), D [n][n]
  static constexpr int EOS = 2 * (P / 2) * (P / 2) + 2 * (P / 2);
  static constexpr int HMS = 2 * (2 * ((P / 2 + 1) / 2) * (P / 2) + (P / 2 + 1) / 2 + P / 2 + 2);   // >= MSTR
  static constexpr size_t OFF_TAB = OFF_RX + (size_t)KMAX * N2;
  static constexpr int TABSZ = EOS + 2 * HMS + N * N;
  static constexpr size_t OFF_BAR = OFF_TAB + ((TABSZ + 1) & ~1);
  static constexpr size_t SMEM = OFF_BAR * 8 + 8 * (NCH + 1);
};

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa_shared(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// asynchronous DSMEM store whose completion is counted in transaction bytes on the remote mbarrier
__device__ __forceinline__ void st_async_f64(unsigned addr, double v, unsigned remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// One x- or y-line pass with two threads per line: lanes 2L and 2L + 1 share line L, both read it and
// form its even/odd parts, and lane hh computes the output pairs (i, n-1-i) for i in [hh c/2, (hh+1) c/2)
// of M L (M = D or D^T; hh = 1 also the centre).  The coefficients come from the half-table of lane hh
// in shared memory (rows interleaved so the two halves' rows sit in different banks).
// Half-table layout per matrix, per hh (HSTR doubles): A rows [4][c], B rows [4][c], M[i][c] for the 4
// rows, centre row M[c][m] [c].
template <int P>
struct HalfTab {
  static constexpr int c = P / 2, R = (c + 1) / 2;            // output pairs per lane (hh = 1: c - R real)
  static constexpr int SZ = 2 * R * c + R + c;
  static constexpr int HSTR = (SZ % 2 == 0) ? SZ + 2 : SZ + 1; // even (16-byte rows), != 0 mod 32 banks
  static constexpr int MSTR = 2 * HSTR;                        // per matrix
};

template <int P>
__device__ __forceinline__ void line_pass_half(const double* __restrict__ ht, double* line, int stride, int hh,
                                               bool act) {
  using H = HalfTab<P>;
  constexpr int N = P + 1, c = H::c, R = H::R;
  double L[N];
#pragma unroll
  for (int m = 0; m < N; ++m) L[m] = line[m * stride];
  __syncwarp();   // both lanes of the pair hold the whole line before either overwrites its part
  double ev[c], od[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    ev[m] = L[m] + L[N - 1 - m];
    od[m] = L[m] - L[N - 1 - m];
  }
  const double* tb = ht + hh * H::HSTR;
  const int i0 = hh * R;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double S = 0.0, T = tb[2 * R * c + r] * L[c];
#pragma unroll
    for (int m = 0; m < c; ++m) {
      S = fma(tb[r * c + m], od[m], S);
      T = fma(tb[R * c + r * c + m], ev[m], T);
    }
    if (act && i0 + r < c) {
      line[(i0 + r) * stride] = S + T;
      line[(N - 1 - i0 - r) * stride] = S - T;
    }
  }
  double M = 0.0;
#pragma unroll
  for (int m = 0; m < c; ++m) M = fma(tb[2 * R * c + R + m], od[m], M);
  if (act && hh) line[c * stride] = M;
}

// The x-line and the y-line of one lane pair at once (independent FMA chains interleave: the passes are
// latency-bound at one CTA of 10 warps per SM)
template <int P>
__device__ __forceinline__ void line_pass_half2(const double* __restrict__ ht, double* la, int sa, double* lb, int sb,
                                                int hh, bool act) {
  using H = HalfTab<P>;
  constexpr int N = P + 1, c = H::c, R = H::R;
  double A[N], B[N];
#pragma unroll
  for (int m = 0; m < N; ++m) {
    A[m] = la[m * sa];
    B[m] = lb[m * sb];
  }
  __syncwarp();   // both lanes of each pair hold their lines before either overwrites its part
  double eva[c], oda[c], evb[c], odb[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    eva[m] = A[m] + A[N - 1 - m];
    oda[m] = A[m] - A[N - 1 - m];
    evb[m] = B[m] + B[N - 1 - m];
    odb[m] = B[m] - B[N - 1 - m];
  }
  const double* tb = ht + hh * H::HSTR;
  const int i0 = hh * R;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double dc = tb[2 * R * c + r];
    double Sa = 0.0, Ta = dc * A[c], Sb = 0.0, Tb = dc * B[c];
#pragma unroll
    for (int m = 0; m < c; ++m) {
      const double a = tb[r * c + m], b = tb[R * c + r * c + m];
      Sa = fma(a, oda[m], Sa);
      Sb = fma(a, odb[m], Sb);
      Ta = fma(b, eva[m], Ta);
      Tb = fma(b, evb[m], Tb);
    }
    if (act && i0 + r < c) {
      la[(i0 + r) * sa] = Sa + Ta;
      la[(N - 1 - i0 - r) * sa] = Sa - Ta;
      lb[(i0 + r) * sb] = Sb + Tb;
      lb[(N - 1 - i0 - r) * sb] = Sb - Tb;
    }
  }
  double Ma = 0.0, Mb = 0.0;
#pragma unroll
  for (int m = 0; m < c; ++m) {
    const double w = tb[2 * R * c + R + m];
    Ma = fma(w, oda[m], Ma);
    Mb = fma(w, odb[m], Mb);
  }
  if (act && hh) {
    la[c * sa] = Ma;
    lb[c * sb] = Mb;
  }
}

// z-line product (all outputs, one thread) with the full even-odd table of D in shared memory
template <int P>
__device__ __forceinline__ void eo_line_tab(const double* __restrict__ tab, const double (&L)[P + 1],
                                            double (&out)[P + 1]) {
  constexpr int N = P + 1, c = P / 2;
  double ev[c], od[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    ev[m] = L[m] + L[N - 1 - m];
    od[m] = L[m] - L[N - 1 - m];
  }
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

#ifdef SFMG_KS_DBG
__device__ unsigned long long g_ksdbg[148 * 16 * 10];   // [block][element <= 16][mark]
#define KSDBG(el, s)                                                                     \
  if (threadIdx.x == 0 && blockIdx.x < 148 && (el) < 16) {                               \
    unsigned long long t_;                                                               \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
    g_ksdbg[(blockIdx.x * 16 + (el)) * 10 + (s)] = t_;                                   \
  }
#else
#define KSDBG(el, s)
#endif

// The body for cluster rank H (compile-time: every slice index, the own/partner split of the z-outputs
// and the DSMEM offsets are constants).
template <int P, bool DIR, bool IPS, int H>
__device__ __forceinline__ void ks_body(const MeshDev& m, const double* __restrict__ G, const double* __restrict__ u,
                                        double* __restrict__ v, int wait_mode, int write_bnd, double* smem) {
  using C = KsCfg<P>;
  using HT = HalfTab<P>;
  static_assert(HT::MSTR <= C::HMS, "half-table size");
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3;
  constexpr int KH = H ? C::KH1 : C::KH0, K0 = H ? C::KH0 : 0, K0P = H ? 0 : C::KH0;
  constexpr int NCH = (KH + C::kChunk - 1) / C::kChunk;
  constexpr int NL = N * KH;                  // own x-lines (= own y-lines)
  double* sG = smem;
  double* s0 = smem + C::OFF_S0;
  double* su = smem + C::OFF_SU;
  double* sz = smem + C::OFF_SZ;
  double* rx = smem + C::OFF_RX;
  double* eoD = smem + C::OFF_TAB;            // even-odd D (full)
  double* htD = eoD + C::EOS;                 // half tables of D (P1/P2), then of D^T (P4/P5)
  double* htDT = htD + C::HMS;
  double* sD = htD + 2 * C::HMS;              // D [n][n]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* rxbar = bar + C::NCH;
  const int t = threadIdx.x;
  const long long cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const long long sxy = (long long)m.Mx * m.My;
  const unsigned rx_remote = mapa_shared(smem_u32(rx), H ^ 1);
  const unsigned rxbar_remote = mapa_shared(smem_u32(rxbar), H ^ 1);
  constexpr unsigned RX_BYTES = (unsigned)(KH * N2 * 8);   // partner's partial Z for my slices

  KSDBG(15, 0);
  {  // tables (host-built, g_kstab): 16-byte loads, L2-resident after the first block
    const double2* src = reinterpret_cast<const double2*>(g_kstab[(P - 12) / 2]);
    double2* dst = reinterpret_cast<double2*>(eoD);
    for (int q = t; q < (C::TABSZ + 1) / 2; q += blockDim.x) dst[q] = src[q];
  }
  auto g_half = [&](long long e) { return G + e * 6 * N3 + (long long)K0 * C::SLICE; };
  auto issue_g = [&](long long e) {   // TMA of element e's own factor slices, one mbarrier per chunk
    const double* src = g_half(e);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      constexpr int S = C::kChunk;
      const int ns = (KH - c * S) < S ? (KH - c * S) : S;
      bulk_load(sG + (size_t)c * S * C::SLICE, src + (size_t)c * S * C::SLICE, (unsigned)(ns * C::SLICE * 8), bar + c);
    }
  };
  auto prefetch_g = [&](long long e) {
    const char* src = (const char*)g_half(e);
    constexpr unsigned total = (unsigned)(KH * C::SLICE * 8);
    for (unsigned o = 0; o < total; o += 65536u) bulk_prefetch_l2(src + o, total - o < 65536u ? total - o : 65536u);
  };
  // this thread's z-column (i, j) and its u column of element e (M u: zero on Dirichlet nodes)
  const bool colact = t < N2;
  const int ci = colact ? t % N : 0, cj = colact ? t / N : 0;
  // gather of element e: own slices of the u column to smem, g2 = D u on own k (registers)
  auto gather = [&](const double (&uc)[N], double (&g2own)[KH]) {
    double g2[N];
    eo_line_tab<P>(eoD, uc, g2);
    if (colact) {
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        s0[t + N2 * kk] = uc[K0 + kk];
        su[t + N2 * kk] = uc[K0 + kk];
      }
    }
#pragma unroll
    for (int kk = 0; kk < KH; ++kk) g2own[kk] = g2[K0 + kk];
  };
  auto load_ucol = [&](long long e, double (&uc)[N]) {
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + ci, J = ey * P + cj;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
    const double* up = u + (long long)(ex * P + ci) + (long long)m.Mx * (ey * P + cj) + sxy * (long long)(ez * P);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      bool ok = colact;
      if (DIR) { const int K = ez * P + k; ok = ok && !(bxy || K == m.Kb0 || K == m.Kb1); }
      uc[k] = ok ? __ldg(up + sxy * k) : 0.0;
    }
  };

  long long e = cl;
  if (t == 0) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) mbar_init(bar + c, 1);
    mbar_init(rxbar, 1);
    if (e < m.E) issue_g(e);
    if (e + ncl < m.E) prefetch_g(e + ncl);
  }
  cluster_arrive();   // both CTAs running (DSMEM targets exist), mbarriers and tables initialised
  cluster_wait();
  cluster_arrive_relaxed();   // "receive buffer free" for the first element
  KSDBG(15, 1);
  if (wait_mode == 2) pdl_wait();
  bool waited = (wait_mode != 1);
  unsigned phase = 0;
  double g2own[KH];
  if (e < m.E) {   // gather of the first element (later ones are fused into the previous scatter)
    double uc[N];
    load_ucol(e, uc);
    gather(uc, g2own);
  }
  __syncthreads();
  // x/y pass task of this thread: line L = t / 2, lane half hh = t & 1
  const int lt = t >> 1, hh = t & 1;
  const bool lact = lt < NL;
  const int la = lact ? lt % N : 0, lkk = lact ? lt / N : 0;
  for (int el = 0; e < m.E; e += ncl, ++el) {
    KSDBG(el, 0);
    if (m.pdl_early && e + ncl >= m.E) pdl_trigger();
    if (t == C::THREADS - 1) mbar_expect_tx(rxbar, RX_BYTES);   // this element's partial Z from the partner
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const long long nx = e + ncl;
    KSDBG(el, 1);
    // ---- P1 / P2: g0 on own x-lines, g1 on own y-lines (in place; two lanes per line)
    line_pass_half2<P>(htD, s0 + N * la + N2 * lkk, 1, su + la + N2 * lkk, N, hh, lact);   // x (j = la), y (i = la)
    __syncthreads();
    // ---- P3: z-columns.  w = G g on own slices (w0 -> s0, w1 -> su), Z_H(c) = sum_own D[k][c] w2(k):
    // own c -> sz, partner's c -> its rx (after it has scattered the previous element)
    KSDBG(el, 2);
    cluster_wait();
    KSDBG(el, 3);
    double uc[N];
    if (nx < m.E) load_ucol(nx, uc);   // the next element's u column, in flight until the scatter
    if (colact) {
      double w2[KH];
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        if (kk % C::kChunk == 0) mbar_wait(bar + kk / C::kChunk, phase);
        const double* Gk = sG + (size_t)kk * C::SLICE + t;
        const double G00 = Gk[0], G01 = Gk[N2], G02 = Gk[2 * N2], G11 = Gk[3 * N2], G12 = Gk[4 * N2],
                     G22 = Gk[5 * N2];
        const double g0 = s0[t + N2 * kk], g1 = su[t + N2 * kk], g2 = g2own[kk];
        s0[t + N2 * kk] = G00 * g0 + G01 * g1 + G02 * g2;
        su[t + N2 * kk] = G01 * g0 + G11 * g1 + G12 * g2;
        w2[kk] = G02 * g0 + G12 * g1 + G22 * g2;
      }
#pragma unroll
      for (int c = 0; c < N; ++c) {   // partial transposed z-contraction, every output slice c
        double z = 0.0;
#pragma unroll
        for (int kk = 0; kk < KH; ++kk) z = fma(sD[(K0 + kk) * N + c], w2[kk], z);
        if (c >= K0 && c < K0 + KH) sz[(c - K0) * N2 + t] = z;
        else st_async_f64(rx_remote + (unsigned)(((c - K0P) * N2 + t) * 8), z, rxbar_remote);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KH; kk += C::kChunk) mbar_wait(bar + kk / C::kChunk, phase);
    }
    __syncthreads();    // factors consumed: the next element's TMA, the L2 prefetch of the one after
    KSDBG(el, 4);
    phase ^= 1u;
    if (t == C::THREADS - 1 && nx < m.E) {   // the last warp has (almost) no x/y lines to run
      fence_proxy_async_smem();
      issue_g(nx);
      if (nx + ncl < m.E) prefetch_g(nx + ncl);
    }
    // ---- P4 / P5: X = D^T w0 on own x-lines, Y = D^T w1 on own y-lines (in place)
    line_pass_half2<P>(htDT, s0 + N * la + N2 * lkk, 1, su + la + N2 * lkk, N, hh, lact);
    __syncthreads();
    KSDBG(el, 5);
    mbar_wait(rxbar, phase ^ 1u);   // the partner's partial Z (phase already advanced above)
    KSDBG(el, 6);
    if (!waited) {
      pdl_wait();
      waited = true;
    }
    // ---- P6: v = X + Y + Z_own + Z_partner on own slices, scatter; then the next element's gather into
    // the same (own-column) smem locations
    if (colact) {
      bool bxy = false;
      if (DIR) {
        const int I = ex * P + ci, J = ey * P + cj;
        bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
      }
      const bool own_xy = (ci > 0 || ex == 0) && (cj > 0 || ey == 0);
      const long long gcol = (long long)(ex * P + ci) + (long long)m.Mx * (ey * P + cj) + sxy * (long long)(ez * P);
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        constexpr int zero = 0;
        const int c = K0 + kk + zero;
        bool bnd = false;
        if (DIR) { const int K = ez * P + c; bnd = bxy || K == m.Kb0 || K == m.Kb1; }
        const double val = s0[t + N2 * kk] + su[t + N2 * kk] + sz[kk * N2 + t] + rx[kk * N2 + t];
        const long long g = gcol + sxy * c;
        if (IPS && ci > 0 && ci < P && cj > 0 && cj < P && c > 0 && c < P) v[g] = val;
        else if (!bnd) atomicAdd(v + g, val);
        else if (write_bnd && own_xy && (c > 0 || ez == 0)) v[g] = u[g];
      }
    }
    if (nx < m.E) gather(uc, g2own);
    __syncthreads();           // sz / rx reads done, next element's s0 / su staged
    KSDBG(el, 7);
    cluster_arrive_relaxed();  // my rx is free for the partner's next element
  }
  cluster_wait();              // pairs the last arrive: the partner is past its last remote store
  KSDBG(15, 2);
}

template <int P, bool DIR, bool IPS>
__global__ void __launch_bounds__(KsCfg<P>::THREADS, 1)
    k_apply_ks(MeshDev m, const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ v,
               int wait_mode, int write_bnd) {
  extern __shared__ __align__(128) double smem[];
  if (cluster_ctarank() == 0) ks_body<P, DIR, IPS, 0>(m, G, u, v, wait_mode, write_bnd, smem);
  else ks_body<P, DIR, IPS, 1>(m, G, u, v, wait_mode, write_bnd, smem);
}
