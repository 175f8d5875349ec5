// K2 apply, v5 (even p >= 4): two threads per 1-D line.  Included from k_operator.cu (uses its
// __constant__ even-odd tables c_EO, the TMA / mbarrier helpers and the V4 prefetch knobs).
//
// Same element operator as k_apply_v4; what changes is the work split.
// v4 gives each thread a whole line per pass (n^2 threads per element, 148-168 registers, 3 warps per
// element at p = 8 and 10 at p = 16) and ncu shows it latency-bound (issue 28-39 %, FP64 pipe 21-25 %,
// HBM 30-52 %).  v5 splits every line between two threads: with the even-odd form of D
// (k_operator.cu, eo_line) the n outputs of a line are c = p/2 output pairs (i, n-1-i) plus the
// centre, and half h of a line owns the pairs [lo_h, lo_h + np_h) (h = 1 also the centre).  Both
// halves read the whole line (the even/odd sums need it) but each does half of the FMAs and keeps
// half of the outputs, so an element has twice the warps and each thread holds half the state.
// h is warp-uniform (threads [h*HALF, h*HALF + n^2) of an element), so every warp reads D through
// uniform constant operands with compile-time indices.
//
// Per element, with three n^3 smem arrays sU, s0, s1 (plus the TMA-staged factors when GS):
//   gather  u column t, own k slots                      -> sU                      | barrier
//   A       x-line D u -> s0, y-line D u -> s1, z-line D u -> g2 (own k, registers) | barrier
//   B       pointwise at (t, own k): w = G g; w0 -> s0, w1 -> s1, w2 -> sU          | barrier
//   C1      X = D^T w0 (x-line), Y = D^T w1 (y-line), own outputs in registers      | barrier
//   C2      X -> s0, Y -> s1 in place (every read of C1 is done)                    | barrier
//   C3      z-line: Z = D^T w2 from sU; v = s0 + s1 + Z at own k -> fp64 RED into v
// Five barriers per element (v4: six).

template <int P>
struct V5Half {
  static constexpr int N = P + 1, C = P / 2;
  static constexpr int C0 = (C + 1) / 2;   // pair indices [0, C0) -> half 0, [C0, C) -> half 1 (+ centre)
  template <int H> static constexpr int lo() { return H == 0 ? 0 : C0; }
  template <int H> static constexpr int np() { return H == 0 ? C0 : C - C0; }
  template <int H> static constexpr int ns() { return 2 * np<H>() + (H == 1 ? 1 : 0); }
  static constexpr int NSMAX = (2 * C0 > 2 * (C - C0) + 1) ? 2 * C0 : 2 * (C - C0) + 1;
  // own slot s -> 1-D index: pairs' first members, their mirrors, then the centre
  template <int H> static constexpr int idx(int s) {
    return s < np<H>() ? lo<H>() + s : (s < 2 * np<H>() ? N - 1 - (lo<H>() + s - np<H>()) : C);
  }
};

// own outputs of M L (M = D for SET 0..2, D^T for SET 3..5), slot order of V5Half::idx
template <int P, int SET, int H>
__device__ __forceinline__ void eo_half(const double (&L)[P + 1], double (&out)[V5Half<P>::NSMAX]) {
  using S = V5Half<P>;
  constexpr int N = P + 1, c = P / 2;
  constexpr int base = eoOffset(P) + SET * eoSize(P);
  constexpr int lo = S::template lo<H>(), np = S::template np<H>();
  double ev[c], od[c];
#pragma unroll
  for (int m = 0; m < c; ++m) {
    ev[m] = L[m] + L[N - 1 - m];
    od[m] = L[m] - L[N - 1 - m];
  }
#pragma unroll
  for (int q = 0; q < np; ++q) {
    const int i = lo + q;
    double Sx = 0.0, T = c_EO[base + 2 * c * c + i] * L[c];
#pragma unroll
    for (int m = 0; m < c; ++m) {
      Sx = fma(c_EO[base + i * c + m], od[m], Sx);
      T = fma(c_EO[base + c * c + i * c + m], ev[m], T);
    }
    out[q] = Sx + T;
    out[np + q] = Sx - T;
  }
  if constexpr (H == 1) {
    double M = 0.0;
#pragma unroll
    for (int m = 0; m < c; ++m) M = fma(c_EO[base + 2 * c * c + c + m], od[m], M);
    out[2 * np] = M;
  }
}

#ifndef SFMG_V5_MINB
#define SFMG_V5_MINB 0   // 0: as many blocks per SM as the smem allows (GS), else 1
#endif

template <int P, bool GS>
struct V5Cfg {
  static constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  static constexpr int HALF = ((N2 + 31) / 32) * 32;        // threads per half-element (warp multiple)
  static constexpr int PER_ELEM = (GS ? 9 : 3) * N3 * 8;    // smem bytes per element
  static constexpr int EPB_SMEM = SFMG_V5_SMEM_BUDGET / PER_ELEM > 0 ? SFMG_V5_SMEM_BUDGET / PER_ELEM : 1;
  static constexpr int EPB_THR = 512 / (2 * HALF) > 0 ? 512 / (2 * HALF) : 1;
  static constexpr int EPB = EPB_SMEM < EPB_THR ? EPB_SMEM : EPB_THR;
  static constexpr int THREADS = EPB * 2 * HALF;
  static constexpr size_t SMEM = (size_t)EPB * PER_ELEM + 16;
  static constexpr int MINB_SMEM = (227 * 1024) / (SMEM + 1024) < 8 ? (227 * 1024) / (SMEM + 1024) : 8;
  static constexpr int MINB = SFMG_V5_MINB > 0 ? SFMG_V5_MINB : (GS ? MINB_SMEM : 1);
};

template <int P, bool DIR, bool GS, int H>
__device__ __forceinline__ void v5_element(const MeshDev& m, const double* __restrict__ G,
                                           const double* __restrict__ u, double* __restrict__ v, long long grp,
                                           long long ngroups, long long gstride, int le, int t, double* sU,
                                           double* s0, double* s1, const double* gE, double* sG, uint64_t* bar,
                                           unsigned& phase, bool& waited, int write_bnd,
                                           double (&ru)[V5Half<P>::NSMAX]) {
  using C = V5Cfg<P, GS>;
  using S = V5Half<P>;
  constexpr int N = C::N, N2 = C::N2, N3 = C::N3, NS = S::template ns<H>(), NSM = S::NSMAX;
  constexpr bool EARLY = (P <= 8);
  constexpr int PF = GS ? 2 : SFMG_PF_AHEAD;
  const bool lt = t < N2;
  const int tt = lt ? t : 0;
  const int t0 = tt % N, t1 = tt / N;
  const long long sxy = (long long)m.Mx * m.My;
  auto group_bytes = [&](long long g) -> unsigned {
    long long nel = m.E - g * C::EPB;
    if (nel > C::EPB) nel = C::EPB;
    return (unsigned)(nel * 6 * N3 * sizeof(double));
  };
  auto prefetch_group_l2 = [&](long long g) {
    const char* src = (const char*)(G + g * C::EPB * 6 * N3);
    const unsigned total = group_bytes(g);
    for (unsigned o = 0; o < total; o += 65536u) bulk_prefetch_l2(src + o, total - o < 65536u ? total - o : 65536u);
  };
  // own k slots of this thread's u column of group g (M u: zero on Dirichlet nodes, R4)
  auto load_column = [&](long long g, double (&r)[NSM]) {
    const long long e = g * C::EPB + le;
    const bool act = e < m.E && lt;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    const long long col = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + t0, J = ey * P + t1;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = S::template idx<H>(s);
      bool ok = act;
      if (DIR) { const int K = ez * P + k; ok = ok && !(bxy || K == m.Kb0 || K == m.Kb1); }
      r[s] = ok ? __ldg(u + col + sxy * k) : 0.0;
    }
  };
  auto prefetch_column = [&](long long g) {
    const long long e = g * C::EPB + le;
    if (e >= m.E || !lt) return;
    int ex, ey, ez;
    elem_coords(m, e, ex, ey, ez);
    const double* pu = u + (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
#pragma unroll
    for (int s = 0; s < NS; ++s) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + sxy * S::template idx<H>(s)));
  };

  const long long e = grp * C::EPB + le;
  const bool act = e < m.E;
  int ex = 0, ey = 0, ez = 0;
  if (act) elem_coords(m, e, ex, ey, ez);
  const long long gcol = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
  bool bxy = false;
  if (DIR) {
    const int I = ex * P + t0, J = ey * P + t1;
    bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
  }
  if (!EARLY) load_column(grp, ru);
  if (lt) {
#pragma unroll
    for (int s = 0; s < NS; ++s) sU[t + N2 * S::template idx<H>(s)] = ru[s];
  }
  if (EARLY && grp + gstride < ngroups) {   // next group's own slots, in flight during the element
    load_column(grp + gstride, ru);
    if (grp + 2 * gstride < ngroups) prefetch_column(grp + 2 * gstride);
  } else if (!EARLY && grp + gstride < ngroups) {
    prefetch_column(grp + gstride);
  }
  const double* Gg = G + (act ? e : 0) * 6 * N3 + tt;   // !GS: this thread's factor column
  constexpr int RG = SFMG_RING < NS + 1 ? SFMG_RING : NS + 1;
  double gb[RG][6];
  if (!GS) {
#pragma unroll
    for (int kk = 0; kk < RG - 1 && kk < NS; ++kk)
#pragma unroll
      for (int c = 0; c < 6; ++c) gb[kk][c] = __ldcs(Gg + gofs<N>(c, 0, S::template idx<H>(kk)));
  }
  __syncthreads();
  double g2[NSM];
  if (lt) {  // A: forward contractions of the three lines through (t0, t1)
    double L[N], o[NSM];
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = sU[mm + N * t0 + N2 * t1];
    eo_half<P, 0, H>(L, o);
#pragma unroll
    for (int s = 0; s < NS; ++s) s0[S::template idx<H>(s) + N * t0 + N2 * t1] = o[s];
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = sU[t0 + N * mm + N2 * t1];
    eo_half<P, 1, H>(L, o);
#pragma unroll
    for (int s = 0; s < NS; ++s) s1[t0 + N * S::template idx<H>(s) + N2 * t1] = o[s];
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = sU[t + N2 * mm];
    eo_half<P, 2, H>(L, g2);
  }
  __syncthreads();
  if (GS) {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  if (lt) {  // B: pointwise w = G g at (t, own k)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = S::template idx<H>(s);
      double G00, G01, G02, G11, G12, G22;
      if (GS) {
        const double* Gk = gE + gofs<N>(0, t, k);
        G00 = Gk[0]; G01 = Gk[N2]; G02 = Gk[2 * N2]; G11 = Gk[3 * N2]; G12 = Gk[4 * N2]; G22 = Gk[5 * N2];
      } else {
        if (s + RG - 1 < NS) {
#pragma unroll
          for (int c = 0; c < 6; ++c)
            gb[(s + RG - 1) % RG][c] = __ldcs(Gg + gofs<N>(c, 0, S::template idx<H>(s + RG - 1)));
        }
        G00 = gb[s % RG][0]; G01 = gb[s % RG][1]; G02 = gb[s % RG][2];
        G11 = gb[s % RG][3]; G12 = gb[s % RG][4]; G22 = gb[s % RG][5];
      }
      const int q = t + N2 * k;
      const double a0 = s0[q], a1 = s1[q], a2 = g2[s];
      s0[q] = G00 * a0 + G01 * a1 + G02 * a2;
      s1[q] = G01 * a0 + G11 * a1 + G12 * a2;
      sU[q] = G02 * a0 + G12 * a1 + G22 * a2;
    }
  }
  __syncthreads();
  {  // factors consumed: next group's G (TMA) and the L2 prefetch ahead of it
    const long long nx = grp + gstride;
    if (nx < ngroups && threadIdx.x == 0) {
      if (GS) {
        fence_proxy_async_smem();
        bulk_load(sG, G + nx * C::EPB * 6 * N3, group_bytes(nx), bar);
      }
      if (PF >= 2 && nx + gstride < ngroups) prefetch_group_l2(nx + gstride);
      else if (PF == 1) prefetch_group_l2(nx);
    }
  }
  double X[NSM], Y[NSM];
  if (lt) {  // C1: transposed contractions of the x- and y-lines (own outputs kept in registers)
    double L[N];
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = s0[mm + N * t0 + N2 * t1];
    eo_half<P, 4, H>(L, X);
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = s1[t0 + N * mm + N2 * t1];
    eo_half<P, 5, H>(L, Y);
  }
  __syncthreads();
  if (lt) {  // C2: in place
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      s0[S::template idx<H>(s) + N * t0 + N2 * t1] = X[s];
      s1[t0 + N * S::template idx<H>(s) + N2 * t1] = Y[s];
    }
  }
  __syncthreads();
  if (!waited) {
    pdl_wait();
    waited = true;
  }
  if (act && lt) {  // C3: z-line D^T w2, v = X + Y + Z at own k, scatter
    double L[N], Z[NSM];
#pragma unroll
    for (int mm = 0; mm < N; ++mm) L[mm] = sU[t + N2 * mm];
    eo_half<P, 3, H>(L, Z);
    const bool own_xy = (t0 > 0 || ex == 0) && (t1 > 0 || ey == 0);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int c = S::template idx<H>(s);
      bool bnd = false;
      if (DIR) { const int K = ez * P + c; bnd = bxy || K == m.Kb0 || K == m.Kb1; }
      if (!bnd) atomicAdd(v + gcol + sxy * c, s0[t + N2 * c] + s1[t + N2 * c] + Z[s]);
      else if (write_bnd && own_xy && (c > 0 || ez == 0)) v[gcol + sxy * c] = u[gcol + sxy * c];   // (I-M) u
    }
  }
}

template <int P, bool DIR, bool GS>
__global__ void __launch_bounds__(V5Cfg<P, GS>::THREADS, V5Cfg<P, GS>::MINB)
    k_apply_v5(MeshDev m, const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ v,
               long long ngroups, int wait_mode, int write_bnd) {
  using C = V5Cfg<P, GS>;
  using S = V5Half<P>;
  constexpr int N3 = C::N3;
  extern __shared__ __align__(128) double smem[];
  double* sG = smem;                                   // [EPB][k][6][n^2] (GS)
  const int wsel = threadIdx.x / C::HALF;              // 2 le + h, warp-uniform
  const int le = wsel >> 1, h = wsel & 1;
  const int t = threadIdx.x - wsel * C::HALF;
  double* sU = smem + (GS ? C::EPB * 6 * N3 : 0) + le * 3 * N3;
  double* s0 = sU + N3;
  double* s1 = s0 + N3;
  uint64_t* bar = (uint64_t*)(smem + C::EPB * (GS ? 9 : 3) * N3);
  const double* gE = sG + le * 6 * N3;
  const long long gstride = gridDim.x;
  long long grp = blockIdx.x;
  if (threadIdx.x == 0) {
    auto group_bytes = [&](long long g) -> unsigned {
      long long nel = m.E - g * C::EPB;
      if (nel > C::EPB) nel = C::EPB;
      return (unsigned)(nel * 6 * N3 * sizeof(double));
    };
    auto pf = [&](long long g) {
      const char* src = (const char*)(G + g * C::EPB * 6 * N3);
      const unsigned total = group_bytes(g);
      for (unsigned o = 0; o < total; o += 65536u) bulk_prefetch_l2(src + o, total - o < 65536u ? total - o : 65536u);
    };
    constexpr int PF = GS ? 2 : SFMG_PF_AHEAD;
    if (GS) {
      mbar_init(bar, 1);
      if (grp < ngroups) bulk_load(sG, G + grp * C::EPB * 6 * N3, group_bytes(grp), bar);
    } else if (grp < ngroups && PF >= 1) {
      pf(grp);
    }
    if (PF >= 2 && grp + gstride < ngroups) pf(grp + gstride);
  }
  if (wait_mode == 2) pdl_wait();
  bool waited = (wait_mode != 1);
  unsigned phase = 0;
  double ru[S::NSMAX];
  // first column (EARLY path): identical to v5_element's load_column for group grp
  if (P <= 8 && grp < ngroups) {
    const long long e = grp * C::EPB + le;
    const bool act = e < m.E && t < C::N2;
    const int tt = t < C::N2 ? t : 0, t0 = tt % C::N, t1 = tt / C::N;
    int ex = 0, ey = 0, ez = 0;
    if (act) elem_coords(m, e, ex, ey, ez);
    const long long sxy = (long long)m.Mx * m.My;
    const long long col = (long long)(ex * P + t0) + (long long)m.Mx * (ey * P + t1) + sxy * (long long)(ez * P);
    bool bxy = false;
    if (DIR) {
      const int I = ex * P + t0, J = ey * P + t1;
      bxy = (I == 0) || (I == m.Mx - 1) || (J == 0) || (J == m.My - 1);
    }
    if (h == 0) {
#pragma unroll
      for (int s = 0; s < S::template ns<0>(); ++s) {
        const int k = S::template idx<0>(s);
        bool ok = act;
        if (DIR) { const int K = ez * P + k; ok = ok && !(bxy || K == m.Kb0 || K == m.Kb1); }
        ru[s] = ok ? __ldg(u + col + sxy * k) : 0.0;
      }
    } else {
#pragma unroll
      for (int s = 0; s < S::template ns<1>(); ++s) {
        const int k = S::template idx<1>(s);
        bool ok = act;
        if (DIR) { const int K = ez * P + k; ok = ok && !(bxy || K == m.Kb0 || K == m.Kb1); }
        ru[s] = ok ? __ldg(u + col + sxy * k) : 0.0;
      }
    }
  }
  for (; grp < ngroups; grp += gstride) {
    if (h == 0)
      v5_element<P, DIR, GS, 0>(m, G, u, v, grp, ngroups, gstride, le, t, sU, s0, s1, gE, sG, bar, phase, waited,
                                write_bnd, ru);
    else
      v5_element<P, DIR, GS, 1>(m, G, u, v, grp, ngroups, gstride, le, t, sU, s0, s1, gE, sG, bar, phase, waited,
                                write_bnd, ru);
  }
}
