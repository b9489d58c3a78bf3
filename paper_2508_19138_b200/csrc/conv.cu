// Energy convolutions of the GW step, fused per entry row (sm_100a).
//
// Reference: negfgw/convolve.py
//   convolve_energy  convolve.py:39-71   linear convolution / correlation via FFT
//   retarded_from_lg convolve.py:101-129 r = ifft_m(theta * fft_m(X^> - X^<))[:N],
//                    m = next_fast_len(2N) (even), theta = [1/2, 1, .., 1, 1/2, 0, ..]
// and the pipeline around them in scba_run: P (scba.py:1035-1048),
// Sigma (scba.py:1118-1132), diagonal projection (scba.py:406-409).
//
// Every operation here is a linear convolution of length-N energy series, so
// one power-of-two circular length L >= 2N-1 reproduces all of them exactly
// (to roundoff) independent of scipy's padding: the causal reconstruction is
// the convolution of d with the fixed kernel K = ifft_m(theta) restricted to
// lags |n| < N, whose spectrum on the L grid (kf, and kcf for conj(K)) is
// precomputed once per N on the host.
//
// One CTA of L/8 threads owns one entry row (HBM traffic: one read of the
// input series, one write of the outputs): radix-8 Stockham transforms with
// the data in registers and padded shared memory only between passes (see
// the row FFT engine below); spectra stay in natural order, so pointwise
// products and the next transform need no permutation. Polarization uses
//   P^<_hat = G^<_hat * (-conj G^>_hat)   and   P^>[k] = conj(p^<[-k]),
// i.e. one inverse transform yields both P^< and P^>.
#include "../../include/negf_b200.h"
#include "common.cuh"
#include "prof.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace negf {
namespace {

// ---------------------------------------------------------------------------
// Row FFT engine: Stockham (auto-sort) passes of radix E (8 or 16) with the
// data of a pass held in registers, shared memory only for the exchange
// between passes. A CTA of L/E threads owns one row; thread t holds the E
// elements at positions t + s*L/E (s < E). Every pass READS exactly those
// positions, and the last pass WRITES them (Stockham with Ns*R = L), so the
// spectrum left in registers by a forward transform is where the pointwise
// products and the next inverse transform expect it: consecutive transforms
// never round-trip through shared memory. log2(L) = log2(E) pE + log2(Rs):
// the small radix Rs runs first in forward and last in inverse transforms
// (the same positions rule holds for it). Shared indices are padded by one
// element per 8 (conflict-free 16-byte accesses).

__device__ __forceinline__ int pidx(int i) { return i + (i >> 3); }

template <bool INV>
__device__ __forceinline__ z_t rot(z_t a) {  // * (-i) forward, * (+i) inverse
  return INV ? zmake(-a.y, a.x) : zmake(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(z_t& a, z_t& b) {
  const z_t t = a;
  a = zadd(t, b);
  b = zsub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(z_t& v0, z_t& v1, z_t& v2, z_t& v3) {
  const z_t t0 = zadd(v0, v2), t1 = zsub(v0, v2), t2 = zadd(v1, v3), t3 = rot<INV>(zsub(v1, v3));
  v0 = zadd(t0, t2);
  v1 = zadd(t1, t3);
  v2 = zsub(t0, t2);
  v3 = zsub(t1, t3);
}

// x * exp(-/+ 2 pi i q / 16), q static
template <bool INV, int q>
__device__ __forceinline__ z_t w16(z_t x) {
  constexpr double c[5] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173, 0.0};
  constexpr int qq = q & 15;
  if constexpr (qq == 0) return x;
  if constexpr (qq == 4) return rot<INV>(x);
  if constexpr (qq == 8) return zmake(-x.x, -x.y);
  if constexpr (qq == 12) return rot<!INV>(x);
  // cos and sin of 2 pi qq / 16
  constexpr int a = qq % 8;
  constexpr double cs = a <= 4 ? c[a] : -c[8 - a];
  constexpr double sn = a <= 4 ? c[4 - a] : c[a - 4];
  constexpr double cq = qq < 8 ? cs : -cs, sq = qq < 8 ? sn : -sn;
  // forward: * (cos - i sin), inverse: * (cos + i sin)
  return INV ? zmake(x.x * cq - x.y * sq, x.x * sq + x.y * cq) : zmake(x.x * cq + x.y * sq, x.y * cq - x.x * sq);
}

template <bool INV>
__device__ __forceinline__ void dft8(z_t* v) {
  z_t e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  z_t o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = w16<INV, 2>(o1);
  o2 = w16<INV, 4>(o2);
  o3 = w16<INV, 6>(o3);
  v[0] = zadd(e0, o0); v[4] = zsub(e0, o0);
  v[1] = zadd(e1, o1); v[5] = zsub(e1, o1);
  v[2] = zadd(e2, o2); v[6] = zsub(e2, o2);
  v[3] = zadd(e3, o3); v[7] = zsub(e3, o3);
}

// natural order in and out: n = 4 n1 + n2, k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft16(z_t* v) {
  z_t a[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    z_t x0 = v[n2], x1 = v[n2 + 4], x2 = v[n2 + 8], x3 = v[n2 + 12];
    dft4<INV>(x0, x1, x2, x3);  // over n1 -> k1
    a[0][n2] = x0; a[1][n2] = x1; a[2][n2] = x2; a[3][n2] = x3;
  }
  a[1][1] = w16<INV, 1>(a[1][1]); a[1][2] = w16<INV, 2>(a[1][2]); a[1][3] = w16<INV, 3>(a[1][3]);
  a[2][1] = w16<INV, 2>(a[2][1]); a[2][2] = w16<INV, 4>(a[2][2]); a[2][3] = w16<INV, 6>(a[2][3]);
  a[3][1] = w16<INV, 3>(a[3][1]); a[3][2] = w16<INV, 6>(a[3][2]); a[3][3] = w16<INV, 9>(a[3][3]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    dft4<INV>(a[k1][0], a[k1][1], a[k1][2], a[k1][3]);  // over n2 -> k2
    v[k1] = a[k1][0]; v[k1 + 4] = a[k1][1]; v[k1 + 8] = a[k1][2]; v[k1 + 12] = a[k1][3];
  }
}

template <bool INV, int R>
__device__ __forceinline__ void dft_r(z_t* e) {
  if constexpr (R == 16) dft16<INV>(e);
  else if constexpr (R == 8) dft8<INV>(e);
  else if constexpr (R == 4) dft4<INV>(e[0], e[1], e[2], e[3]);
  else dft2<INV>(e[0], e[1]);
}

// CTAs of PACK_T threads are register-capped for 3 resident CTAs per SM
// (the Sigma kernel otherwise takes 173 registers and drops to 2).
// Short rows (Q = L/E < PACK_T threads) are packed PACK_T / Q to a CTA of
// PACK_T threads, each row with its own shared-memory slice: one row per CTA
// at L = 16 would run 2 of 32 threads and launch one CTA per entry row.
constexpr int PACK_T = 128;
#ifndef NEGF_CONV_PACK_MINB
#define NEGF_CONV_PACK_MINB 3
#endif
constexpr int kPackMinB = NEGF_CONV_PACK_MINB;  // resident CTAs per SM of the packed-row kernels

__host__ __device__ __forceinline__ int rows_per_cta(int L, int E) {
  const int q = L / E;
  return q < PACK_T ? PACK_T / q : 1;
}

template <int E>
struct RowGeom {
  int L, Q;    // Q = L/E threads carry data
  int pE, rs;  // radix-E passes, small radix (0 or 2 .. E/2)
  int tws;     // stride of the twiddle table (2: the L/2-point engine of the cluster kernels reads the L table)
  int t;
  int sub;     // row slot within the CTA
  bool act;
};

template <int E>
__device__ __forceinline__ RowGeom<E> row_geom(int L, long long n_rows, long long& row) {
  constexpr int lg = E == 16 ? 4 : 3;
  RowGeom<E> g;
  g.L = L;
  g.Q = L / E;
  const int m = 31 - __clz(L);
  g.pE = m / lg;
  g.rs = (m % lg) ? (1 << (m % lg)) : 0;
  const int rpc = rows_per_cta(L, E);
  g.tws = 1;
  g.t = rpc > 1 ? threadIdx.x % g.Q : threadIdx.x;
  g.sub = rpc > 1 ? threadIdx.x / g.Q : 0;
  row = (long long)blockIdx.x * rpc + g.sub;
  g.act = g.t < g.Q && row < n_rows;
  if (row >= n_rows) row = n_rows - 1;  // idle slot: keep table reads in bounds
  return g;
}

// One Stockham pass of radix R on NA arrays held in registers (in place).
// R is a template parameter so every register index is static.
template <bool INV, int E, int NA, int R>
__device__ __forceinline__ void pass_compute(z_t (*v)[E], const RowGeom<E>& g, int Ns, const z_t* __restrict__ tw) {
  constexpr int NB = E / R;  // butterflies per thread; element r of butterfly u in slot u + r*NB
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int j = g.t + u * g.Q, k = j & (Ns - 1);
    if (Ns > 1) {
      // one table twiddle per butterfly, its powers by multiplication (the
      // L1/shared pipe, not FP64, bounds these kernels)
      const int step = k * (g.L / (Ns * R)) * g.tws;
      z_t w1 = __ldg(&tw[step]);
      if (INV) w1 = zconj(w1);
      z_t w = w1;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        if (r > 1) w = zmul(w, w1);
#pragma unroll
        for (int a = 0; a < NA; ++a) v[a][u + r * NB] = zmul(v[a][u + r * NB], w);
      }
    }
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      if constexpr (NB == 1) {
        dft_r<INV, R>(v[a]);
      } else {
        z_t e[R];
#pragma unroll
        for (int r = 0; r < R; ++r) e[r] = v[a][u + r * NB];
        dft_r<INV, R>(e);
#pragma unroll
        for (int r = 0; r < R; ++r) v[a][u + r * NB] = e[r];
      }
    }
  }
}

template <int E, int NA, int R>
__device__ __forceinline__ void pass_store(z_t (*v)[E], z_t* const* sm, const RowGeom<E>& g, int Ns) {
  constexpr int NB = E / R;
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int j = g.t + u * g.Q, k = j & (Ns - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int a = 0; a < NA; ++a) sm[a][pidx(base + r * Ns)] = v[a][u + r * NB];
  }
}

template <bool INV, int E, int NA, int R>
__device__ __forceinline__ void fft_pass(z_t (*v)[E], z_t* const* sm, const RowGeom<E>& g, int Ns,
                                         const z_t* __restrict__ tw, bool load, bool store) {
  if (load) {
    if (g.act) {
#pragma unroll
      for (int s = 0; s < E; ++s)
#pragma unroll
        for (int a = 0; a < NA; ++a) v[a][s] = sm[a][pidx(g.t + s * g.Q)];
    }
    __syncthreads();
  }
  if (g.act) pass_compute<INV, E, NA, R>(v, g, Ns, tw);
  if (store) {
    if (g.act) pass_store<E, NA, R>(v, sm, g, Ns);
    __syncthreads();
  }
}

// Forward (INV = false) or unscaled inverse transform of NA rows in registers.
template <bool INV, int E, int NA>
__device__ void fft_rows(z_t (*v)[E], z_t* const* sm, const RowGeom<E>& g, const z_t* __restrict__ tw) {
  const int npass = g.pE + (g.rs ? 1 : 0);
  int Ns = 1;
  for (int p = 0; p < npass; ++p) {
    const bool small = g.rs && (INV ? p == npass - 1 : p == 0);
    const bool load = p > 0, store = p != npass - 1;
    if (!small) {
      fft_pass<INV, E, NA, E>(v, sm, g, Ns, tw, load, store);
      Ns *= E;
    } else if (E == 16 && g.rs == 8) {
      fft_pass<INV, E, NA, (E == 16 ? 8 : 4)>(v, sm, g, Ns, tw, load, store);
      Ns *= 8;
    } else if (g.rs == 4) {
      fft_pass<INV, E, NA, 4>(v, sm, g, Ns, tw, load, store);
      Ns *= 4;
    } else {
      fft_pass<INV, E, NA, 2>(v, sm, g, Ns, tw, load, store);
      Ns *= 2;
    }
  }
}

__device__ __forceinline__ z_t proj(z_t v, bool diag) {
  // (v - conj v)/2 on diagonal entries (scba.py:406-409)
  return diag ? make_double2(0.0, v.y) : v;
}

// d (registers, natural positions) -> r_up = K*d, r_lo = -conj(conj(K)*d)
template <int E>
__device__ void retarded_tail(z_t* d, z_t* A, z_t* B, const RowGeom<E>& g, int n, const z_t* tw, const z_t* kf,
                              const z_t* kcf, z_t* r_up, z_t* r_lo) {
  z_t* sB[1] = {B};
  z_t dv[1][E];
#pragma unroll
  for (int s = 0; s < E; ++s) dv[0][s] = d[s];
  fft_rows<false, E, 1>(dv, sB, g, tw);
  z_t xy[2][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int q = g.t + s * g.Q;
    xy[0][s] = g.act ? zmul(dv[0][s], __ldg(&kf[q])) : make_double2(0.0, 0.0);
    xy[1][s] = g.act && kcf ? zmul(dv[0][s], __ldg(&kcf[q])) : make_double2(0.0, 0.0);
  }
  z_t* sAB[2] = {A, B};
  fft_rows<true, E, 2>(xy, sAB, g, tw);
  const double inv = 1.0 / g.L;
  if (g.act) {
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = g.t + s * g.Q;
      if (k < n) {
        if (r_up) r_up[k] = zscale(inv, xy[0][s]);
        if (r_lo) r_lo[k] = zscale(-inv, zconj(xy[1][s]));
      }
    }
  }
}

template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == PACK_T ? kPackMinB : MAXT == 256 ? 2 : 1) pol_kernel(const z_t* __restrict__ gl, const z_t* __restrict__ gg, int n,
                                                   int L, const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                                                   const z_t* __restrict__ kcf,
                                                   const unsigned char* __restrict__ diag, double2 scale, z_t* pl,
                                                   z_t* pg, z_t* pr_up, z_t* pr_lo, long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  long long row;
  const RowGeom<E> g = row_geom<E>(L, n_rows, row);
  z_t* A = sm + 2 * g.sub * pidx(L);
  z_t* B = A + pidx(L);
  const long long o = row * n;
  const bool dg = diag && diag[row];
  z_t v[2][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k = g.t + s * g.Q;
    const bool in = g.act && k < n;
    v[0][s] = in ? gl[o + k] : make_double2(0.0, 0.0);
    v[1][s] = in ? gg[o + k] : make_double2(0.0, 0.0);
  }
  z_t* sAB[2] = {A, B};
  fft_rows<false, E, 2>(v, sAB, g, tw);
#pragma unroll
  for (int s = 0; s < E; ++s) v[0][s] = zmul(v[0][s], make_double2(-v[1][s].x, v[1][s].y));  // * (-conj G^>)
  z_t* sA[1] = {A};
  fft_rows<true, E, 1>(v, sA, g, tw);
  // P^>[k] = conj(p[-k]): exchange p through shared memory
  if (g.act) {
#pragma unroll
    for (int s = 0; s < E; ++s) A[pidx(g.t + s * g.Q)] = v[0][s];
  }
  __syncthreads();
  const z_t sc = zscale(1.0 / L, scale);
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k = g.t + s * g.Q;
    z_t d = make_double2(0.0, 0.0);
    if (g.act && k < n) {
      const z_t lo = proj(zmul(sc, v[0][s]), dg);
      const z_t gr = proj(zmul(sc, zconj(A[pidx((L - k) & (L - 1))])), dg);
      pl[o + k] = lo;
      pg[o + k] = gr;
      d = zsub(gr, lo);
    }
    v[1][s] = d;
  }
  __syncthreads();
  retarded_tail<E>(v[1], A, B, g, n, tw, kf, kcf, pr_up ? pr_up + o : nullptr, pr_lo ? pr_lo + o : nullptr);
}

template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == PACK_T ? kPackMinB : MAXT == 256 ? 2 : 1) sigma_kernel(const z_t* __restrict__ gl, const z_t* __restrict__ gg,
                                                     const z_t* __restrict__ wl, const z_t* __restrict__ wg,
                                                     const long long* __restrict__ w_rows, int n, int L,
                                                     const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                                                     const z_t* __restrict__ kcf,
                                                     const unsigned char* __restrict__ diag, double2 scale, z_t* sl,
                                                     z_t* sg, z_t* sr_up, z_t* sr_lo, long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  long long row;
  const RowGeom<E> g = row_geom<E>(L, n_rows, row);
  z_t* A = sm + 2 * g.sub * pidx(L);
  z_t* B = A + pidx(L);
  const long long o = row * n;
  const long long ow = (w_rows ? w_rows[row] : row) * n;
  const bool dg = diag && diag[row];
  const z_t sc = zscale(1.0 / L, scale);
  z_t* sAB[2] = {A, B};
  z_t* sA[1] = {A};
  z_t v[2][E];
#pragma unroll 1
  for (int kind = 0; kind < 2; ++kind) {
    const z_t* gx = kind ? gg : gl;
    const z_t* wx = kind ? wg : wl;
    z_t* out = kind ? sg : sl;
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = g.t + s * g.Q;
      const bool in = g.act && k < n;
      v[0][s] = in ? gx[o + k] : make_double2(0.0, 0.0);
      v[1][s] = in ? wx[ow + k] : make_double2(0.0, 0.0);
    }
    fft_rows<false, E, 2>(v, sAB, g, tw);
#pragma unroll
    for (int s = 0; s < E; ++s) v[0][s] = zmul(v[0][s], v[1][s]);
    fft_rows<true, E, 1>(v, sA, g, tw);
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = g.t + s * g.Q;
      // after the second kind, v[1] <- d = Sigma^> - Sigma^<, Sigma^< re-read
      // from the values this thread wrote itself
      v[1][s] = make_double2(0.0, 0.0);
      if (g.act && k < n) {
        const z_t val = proj(zmul(sc, v[0][s]), dg);
        out[o + k] = val;
        if (kind == 1) v[1][s] = zsub(val, sl[o + k]);
      }
    }
  }
  retarded_tail<E>(v[1], A, B, g, n, tw, kf, kcf, sr_up ? sr_up + o : nullptr, sr_lo ? sr_lo + o : nullptr);
}

// ---------------------------------------------------------------------------
// N_E in (2048, 4096] (C4's 4096 energies): circular grid L = 8192, split
// over a CLUSTER OF TWO CTAs (one per SM, distributed shared memory), each
// running the L/2-point engine above. A zero-padded length-L transform is two
// length-M = L/2 transforms, of x and of x w^j (w = e^{-2 pi i / L}): the
// even and the odd frequency bins. The pointwise spectral products act bin by
// bin, so CTA h (= cluster rank) owns the bins of parity h end to end:
//   forward M-point transforms of x w^{h j} -> product -> inverse -> Y_h,
// and the length-L inverse comes back as
//   L y[j] = Y_0[j mod M] + e^{+2 pi i j / L} Y_1[j mod M],
// each CTA reading its peer's Y through DSMEM and writing half of the outputs.
// The difference series d feeding the causal (retarded) kernel is exchanged
// the same way, and the kernel spectra are read at bins 2q + h. HBM traffic is
// that of the one-CTA kernels (each CTA reads the whole input row; the peer's
// read of the same row is served by L2).

template <int E>
__device__ __forceinline__ RowGeom<E> geom_x2(int M) {
  constexpr int lg = E == 16 ? 4 : 3;
  RowGeom<E> g;
  g.L = M;
  g.Q = M / E;
  const int m = 31 - __clz(M);
  g.pE = m / lg;
  g.rs = (m % lg) ? (1 << (m % lg)) : 0;
  g.tws = 2;
  g.t = threadIdx.x;
  g.sub = 0;
  g.act = true;
  return g;
}

// L y[k] (and L y[-k mod L] when REV) from the two CTAs' inverse halves
// Ye (bins of parity 0) / Yo (parity 1), k < M.
__device__ __forceinline__ z_t combine_x2(const z_t* Ye, const z_t* Yo, int k, z_t wk) {
  return zadd(Ye[pidx(k)], zmul(zconj(wk), Yo[pidx(k)]));
}
__device__ __forceinline__ z_t combine_x2_rev(const z_t* Ye, const z_t* Yo, int k, int M, z_t wk) {
  const int km = (M - k) & (M - 1);
  return zadd(Ye[pidx(km)], zmul(wk, Yo[pidx(km)]));
}

// Causal tail on the split grid: d (length M, zero beyond n) sits in this
// CTA's B; r_up = K*d, r_lo = -conj(conj(K)*d) for this CTA's output half.
template <int E>
__device__ void retarded_tail_x2(cg::cluster_group& cl, int h, z_t* A, z_t* B, const RowGeom<E>& g, int n, int L,
                                 const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                                 const z_t* __restrict__ kcf, z_t* r_up, z_t* r_lo) {
  z_t dv[1][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int j = g.t + s * g.Q;
    const z_t x = B[pidx(j)];
    dv[0][s] = h ? zmul(x, __ldg(&tw[j])) : x;
  }
  z_t* sA[1] = {A};
  fft_rows<false, E, 1>(dv, sA, g, tw);
  z_t xy[2][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int q = 2 * (g.t + s * g.Q) + h;
    xy[0][s] = zmul(dv[0][s], __ldg(&kf[q]));
    xy[1][s] = kcf ? zmul(dv[0][s], __ldg(&kcf[q])) : make_double2(0.0, 0.0);
  }
  z_t* sAB[2] = {A, B};
  fft_rows<true, E, 2>(xy, sAB, g, tw);
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int j = g.t + s * g.Q;
    A[pidx(j)] = xy[0][s];
    B[pidx(j)] = xy[1][s];
  }
  cl.sync();
  const int M = g.L;
  const z_t* Ar = cl.map_shared_rank(A, h ^ 1);
  const z_t* Br = cl.map_shared_rank(B, h ^ 1);
  const z_t *Ue = h ? Ar : A, *Uo = h ? A : Ar, *Le = h ? Br : B, *Lo = h ? B : Br;
  const double inv = 1.0 / L;
#pragma unroll
  for (int si = 0; si < E / 2; ++si) {
    const int k = g.t + (h * (E / 2) + si) * g.Q;
    if (k < n) {
      const z_t wk = __ldg(&tw[k]);
      if (r_up) r_up[k] = zscale(inv, combine_x2(Ue, Uo, k, wk));
      if (r_lo) r_lo[k] = zscale(-inv, zconj(combine_x2(Le, Lo, k, wk)));
    }
  }
  (void)M;
  cl.sync();  // the peer may still read this CTA's A / B
}

template <int E>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    pol_kernel_x2(const z_t* __restrict__ gl, const z_t* __restrict__ gg, int n, int L, const z_t* __restrict__ tw,
                  const z_t* __restrict__ kf, const z_t* __restrict__ kcf, const unsigned char* __restrict__ diag,
                  double2 scale, z_t* pl, z_t* pg, z_t* pr_up, z_t* pr_lo, long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int h = (int)cl.block_rank();
  const long long row = blockIdx.x >> 1;
  const int M = L >> 1;
  const RowGeom<E> g = geom_x2<E>(M);
  z_t* A = sm;
  z_t* B = sm + pidx(M);
  const long long o = row * n;
  const bool dg = diag && diag[row];
  z_t v[2][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int j = g.t + s * g.Q;
    z_t a = make_double2(0.0, 0.0), b = a;
    if (j < n) {
      a = gl[o + j];
      b = gg[o + j];
      if (h) {
        const z_t w = __ldg(&tw[j]);
        a = zmul(a, w);
        b = zmul(b, w);
      }
    }
    v[0][s] = a;
    v[1][s] = b;
  }
  z_t* sAB[2] = {A, B};
  fft_rows<false, E, 2>(v, sAB, g, tw);
#pragma unroll
  for (int s = 0; s < E; ++s) v[0][s] = zmul(v[0][s], make_double2(-v[1][s].x, v[1][s].y));  // * (-conj G^>)
  z_t* sA[1] = {A};
  fft_rows<true, E, 1>(v, sA, g, tw);
#pragma unroll
  for (int s = 0; s < E; ++s) A[pidx(g.t + s * g.Q)] = v[0][s];
  cl.sync();
  const z_t* Ar = cl.map_shared_rank(A, h ^ 1);
  z_t* Br = cl.map_shared_rank(B, h ^ 1);
  const z_t *Ye = h ? Ar : A, *Yo = h ? A : Ar;
  const z_t sc = zscale(1.0 / L, scale);
#pragma unroll
  for (int si = 0; si < E / 2; ++si) {
    const int k = g.t + (h * (E / 2) + si) * g.Q;
    z_t d = make_double2(0.0, 0.0);
    if (k < n) {
      const z_t wk = __ldg(&tw[k]);
      const z_t lo = proj(zmul(sc, combine_x2(Ye, Yo, k, wk)), dg);
      const z_t gr = proj(zmul(sc, zconj(combine_x2_rev(Ye, Yo, k, M, wk))), dg);
      pl[o + k] = lo;
      pg[o + k] = gr;
      d = zsub(gr, lo);
    }
    B[pidx(k)] = d;  // both CTAs need the whole difference series
    Br[pidx(k)] = d;
  }
  cl.sync();
  retarded_tail_x2<E>(cl, h, A, B, g, n, L, tw, kf, kcf, pr_up ? pr_up + o : nullptr, pr_lo ? pr_lo + o : nullptr);
}

template <int E>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    sigma_kernel_x2(const z_t* __restrict__ gl, const z_t* __restrict__ gg, const z_t* __restrict__ wl,
                    const z_t* __restrict__ wg, const long long* __restrict__ w_rows, int n, int L,
                    const z_t* __restrict__ tw, const z_t* __restrict__ kf, const z_t* __restrict__ kcf,
                    const unsigned char* __restrict__ diag, double2 scale, z_t* sl, z_t* sg, z_t* sr_up, z_t* sr_lo,
                    long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int h = (int)cl.block_rank();
  const long long row = blockIdx.x >> 1;
  const int M = L >> 1;
  const RowGeom<E> g = geom_x2<E>(M);
  z_t* A = sm;
  z_t* B = sm + pidx(M);
  const long long o = row * n;
  const long long ow = (w_rows ? w_rows[row] : row) * n;
  const bool dg = diag && diag[row];
  const z_t sc = zscale(1.0 / L, scale);
  const z_t* Ar = cl.map_shared_rank(A, h ^ 1);
  z_t* Br = cl.map_shared_rank(B, h ^ 1);
  const z_t *Ye = h ? Ar : A, *Yo = h ? A : Ar;
  z_t* sAB[2] = {A, B};
  z_t* sA[1] = {A};
  z_t s_less[E / 2];
  z_t v[2][E];
#pragma unroll 1
  for (int kind = 0; kind < 2; ++kind) {
    const z_t* gx = kind ? gg : gl;
    const z_t* wx = kind ? wg : wl;
    z_t* out = kind ? sg : sl;
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int j = g.t + s * g.Q;
      z_t a = make_double2(0.0, 0.0), b = a;
      if (j < n) {
        a = gx[o + j];
        b = wx[ow + j];
        if (h) {
          const z_t w = __ldg(&tw[j]);
          a = zmul(a, w);
          b = zmul(b, w);
        }
      }
      v[0][s] = a;
      v[1][s] = b;
    }
    fft_rows<false, E, 2>(v, sAB, g, tw);
#pragma unroll
    for (int s = 0; s < E; ++s) v[0][s] = zmul(v[0][s], v[1][s]);
    fft_rows<true, E, 1>(v, sA, g, tw);
#pragma unroll
    for (int s = 0; s < E; ++s) A[pidx(g.t + s * g.Q)] = v[0][s];
    cl.sync();
#pragma unroll
    for (int si = 0; si < E / 2; ++si) {
      const int k = g.t + (h * (E / 2) + si) * g.Q;
      z_t val = make_double2(0.0, 0.0);
      if (k < n) {
        val = proj(zmul(sc, combine_x2(Ye, Yo, k, __ldg(&tw[k]))), dg);
        out[o + k] = val;
      }
      if (kind == 0) {
        s_less[si] = val;
      } else {
        const z_t d = zsub(val, s_less[si]);
        B[pidx(k)] = d;
        Br[pidx(k)] = d;
      }
    }
    cl.sync();  // the peer is done reading this CTA's A before it is rewritten
  }
  retarded_tail_x2<E>(cl, h, A, B, g, n, L, tw, kf, kcf, sr_up ? sr_up + o : nullptr, sr_lo ? sr_lo + o : nullptr);
}

// Generic convolve_energy (convolve.py:39-71): mode 0 convolution, 1 correlation.
template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == PACK_T ? kPackMinB : MAXT == 256 ? 2 : 1) conv_kernel(const z_t* __restrict__ x1, const z_t* __restrict__ x2, int n,
                                                    int L, int mode, const z_t* __restrict__ tw, double2 scale,
                                                    z_t* out, long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  long long row;
  const RowGeom<E> g = row_geom<E>(L, n_rows, row);
  z_t* A = sm + 2 * g.sub * pidx(L);
  z_t* B = A + pidx(L);
  const long long o = row * n;
  z_t v[2][E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k = g.t + s * g.Q;
    v[0][s] = g.act && k < n ? x1[o + k] : make_double2(0.0, 0.0);
    // correlation: y[j] = x2[-j] placed circularly
    const int j = mode == 0 ? k : ((L - k) & (L - 1));
    v[1][s] = g.act && j < n ? x2[o + j] : make_double2(0.0, 0.0);
  }
  z_t* sAB[2] = {A, B};
  fft_rows<false, E, 2>(v, sAB, g, tw);
#pragma unroll
  for (int s = 0; s < E; ++s) v[0][s] = zmul(v[0][s], v[1][s]);
  z_t* sA[1] = {A};
  fft_rows<true, E, 1>(v, sA, g, tw);
  const z_t sc = zscale(1.0 / L, scale);
  if (g.act) {
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = g.t + s * g.Q;
      if (k < n) out[o + k] = zmul(sc, v[0][s]);
    }
  }
}

template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == PACK_T ? kPackMinB : MAXT == 256 ? 2 : 1) ret_kernel(const z_t* __restrict__ xl, const z_t* __restrict__ xg, int n,
                                                   int L, const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                                                   z_t* out, long long n_rows) {
  extern __shared__ __align__(16) z_t sm[];
  long long row;
  const RowGeom<E> g = row_geom<E>(L, n_rows, row);
  z_t* A = sm + 2 * g.sub * pidx(L);
  z_t* B = A + pidx(L);
  const long long o = row * n;
  z_t d[E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k = g.t + s * g.Q;
    d[s] = g.act && k < n ? zsub(xg[o + k], xl[o + k]) : make_double2(0.0, 0.0);
  }
  retarded_tail<E>(d, A, B, g, n, tw, kf, nullptr, out + o, nullptr);
}

// Elements per thread: 8. (E = 16 halves the exchanges of a 1024-point
// transform, but at ~250 registers it measured no faster for P and 20 %
// slower for Sigma on B200; the engine keeps both.)
int ept_for(int) { return 8; }
int threads_for(int L) { const int q = L / ept_for(L); return q >= PACK_T ? q : PACK_T; }

size_t smem_for(int L) { return (size_t)rows_per_cta(L, ept_for(L)) * 2 * (L + L / 8) * sizeof(z_t); }

unsigned grid_for(long long n_rows, int L) {
  const int r = rows_per_cta(L, ept_for(L));
  return (unsigned)((n_rows + r - 1) / r);
}

int smem_setup(const void* fn, int L) {
  if (smem_for(L) > 200 * 1024 || threads_for(L) > 512) return -5;
  NEGF_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  return 0;
}

bool pow2(int L) { return L >= 8 && (L & (L - 1)) == 0; }

constexpr int kMaxL1 = 4096;  // longest grid of the one-CTA engine; 2 kMaxL1 runs on a cluster pair
size_t smem_x2(int L) { return 2 * (size_t)((L / 2) + (L / 2) / 8) * sizeof(z_t); }
bool attr_x2(const void* fn, unsigned* done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32) return false;
  if (__atomic_load_n(done, __ATOMIC_ACQUIRE) & (1u << dev)) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x2(2 * kMaxL1)) != cudaSuccess)
    return false;
  __atomic_fetch_or(done, 1u << dev, __ATOMIC_RELEASE);
  return true;
}

}  // namespace
}  // namespace negf

using namespace negf;

extern "C" {

int negf_conv_polarization(long long n_rows, int n_e, int L, const void* gl, const void* gg,
                           const void* tw, const void* kf, const void* kcf,
                           const unsigned char* diag, double scale_re, double scale_im, void* pl,
                           void* pg, void* pr_up, void* pr_lo, void* stream) {
  if (n_rows < 0 || n_e < 1 || !pow2(L) || L < 2 * n_e - 1 || !gl || !gg || !tw || !kf || !kcf ||
      !pl || !pg)
    return -1;
  if (n_rows == 0) return 0;
  if (L == 2 * kMaxL1) {  // cluster pair of L/2-point engines
    static unsigned attr = 0;
    if (!attr_x2((const void*)pol_kernel_x2<8>, &attr)) return -5;
    ProfSpan ps_pol_kernel(PROF_CONV, (cudaStream_t)(stream), 0.0, 96.0 * (double)n_rows * n_e);
    pol_kernel_x2<8><<<(unsigned)(2 * n_rows), 512, smem_x2(L), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, n_e, L, (const z_t*)tw, (const z_t*)kf, (const z_t*)kcf, diag,
        make_double2(scale_re, scale_im), (z_t*)pl, (z_t*)pg, (z_t*)pr_up, (z_t*)pr_lo, n_rows);
    NEGF_LAUNCHED();
    return 0;
  }
  auto* kfn = threads_for(L) > 256 ? pol_kernel<8, 512> : threads_for(L) > PACK_T ? pol_kernel<8, 256> : pol_kernel<8, PACK_T>;
  int rc = smem_setup((const void*)kfn, L);
  if (rc) return rc;
  {
    // algorithmic HBM bytes: read G^<, G^> rows, write P^<, P^>, P^R_up, P^R_lo (96 B per entry-energy)
    ProfSpan ps_pol_kernel(PROF_CONV, (cudaStream_t)(stream), 0.0, 96.0 * (double)n_rows * n_e);
    kfn<<<grid_for(n_rows, L), threads_for(L), smem_for(L), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, n_e, L, (const z_t*)tw, (const z_t*)kf, (const z_t*)kcf, diag,
        make_double2(scale_re, scale_im), (z_t*)pl, (z_t*)pg, (z_t*)pr_up, (z_t*)pr_lo, n_rows);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_conv_sigma(long long n_rows, int n_e, int L, const void* gl, const void* gg,
                    const void* wl, const void* wg, const long long* w_rows, const void* tw,
                    const void* kf, const void* kcf, const unsigned char* diag, double scale_re,
                    double scale_im, void* sl, void* sg, void* sr_up, void* sr_lo, void* stream) {
  if (n_rows < 0 || n_e < 1 || !pow2(L) || L < 2 * n_e - 1 || !gl || !gg || !wl || !wg || !tw ||
      !kf || !kcf || !sl || !sg)
    return -1;
  if (n_rows == 0) return 0;
  if (L == 2 * kMaxL1) {
    static unsigned attr = 0;
    if (!attr_x2((const void*)sigma_kernel_x2<8>, &attr)) return -5;
    ProfSpan ps_sigma_kernel(PROF_CONV, (cudaStream_t)(stream), 0.0, 128.0 * (double)n_rows * n_e);
    sigma_kernel_x2<8><<<(unsigned)(2 * n_rows), 512, smem_x2(L), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, (const z_t*)wl, (const z_t*)wg, w_rows, n_e, L, (const z_t*)tw,
        (const z_t*)kf, (const z_t*)kcf, diag, make_double2(scale_re, scale_im), (z_t*)sl, (z_t*)sg,
        (z_t*)sr_up, (z_t*)sr_lo, n_rows);
    NEGF_LAUNCHED();
    return 0;
  }
  auto* kfn = threads_for(L) > 256 ? sigma_kernel<8, 512> : threads_for(L) > PACK_T ? sigma_kernel<8, 256> : sigma_kernel<8, PACK_T>;
  int rc = smem_setup((const void*)kfn, L);
  if (rc) return rc;
  {
    // read G^<, G^>, W^<, W^> rows, write four Sigma series (128 B per entry-energy)
    ProfSpan ps_sigma_kernel(PROF_CONV, (cudaStream_t)(stream), 0.0, 128.0 * (double)n_rows * n_e);
    kfn<<<grid_for(n_rows, L), threads_for(L), smem_for(L), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, (const z_t*)wl, (const z_t*)wg, w_rows, n_e, L, (const z_t*)tw,
        (const z_t*)kf, (const z_t*)kcf, diag, make_double2(scale_re, scale_im), (z_t*)sl, (z_t*)sg,
        (z_t*)sr_up, (z_t*)sr_lo, n_rows);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_convolve_energy(long long n_rows, int n_e, int L, const void* x1, const void* x2,
                         int mode, double scale_re, double scale_im, const void* tw, void* out,
                         void* stream) {
  if (n_rows < 0 || n_e < 1 || !pow2(L) || L < 2 * n_e - 1 || (mode != 0 && mode != 1) || !x1 ||
      !x2 || !tw || !out)
    return -1;
  if (n_rows == 0) return 0;
  auto* kfn = threads_for(L) > 256 ? conv_kernel<8, 512> : threads_for(L) > PACK_T ? conv_kernel<8, 256> : conv_kernel<8, PACK_T>;
  int rc = smem_setup((const void*)kfn, L);
  if (rc) return rc;
  {
    ProfScope ps_conv_kernel(PROF_OTHER, (cudaStream_t)(stream));
    kfn<<<grid_for(n_rows, L), threads_for(L), smem_for(L), (cudaStream_t)stream>>>(
        (const z_t*)x1, (const z_t*)x2, n_e, L, mode, (const z_t*)tw, make_double2(scale_re, scale_im),
        (z_t*)out, n_rows);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_retarded_from_lg(long long n_rows, int n_e, int L, const void* x_lesser,
                          const void* x_greater, const void* tw, const void* kf, void* out,
                          void* stream) {
  if (n_rows < 0 || n_e < 1 || !pow2(L) || L < 2 * n_e - 1 || !x_lesser || !x_greater || !tw ||
      !kf || !out)
    return -1;
  if (n_rows == 0) return 0;
  auto* kfn = threads_for(L) > 256 ? ret_kernel<8, 512> : threads_for(L) > PACK_T ? ret_kernel<8, 256> : ret_kernel<8, PACK_T>;
  int rc = smem_setup((const void*)kfn, L);
  if (rc) return rc;
  {
    ProfScope ps_ret_kernel(PROF_OTHER, (cudaStream_t)(stream));
    kfn<<<grid_for(n_rows, L), threads_for(L), smem_for(L), (cudaStream_t)stream>>>(
        (const z_t*)x_lesser, (const z_t*)x_greater, n_e, L, (const z_t*)tw, (const z_t*)kf, (z_t*)out, n_rows);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // extern "C"
