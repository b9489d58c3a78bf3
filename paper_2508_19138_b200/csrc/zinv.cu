#include <type_traits>
// Batched complex-FP64 block inversion with partial pivoting (sm_100a).
//
// Replaces negfgw/_linalg.py:30-52 `invert` (scipy lu_factor + lu_solve(I)):
// same pivoting rule as LAPACK zgetrf (max |re|+|im| in the column), same
// singularity rule (a pivot that is exactly zero or non-finite), and the
// same conditioning proxy u_spread = max|U_jj| / min|U_jj|.
//
// Algorithm: blocked in-place Gauss-Jordan sweeps. For a panel of NB columns
//   1. one CTA per matrix runs the unblocked pivoted LU of the (N-k0) x NB
//      panel in shared memory -> pivot rows, and Pinv = (pivot block)^-1;
//   2. a swap kernel applies the NB row interchanges to the whole matrix and
//      emits C' = A[:,K] (rows K zeroed) and R = A[K,:];
//   3. T = Pinv R                        (DMMA GEMM, M=NB, N=N, K=NB)
//   4. A[:, not K] -= C' T, A[:, K] = -C' Pinv   (one grouped DMMA launch)
//   5. rows K <- [T | Pinv]
// Every entry is produced by the textbook Gauss-Jordan formula (no
// cancellation-prone identity tricks), so the error matches LU-based inversion.
// which leaves inv(PA) after the last panel; a final kernel undoes the row
// permutation on the columns (LAPACK zgetri order) while copying to the
// destination. The O(N^3) work runs on the DMMA GEMM; the panel kernels are
// O(N^2 NB). Blocks with N <= 64 are inverted by one CTA entirely in smem.
#include "prof.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

namespace negf {

#define RC_(x) do { int _rc = (x); if (_rc) return _rc; } while (0)

namespace {

__device__ __forceinline__ void block_argmax(double v, int idx, double* sv, int* si, double& out_v,
                                             int& out_i) {
  // reduce (v, idx) to the max v; ties -> smallest idx (LAPACK izamax picks the first)
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, off);
    int oi = __shfl_down_sync(0xffffffffu, idx, off);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = v; si[warp] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) / 32;
    double bv = sv[0];
    int bi = si[0];
    for (int w = 1; w < nw; ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) { bv = sv[w]; bi = si[w]; }
    sv[0] = bv; si[0] = bi;
  }
  __syncthreads();
  out_v = sv[0];
  out_i = si[0];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Small path: whole matrix in smem, one CTA per matrix, Gauss-Jordan with
// partial pivoting (row interchanges, undone on the columns at the end).
__global__ void zinv_small_kernel(const z_t* __restrict__ S, long long sS, int lds, z_t* X,
                                  long long sX, int ldx, int n, InvAux aux) {
  extern __shared__ __align__(16) unsigned char raw[];
  const int ld = n + 1;  // odd stride: column walks spread over banks
  z_t* a = reinterpret_cast<z_t*>(raw);
  int* piv = reinterpret_cast<int*>(a + n * ld);
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ double umax, umin;
  __shared__ int bad;
  const int b = blockIdx.x;
  if (aux.active && !aux.active[b]) return;
  const z_t* src = S + (long long)b * sS;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) a[(e / n) * ld + e % n] = src[(long long)(e / n) * lds + e % n];
  if (threadIdx.x == 0) { umax = 0.0; umin = INFINITY; bad = 0; }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double v = -1.0;
    int idx = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      double c = zabs1(a[i * ld + k]);
      if (c != c) c = INFINITY;  // NaN -> treat as pivot candidate, flagged below
      if (c > v) { v = c; idx = i; }
    }
    double bv; int p;
    block_argmax(v, idx, sv, si, bv, p);
    if (threadIdx.x == 0) piv[k] = p;
    if (p != k)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        z_t t = a[k * ld + j]; a[k * ld + j] = a[p * ld + j]; a[p * ld + j] = t;
      }
    __syncthreads();
    const z_t pv = a[k * ld + k];
    if (threadIdx.x == 0) {
      double m = hypot(pv.x, pv.y);
      if (!(m > 0.0) || !isfinite(m)) bad = 1;
      umax = fmax(umax, m);
      umin = fmin(umin, m);
    }
    const z_t ip = zinv(pv);
    // scale pivot row (the pivot element itself becomes 1/pivot)
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      a[k * ld + j] = (j == k) ? ip : zmul(a[k * ld + j], ip);
    __syncthreads();
    // eliminate column k from all other rows
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      int i = e / n, j = e % n;
      if (i == k) continue;
      z_t f = a[i * ld + k];
      if (j == k) continue;
      a[i * ld + j] = zsub(a[i * ld + j], zmul(f, a[k * ld + j]));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i != k) a[i * ld + k] = zmul(zmake(-1.0, 0.0), zmul(a[i * ld + k], ip));
    __syncthreads();
  }
  // undo the row interchanges on the columns, last first
  if (threadIdx.x == 0) {
    int* perm = piv + n;
    for (int j = 0; j < n; ++j) perm[j] = j;
    for (int k = n - 1; k >= 0; --k) { int t = perm[k]; perm[k] = perm[piv[k]]; perm[piv[k]] = t; }
  }
  __syncthreads();
  const int* perm = piv + n;
  z_t* dst = X + (long long)b * sX;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    dst[(long long)i * ldx + j] = a[i * ld + perm[j]];
  }
  if (threadIdx.x == 0) {
    if (aux.u_spread) aux.u_spread[(long long)b * aux.spread_stride] = umax / umin;
    if (bad && aux.status) atomicCAS(aux.status + b, 0, aux.status_code);
  }
}

// ---------------------------------------------------------------------------
// Blocked path.
// Panel LU (candidate rows k0..n-1, columns k0..k0+NB-1) held in REGISTERS:
// TPR = NB/16 threads per row, 16 interleaved columns each (slot c of thread h = column c*TPR + h), so the rank-1 updates are
// register FMAs and a column step costs one block argmax (shuffles + barrier)
// and one pivot-row broadcast through smem (barrier). Rows are never moved:
// a pivoted row retires from the active set, and LAPACK's row order is
// tracked through each row's position (pos), which reproduces zgetf2's pivot
// choice including its first-index tie break. Outputs: the LAPACK-equivalent
// interchange sequence ipiv, the net row permutation as a move list, and
// Pinv = (pivot block)^-1 = U^-1 L^-1.
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

template <int NB>
__global__ void __launch_bounds__(512) zinv_panel_kernel(const z_t* __restrict__ A, long long sA,
                                                         z_t* __restrict__ Anew, long long sAn, int n,
                                                         int k0, int w,
                                                         int* ipiv, z_t* pinv, double* umaxmin,
                                                         int* map_src, int* map_dst, InvAux aux) {
  constexpr int TPR = NB / 16;  // threads per row
  constexpr int LD = NB + 1;
  __shared__ z_t prow_s[NB];          // pivot row broadcast
  __shared__ z_t ip_s;                // 1 / pivot
  __shared__ z_t blk[NB * LD];        // pivot rows (L\U) in pivot order, for Pinv
  __shared__ z_t pinv_s[NB * LD];     // Pinv
  __shared__ z_t rdiag_s[NB];         // 1 / U_kk
  __shared__ int posinv_s[1024];      // final position -> physical row
  __shared__ int piv_s[NB];           // pivot position chosen at each column
  __shared__ z_t pval_s[NB];          // pivot values
  __shared__ double rv[32];
  __shared__ int ri[32], rp[32];
  __shared__ int sbad;
  __shared__ double smax, smin;
  const int b = blockIdx.x;
  if (aux.active && !aux.active[b]) return;
  const int rows = n - k0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int r = tid / TPR, h = tid % TPR;  // my row, my 16-column half
  const bool have = r < rows;
  const z_t* a = A + (long long)b * sA;
  z_t v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c)
    v[c] = (have && c * TPR + h < w) ? a[(long long)(k0 + r) * n + k0 + c * TPR + h] : make_double2(0.0, 0.0);
  bool act = have;
  int pos = r;
  if (tid == 0) {
    sbad = 0;
    smax = k0 == 0 ? 0.0 : umaxmin[2 * b];
    smin = k0 == 0 ? INFINITY : umaxmin[2 * b + 1];
  }
#ifdef NEGF_EXP_TIMING
  long long clk0 = clock64();
#endif
  // Column loop: the register slot cj is a compile-time index (16 copies of
  // the column body, the TPR thread-columns of a slot in a rolled loop), so
  // v[cj] needs no select chain and the rank-1 update no per-slot predicates
  // (128 x 256^2 inverse 1.52 -> 1.36 ms). Unrolling all NB columns instead
  // overflows the instruction cache.
#ifdef NEGF_EXP_TIMING
  long long ph_a = 0, ph_b = 0, ph_c = 0, ph_d = 0, tq = clock64();
#define PH(x) do { long long _t = clock64(); x += _t - tq; tq = _t; } while (0)
#else
#define PH(x) do { } while (0)
#endif
  static_for<0, 16>([&](auto cjc) {
  constexpr int cj = decltype(cjc)::value;
#pragma unroll 1
  for (int hj = 0; hj < TPR; ++hj) {
    const int j = cj * TPR + hj;
    if (j >= w) break;
    const z_t vj = v[cj];
    // (1) argmax over active rows of |re|+|im| in column j; ties -> smallest
    // LAPACK position. Non-negative doubles order like their bit patterns, so
    // the warp stage is three REDUX ops (high word, low word, min position).
    double bv = 0.0;
    int bp = 0x7fffffff;
    if (act && h == hj) {
      double c = zabs1(vj);
      if (c != c) c = INFINITY;
      bv = c;
      bp = pos;
    }
    int br;
    {
      const unsigned long long key = __double_as_longlong(bv);
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      const bool best = hi == mhi && lo == mlo;
      const int mpos = (int)__reduce_min_sync(0xffffffffu, best ? (unsigned)bp : 0x7fffffffu);
      const unsigned who = __ballot_sync(0xffffffffu, best && bp == mpos);
      const int src = who ? __ffs(who) - 1 : 0;
      br = __shfl_sync(0xffffffffu, r, src);
      if (lane == 0) {
        rv[warp] = __longlong_as_double(((unsigned long long)mhi << 32) | mlo);
        ri[warp] = mpos == 0x7fffffff ? -1 : br;
        rp[warp] = mpos;
      }
    }
    PH(ph_a);
    __syncthreads();
    {  // cross-warp stage, redundantly in every warp (lanes < nw hold the entries)
      const double wv = lane < nw ? rv[lane] : 0.0;
      const int wp = lane < nw ? rp[lane] : 0x7fffffff;
      const int wr = lane < nw ? ri[lane] : -1;
      const unsigned long long key = __double_as_longlong(wv);
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      const bool best = hi == mhi && lo == mlo && wr >= 0;
      const int mpos = (int)__reduce_min_sync(0xffffffffu, best ? (unsigned)wp : 0x7fffffffu);
      const unsigned who = __ballot_sync(0xffffffffu, best && wp == mpos);
      const int src = who ? __ffs(who) - 1 : 0;
      br = __shfl_sync(0xffffffffu, wr, src);
      bp = mpos;
    }
    PH(ph_b);
    // (2) pivot row broadcast (+ its reciprocal pivot, computed once)
    if (act && r == br) {
#pragma unroll
      for (int c = 0; c < 16; ++c) prow_s[c * TPR + h] = v[c];
      if (h == hj) ip_s = zinv(vj);
    }
    __syncthreads();
    PH(ph_c);
    const z_t pv = prow_s[j];
    const z_t ipv = ip_s;
    // (3) multipliers and rank-1 update of the other active rows (registers)
    // column-j value of my row, from the thread holding it (all lanes shuffle)
    z_t own = vj;
    if (TPR > 1) {
      own.x = __shfl_sync(0xffffffffu, own.x, (lane & ~(TPR - 1)) | hj);
      own.y = __shfl_sync(0xffffffffu, own.y, (lane & ~(TPR - 1)) | hj);
    }
    if (act && r == br) {
      act = false;
      pos = j;
    } else if (act) {
      const z_t l = zmul(own, ipv);
      // slots below cj hold factored columns on every thread
      if (h > hj) v[cj] = zfms(l, prow_s[cj * TPR + h], v[cj]);
      else if (h == hj) v[cj] = l;
#pragma unroll
      for (int c = cj + 1; c < 16; ++c) v[c] = zfms(l, prow_s[c * TPR + h], v[c]);
      if (pos == j) pos = bp;  // LAPACK interchange: the row at position j moves to bp
    } else if (have && pos == j) {
      pos = bp;
    }
    // pivot bookkeeping (ipiv, |pivot| range, singular flag) after the loop,
    // off the column-to-column dependency chain
    if (tid == 0) {
      piv_s[j] = bp;
      pval_s[j] = pv;
    }
    PH(ph_d);
  }
  });
#undef PH
  __syncthreads();
  if (warp == 0) {  // ipiv, |pivot| range and singularity over the panel's w pivots
    double mx = 0.0, mn = INFINITY;
    int bad = 0;
    for (int q = lane; q < w; q += 32) {
      ipiv[(long long)b * n + k0 + q] = k0 + piv_s[q];
      const double m = hypot(pval_s[q].x, pval_s[q].y);
      if (!(m > 0.0) || !isfinite(m)) bad = 1;
      mx = fmax(mx, m);
      mn = fmin(mn, m);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
      mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      smax = fmax(smax, mx);
      smin = fmin(smin, mn);
      if (bad) sbad = 1;
    }
  }
#ifdef NEGF_EXP_TIMING
  __syncthreads();
  long long clk1 = clock64();
#endif
  // pivot rows -> blk (pivot order), positions -> posinv
  if (have) {
    posinv_s[pos] = r;
    if (pos < w) {
#pragma unroll
      for (int c = 0; c < 16; ++c) blk[pos * LD + c * TPR + h] = v[c];
    }
  }
  __syncthreads();
  // Pinv = U^-1 L^-1: warp-parallel substitutions, lane = row, one identity column per pass
  if (tid < w) rdiag_s[tid] = zinv(blk[tid * LD + tid]);
  __syncthreads();
  // Column c of L^-1 is zero above c, so its forward pass starts at k = c;
  // the second pass of each warp takes the mirrored column (w-1-warp) so every
  // warp runs the same number of steps.
  if (lane < 32) {
    for (int pass = 0, c0 = warp; c0 < w; ++pass, c0 += nw) {
      const int c = pass ? w - 1 - (c0 - nw) : c0;
      z_t y = zmake(lane == c ? 1.0 : 0.0, 0.0);
      for (int k = c; k < w; ++k) {
        const z_t yk = make_double2(__shfl_sync(0xffffffffu, y.x, k), __shfl_sync(0xffffffffu, y.y, k));
        if (lane > k && lane < w) y = zfms(blk[lane * LD + k], yk, y);
      }
      for (int k = w - 1; k >= 0; --k) {
        z_t xk = make_double2(__shfl_sync(0xffffffffu, y.x, k), __shfl_sync(0xffffffffu, y.y, k));
        xk = zmul(xk, rdiag_s[k]);
        if (lane == k) y = xk;
        if (lane < k) y = zfms(blk[lane * LD + k], xk, y);
      }
      if (lane < w) {
        pinv[(long long)b * w * w + lane * w + c] = y;
        pinv_s[lane * LD + c] = y;
      }
    }
  }
#ifdef NEGF_EXP_TIMING
  __syncthreads();
  long long clk2 = clock64();
#endif
  // Row maps of the sweep GEMM over the rows outside K (logical m < n - w):
  // destination row, and the A_old row that lands there after the panel's
  // interchanges (rows < k0 stay; rows >= k0 follow posinv).
  for (int m = tid; m < n - w; m += blockDim.x) {
    const int dst = m < k0 ? m : m + w;
    map_dst[(long long)b * n + m] = dst;
    map_src[(long long)b * n + m] = dst < k0 ? dst : k0 + posinv_s[dst - k0];
  }
  __syncthreads();
#ifdef NEGF_EXP_TIMING
  long long clk3 = clock64();
#endif
  // Rows K of A_new: [T | Pinv] with T = Pinv R, R = pivot rows of A_old.
  // One thread per (column j, block of TB output rows); R[q][j] streamed from
  // global (coalesced over j), Pinv broadcast from smem. TB = 8 keeps the
  // accumulators + loads in flight inside the 128-register budget of the
  // 512-thread CTA (16 rows spilled and ran 8x slower).
  z_t* an = Anew + (long long)b * sAn;
  {
    constexpr int TB = 8;
    const int tblocks = (w + TB - 1) / TB;
    for (int e = tid; e < tblocks * n; e += blockDim.x) {
      const int j = e % n, t0 = (e / n) * TB;
      const int t1 = t0 + TB < w ? t0 + TB : w;
      if (j >= k0 && j < k0 + w) {
        for (int t = t0; t < t1; ++t) an[(long long)(k0 + t) * n + j] = pinv_s[t * LD + (j - k0)];
        continue;
      }
      z_t acc[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int q0 = 0; q0 < w; q0 += 8) {
        z_t rq[8];  // 8 independent loads in flight
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          rq[qq] = q0 + qq < w ? a[(long long)(k0 + posinv_s[q0 + qq]) * n + j] : make_double2(0.0, 0.0);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
#pragma unroll
          for (int u = 0; u < TB; ++u)
            acc[u] = zfma(pinv_s[(t0 + u) * LD + q0 + qq], rq[qq], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < TB; ++u)
        if (t0 + u < t1) an[(long long)(k0 + t0 + u) * n + j] = acc[u];
    }
  }
#ifdef NEGF_EXP_TIMING
  __syncthreads();
  if (tid == 0 && b == 0 && k0 == 64)
    printf("PANELCLK cols %lld pinv %lld maps %lld T %lld | argmax-warp %lld cross %lld bcast %lld update %lld\n",
           clk1 - clk0, clk2 - clk1, clk3 - clk2, clock64() - clk3, ph_a, ph_b, ph_c, ph_d);
#endif
  if (tid == 0) {
    umaxmin[2 * b] = smax;
    umaxmin[2 * b + 1] = smin;
    if (sbad && aux.status) atomicCAS(aux.status + b, 0, aux.status_code);
  }
}

// X = inv(PA) P: the row interchanges are undone on the columns (LAPACK
// zgetri order: for k = n-1 .. 0 swap columns k <-> ipiv[k]). perm is built
// once per matrix (ipiv staged in smem), then a wide grid does the copy.
__global__ void zinv_perm_kernel(int n, const int* ipiv, const double* umaxmin, int* perm_out,
                                 InvAux aux) {
  extern __shared__ int sm_i[];
  int* pv = sm_i;
  int* perm = sm_i + n;
  const int b = blockIdx.x;
  if (aux.active && !aux.active[b]) return;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    pv[j] = ipiv[(long long)b * n + j];
    perm[j] = j;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = n - 1; k >= 0; --k) {
      const int r = pv[k];
      const int t = perm[k]; perm[k] = perm[r]; perm[r] = t;
    }
    if (aux.u_spread) aux.u_spread[(long long)b * aux.spread_stride] = umaxmin[2 * b] / umaxmin[2 * b + 1];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) perm_out[(long long)b * n + j] = perm[j];
}

// Rows are staged in smem, so A and X may be the same buffer.
__global__ void zinv_unpermute_kernel(const z_t* A, long long sA, int n, const int* perm_g, z_t* X,
                                      long long sX, int ldx, const int* active) {
  extern __shared__ __align__(16) unsigned char raw_u[];
  z_t* rows = reinterpret_cast<z_t*>(raw_u);           // 8 x n
  int* perm = reinterpret_cast<int*>(rows + 8 * n);
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  for (int j = threadIdx.x; j < n; j += blockDim.x) perm[j] = perm_g[(long long)b * n + j];
  const z_t* a = A + (long long)b * sA;
  z_t* x = X + (long long)b * sX;
  const int r0 = blockIdx.x * 8;
  for (int e = threadIdx.x; e < 8 * n; e += blockDim.x) {
    const int i = r0 + e / n;
    if (i < n) rows[e] = a[(long long)i * n + e % n];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 8 * n; e += blockDim.x) {
    const int i = r0 + e / n, j = e % n;
    if (i < n) x[(long long)i * ldx + j] = rows[(e / n) * n + perm[j]];
  }
}

// dst[b] (rows x cols, ld ldd) = src[b] (ld lds); batch strides sdst / ssrc
__global__ void copy_block_kernel(z_t* __restrict__ dst, long long sdst, int ldd, const z_t* __restrict__ src,
                                  long long ssrc, int lds, int rows, int cols) {
  const long long b = blockIdx.y;
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    dst[b * sdst + (long long)i * ldd + j] = src[b * ssrc + (long long)i * lds + j];
  }
}

int copy_block(z_t* dst, long long sdst, int ldd, const z_t* src, long long ssrc, int lds, int rows, int cols,
               int batch, cudaStream_t st) {
  long long total = (long long)rows * cols;
  int bx = (int)((total + 255) / 256);
  if (bx > 256) bx = 256;
  dim3 grid(bx, batch);
  ProfScope ps_(PROF_ZINV, st);
  copy_block_kernel<<<grid, 256, 0, st>>>(dst, sdst, ldd, src, ssrc, lds, rows, cols);
  NEGF_LAUNCHED();
  return 0;
}

__global__ void fill_nan_kernel(double* x, long long stride, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[(long long)i * stride] = __longlong_as_double(0x7ff8000000000000ll);
}

constexpr int kInvPanelMax = 512;  // one-CTA register panel limit

inline size_t a256z(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t zinv_workspace_bytes(int n, int batch) {
  if (n <= kInvSmallMax) return 0;
  if (n > kInvPanelMax) {  // 2x2 block recursion (zinv_recursive)
    const size_t h = n / 2, r = n - h, zb = sizeof(z_t) * (size_t)batch;
    const size_t sub_h = zinv_workspace_bytes((int)h, batch), sub_r = zinv_workspace_bytes((int)r, batch);
    return a256z(zb * h * h) * 2 + a256z(zb * r * h) * 2 + a256z(zb * r * r) * 2 + (sub_h > sub_r ? sub_h : sub_r);
  }
  const int nb = zinv_panel_width(n);
  size_t per = 4 * sizeof(int) * (size_t)n + sizeof(double) * 2 + sizeof(z_t) * (size_t)nb * nb;
  return per * batch + 256 * 8;
}

namespace {

// Blocks above the register-panel limit: 2x2 block inverse on packed halves,
//   [A B; C D]^-1 = [Ai + Ai B Si C Ai, -Ai B Si; -Si C Ai, Si],  Si = (D - C Ai B)^-1,
// each half inverted by the pivoted kernel (recursively). No pivoting across
// the halves: sound for the carrier Schur complements, whose anti-Hermitian
// part (eta - Im Sigma^R) is positive definite, so every leading block and
// its Schur complement are invertible with norm <= 1/eta. Singular halves
// are reported through aux.status; u_spread is not defined for this path
// (NaN).
int zinv_recursive(z_t* S, long long sS, z_t* X, long long sX, int n, int batch, InvAux aux, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  const int h = n / 2, r = n - h;
  const size_t zb = sizeof(z_t) * (size_t)batch;
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* q = w; w += a256z(bytes); return (z_t*)q; };
  z_t* Ap = take(zb * h * h);
  z_t* Ai = take(zb * h * h);
  z_t* T1 = take(zb * (size_t)r * h);  // C Ai
  z_t* T2 = take(zb * (size_t)h * r);  // Ai B
  z_t* Dp = take(zb * (size_t)r * r);
  z_t* Si = take(zb * (size_t)r * r);
  void* sub = w;
  const size_t sub_bytes = ws_bytes - (size_t)(w - reinterpret_cast<char*>(ws));
  InvAux sa = aux;
  sa.u_spread = nullptr;
  const long long hh = (long long)h * h, rh = (long long)r * h, rr = (long long)r * r;
  const z_t* A = S;
  const z_t* B = S + h;
  const z_t* C = S + (long long)h * n;
  const z_t* D = S + (long long)h * n + h;
  RC_(copy_block(Ap, hh, h, A, sS, n, h, h, batch, st));
  RC_(zinv_batched(Ap, hh, h, Ai, hh, h, h, batch, sa, sub, sub_bytes, st));
  auto desc = [&](const z_t* a, long long sa_, int lda, const z_t* b, long long sb, int ldb, int M, int N, int K,
                  z_t* d, long long sd, int ldd, double alpha, const z_t* c, long long sc, int ldc) {
    ZGemmDesc g = zdesc_default();
    g.M = M; g.N = N; g.batch = batch;
    g.t[0] = zterm(a, sa_, lda, OP_N, b, sb, ldb, OP_N, K);
    for (int i = 1; i < kMaxTerms; ++i) g.t[i] = g.t[0];
    g.alpha = make_double2(alpha, 0.0);
    if (c) { g.C = c; g.sC = sc; g.ldc = ldc; g.beta = make_double2(1.0, 0.0); }
    g.D = d; g.sD = sd; g.ldd = ldd;
    g.active = aux.active;
    return g;
  };
  {  // T1 = C Ai, T2 = Ai B
    ZGemmGroup g;
    g.n = 2;
    g.d[0] = desc(C, sS, n, Ai, hh, h, r, h, h, T1, rh, h, 1.0, nullptr, 0, 0);
    g.d[1] = desc(Ai, hh, h, B, sS, n, h, r, h, T2, rh, r, 1.0, nullptr, 0, 0);
    RC_(zgemm_group_launch(g, st));
  }
  // Dp = D - T1 B ; Si = Dp^-1
  RC_(zgemm_launch(desc(T1, rh, h, B, sS, n, r, r, h, Dp, rr, r, -1.0, D, sS, n), st));
  RC_(zinv_batched(Dp, rr, r, Si, rr, r, r, batch, sa, sub, sub_bytes, st));
  // X22 = Si ; X21 = -Si T1 ; X12 = -T2 Si
  RC_(copy_block(X + (long long)h * n + h, sX, n, Si, rr, r, r, r, batch, st));
  {
    ZGemmGroup g;
    g.n = 2;
    g.d[0] = desc(Si, rr, r, T1, rh, h, r, h, r, X + (long long)h * n, sX, n, -1.0, nullptr, 0, 0);
    g.d[1] = desc(T2, rh, r, Si, rr, r, h, r, r, X + h, sX, n, -1.0, nullptr, 0, 0);
    RC_(zgemm_group_launch(g, st));
  }
  // X11 = Ai - X12 T1
  RC_(zgemm_launch(desc(X + h, sX, n, T1, rh, h, h, h, r, X, sX, n, -1.0, Ai, hh, h), st));
  if (aux.u_spread) {
    fill_nan_kernel<<<(batch + 127) / 128, 128, 0, st>>>(aux.u_spread, aux.spread_stride, batch);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // namespace

int zinv_panel_width(int n) {
  // register panel: n * (nb/16) threads <= 512 per CTA
  if (n <= 256) return 32;
  return 16;
}

// Invert `batch` n x n matrices S (in place for the blocked path: S is
// overwritten) into X. Status/u_spread are reported through `aux`.
int zinv_batched(z_t* S, long long sS, int lds, z_t* X, long long sX, int ldx, int n, int batch,
                 InvAux aux, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (batch <= 0) return 0;
  if (n <= kInvSmallMax) {
    size_t smem = (size_t)n * (n + 1) * sizeof(z_t) + 2 * n * sizeof(int) + 16;
    static bool attr = false;
    if (!attr) {
      NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_small_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    ProfScope ps_(PROF_ZINV, stream);
    zinv_small_kernel<<<batch, 256, smem, stream>>>(S, sS, lds, X, sX, ldx, n, aux);
    NEGF_LAUNCHED();
    return 0;
  }
  if (lds != n || ldx != n) return -2;  // blocked path works on packed matrices
  const int nb = zinv_panel_width(n);
  if (ws_bytes < zinv_workspace_bytes(n, batch)) return -4;
  if (n > kInvPanelMax) return zinv_recursive(S, sS, X, sX, n, batch, aux, ws, ws_bytes, stream);
  // carve workspace
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = w; w += (bytes + 255) & ~size_t(255); return r; };
  int* ipiv = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  double* umm = reinterpret_cast<double*>(take(sizeof(double) * 2 * (size_t)batch));
  z_t* pinv = reinterpret_cast<z_t*>(take(sizeof(z_t) * (size_t)nb * nb * batch));
  int* map_src = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  int* map_dst = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  int* perm = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  const int panel_threads = ((n * (nb / 16) + 31) / 32) * 32;
  static bool attr_u = false;
  if (!attr_u) {
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_unpermute_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr_u = true;
  }
  // Gauss-Jordan sweeps ping-pong between S and X (X is the destination).
  z_t* cur = S;
  z_t* nxt = X;
  long long cs = sS, ns = sX;
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int wd = nb < n - k0 ? nb : n - k0;  // last panel may be narrower
    {
      ProfScope ps_(PROF_ZINV, stream);
      ProfScope psp_(5, stream);
      if (nb == 32)
        zinv_panel_kernel<32><<<batch, panel_threads, 0, stream>>>(cur, cs, nxt, ns, n, k0, wd, ipiv, pinv,
                                                                   umm, map_src, map_dst, aux);
      else
        zinv_panel_kernel<16><<<batch, panel_threads, 0, stream>>>(cur, cs, nxt, ns, n, k0, wd, ipiv, pinv,
                                                                   umm, map_src, map_dst, aux);
      NEGF_LAUNCHED();
    }
    if (n - wd > 0) {
      // rows outside K (row-mapped):  A_new[:, j not in K] = A_old - C' T,  A_new[:, K] = -C' Pinv,
      // with C' = A_old[src][K] and T = rows K of A_new (written by the panel kernel).
      ZGemmGroup grp;
      grp.n = 0;
      auto prob = [&](int c0, int nc, bool colK) {
        if (nc <= 0) return;
        ZGemmDesc& d = grp.d[grp.n++];
        d = zdesc_default();
        d.M = n - wd; d.N = nc; d.batch = batch; d.nterms = 1;
        if (!colK)
          d.t[0] = zterm(cur + k0, cs, n, OP_N, nxt + (long long)k0 * n + c0, ns, n, OP_N, wd);
        else
          d.t[0] = zterm(cur + k0, cs, n, OP_N, pinv, (long long)wd * wd, wd, OP_N, wd);
        d.t[1] = d.t[2] = d.t[3] = d.t[0];
        d.alpha = make_double2(-1.0, 0.0);
        d.beta = make_double2(colK ? 0.0 : 1.0, 0.0);
        d.C = colK ? nullptr : cur + c0; d.sC = cs; d.ldc = n;
        d.D = nxt + c0; d.sD = ns; d.ldd = n;
        d.active = aux.active;
        d.rowmap_a = map_src;
        d.rowmap_c = map_src;
        d.rowmap_d = map_dst;
        d.s_map = n;
      };
      prob(0, k0, false);
      prob(k0 + wd, n - k0 - wd, false);
      prob(k0, wd, true);
      int rc = zgemm_group_launch(grp, stream);
      if (rc) return rc;
    }
    z_t* t = cur; cur = nxt; nxt = t;
    long long ts = cs; cs = ns; ns = ts;
  }
  {
    ProfScope ps3_(PROF_ZINV, stream);
    ProfScope ps3b_(8, stream);
    zinv_perm_kernel<<<batch, 128, 2 * n * sizeof(int), stream>>>(n, ipiv, umm, perm, aux);
    NEGF_LAUNCHED();
    dim3 gu((n + 7) / 8, batch);
    zinv_unpermute_kernel<<<gu, 256, 8 * (size_t)n * sizeof(z_t) + n * sizeof(int), stream>>>(
        cur, cs, n, perm, X, sX, ldx, aux.active);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // namespace negf
