#include <cstdlib>
#include <type_traits>
// Batched complex-FP64 block inversion with partial pivoting (sm_100a).
//
// Replaces negfgw/_linalg.py:30-52 `invert` (scipy lu_factor + lu_solve(I)):
// same pivoting rule as LAPACK zgetrf (max |re|+|im| in the column), same
// singularity rule (a pivot that is exactly zero or non-finite), and the
// same conditioning proxy u_spread = max|U_jj| / min|U_jj|.
//
// Algorithm: blocked Gauss-Jordan sweeps, ping-ponging between S and X. For
// each panel K of NB columns:
//   1. the panel kernel runs the unblocked pivoted LU of the (N-k0) x NB
//      panel with the pivot search over the whole remaining column (one CTA
//      per matrix for N <= 512; a thread-block cluster of up to 16 CTAs sharing
//      the candidates through distributed shared memory for 512 < N <= 4096),
//      and writes Pinv = (pivot block)^-1, the row maps of the interchanges,
//      and rows K of the new matrix: [T | Pinv] with T = Pinv R;
//   2. one row-mapped grouped DMMA launch updates every other row:
//      A[:, not K] -= C' T,  A[:, K] = -C' Pinv.
// This leaves inv(PA) after the last panel; a final kernel undoes the row
// permutation on the columns (LAPACK zgetri order) while copying to the
// destination. Every entry comes from the textbook Gauss-Jordan formula, so
// the error matches LU-based inversion. The O(N^3) work runs on the DMMA
// GEMM; the panel kernels are O(N^2 NB). Blocks with N <= 64 are inverted by
// one CTA entirely in smem.
#include "prof.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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
                                                         int* map_src, int* map_dst, InvAux aux,
                                                         int* prow) {
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
  if (prow) {  // fused sweep: hand over the pivot rows, T = Pinv R is formed there
    if (tid < w) prow[(long long)b * 32 + tid] = k0 + posinv_s[tid];
  } else {
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

// Panel LU for blocks above the one-CTA register panel (n > 512): the panel
// rows are split over a thread-block cluster of C <= 16 CTAs (RPC rows each,
// same register layout as zinv_panel_kernel), and the pivot search spans the
// WHOLE column (LAPACK zgetf2 order, first-index ties) through distributed
// shared memory. Per column: in-CTA argmax (one barrier), then every CTA
// writes its candidate (|pivot|, LAPACK position, row, the 16/32 panel values
// of that row and its reciprocal) into slot [parity][rank] of every CTA of
// the cluster, one cluster barrier, and every thread picks the winner from
// its local copy. Candidate slots are double-buffered by column parity: a
// slot is rewritten two columns later, after an intervening cluster barrier
// that every reader of the old contents has passed. Outputs are those of
// zinv_panel_kernel (ipiv, Pinv, row maps, rows K of A_new = [Pinv R | Pinv])
// with the T columns split over the cluster.
constexpr int kClusterMax = 16;  // 8 portable; 16 with the non-portable cluster attribute

template <int NB, int NT = 512>
__global__ void __launch_bounds__(NT) zinv_panel_cluster_kernel(const z_t* __restrict__ A, long long sA,
                                                                 z_t* __restrict__ Anew, long long sAn, int n,
                                                                 int k0, int w, int* ipiv, z_t* pinv,
                                                                 double* umaxmin, int* map_src, int* map_dst,
                                                                 InvAux aux) {
  constexpr int TPR = NB / 16;   // threads per row
  constexpr int RPC = NT / TPR;  // panel rows per CTA
  constexpr int LD = NB + 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  // the candidate rows are dead after the column loop: Pinv reuses their storage
  constexpr int kCand = 2 * kClusterMax * NB, kPinv = NB * LD;
  __shared__ z_t cand_pinv[kCand > kPinv ? kCand : kPinv];
  auto cand_row = reinterpret_cast<z_t(*)[kClusterMax][NB]>(cand_pinv);
  __shared__ z_t cand_ip[2][kClusterMax];
  __shared__ double cand_v[2][kClusterMax];
  __shared__ int cand_p[2][kClusterMax];
  __shared__ int cand_r[2][kClusterMax];
  __shared__ z_t blk[NB * LD];     // pivot rows (L\U) in pivot order
  z_t* const pinv_s = cand_pinv;  // after the column loop (see cand_pinv)
  __shared__ z_t rdiag_s[NB];
  __shared__ int prow_s[NB];       // panel row of the pivot chosen at column j
  __shared__ int piv_s[NB];
  __shared__ z_t pval_s[NB];
  __shared__ double rv[32];
  __shared__ int ri[32], rp[32];
  const int b = blockIdx.y;  // every CTA of a cluster has the same b
  if (aux.active && !aux.active[b]) return;
  const int rows = n - k0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int r = tid / TPR, h = tid % TPR;
  const int grow = q * RPC + r;  // panel row (0 = matrix row k0)
  const bool have = grow < rows;
  const z_t* a = A + (long long)b * sA;
  z_t v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c)
    v[c] = (have && c * TPR + h < w) ? a[(long long)(k0 + grow) * n + k0 + c * TPR + h] : make_double2(0.0, 0.0);
  bool act = have;
  int pos = grow;
  static_for<0, 16>([&](auto cjc) {
    constexpr int cj = decltype(cjc)::value;
#pragma unroll 1
    for (int hj = 0; hj < TPR; ++hj) {
      const int j = cj * TPR + hj;
      if (j >= w) break;
      const int par = j & 1;
      const z_t vj = v[cj];
      double bv = 0.0;
      int bp = 0x7fffffff;
      if (act && h == hj) {
        double c = zabs1(vj);
        if (c != c) c = INFINITY;
        bv = c;
        bp = pos;
      }
      {  // warp stage (same REDUX scheme as zinv_panel_kernel)
        const unsigned long long key = __double_as_longlong(bv);
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const bool best = hi == mhi && lo == mlo;
        const int mpos = (int)__reduce_min_sync(0xffffffffu, best ? (unsigned)bp : 0x7fffffffu);
        const unsigned who = __ballot_sync(0xffffffffu, best && bp == mpos);
        const int src = who ? __ffs(who) - 1 : 0;
        const int br = __shfl_sync(0xffffffffu, r, src);
        if (lane == 0) {
          rv[warp] = __longlong_as_double(((unsigned long long)mhi << 32) | mlo);
          ri[warp] = mpos == 0x7fffffff ? -1 : br;
          rp[warp] = mpos;
        }
      }
      __syncthreads();
      int br;
      double bval;
      {  // cross-warp stage -> this CTA's candidate
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
        bval = __longlong_as_double(((unsigned long long)mhi << 32) | mlo);
      }
      // publish the candidate to every CTA of the cluster
      if (br >= 0 && r == br) {
        const z_t ipv = zinv(vj);  // valid on the h == hj thread
        for (int d = 0; d < C; ++d) {
          z_t* row = cluster.map_shared_rank(&cand_row[par][q][0], d);
#pragma unroll
          for (int c = 0; c < 16; ++c) row[c * TPR + h] = v[c];
          if (h == hj) {
            *cluster.map_shared_rank(&cand_ip[par][q], d) = ipv;
            *cluster.map_shared_rank(&cand_v[par][q], d) = bval;
            *cluster.map_shared_rank(&cand_p[par][q], d) = bp;
            *cluster.map_shared_rank(&cand_r[par][q], d) = q * RPC + br;
          }
        }
      } else if (br < 0 && tid < C) {
        *cluster.map_shared_rank(&cand_r[par][q], tid) = -1;
      }
      cluster.sync();
      // winner over the cluster: max |pivot|, ties -> smallest LAPACK position
      int qw = -1;
      double wvv = -1.0;
      int wpp = 0x7fffffff;
      for (int d = 0; d < C; ++d) {
        if (cand_r[par][d] < 0) continue;
        const double cv = cand_v[par][d];
        const int cp = cand_p[par][d];
        if (qw < 0 || cv > wvv || (cv == wvv && cp < wpp)) { qw = d; wvv = cv; wpp = cp; }
      }
      const z_t* prow = &cand_row[par][qw][0];
      const z_t ipv = cand_ip[par][qw];
      const int wrow = cand_r[par][qw];
      bp = wpp;
      z_t own = vj;
      if (TPR > 1) {
        own.x = __shfl_sync(0xffffffffu, own.x, (lane & ~(TPR - 1)) | hj);
        own.y = __shfl_sync(0xffffffffu, own.y, (lane & ~(TPR - 1)) | hj);
      }
      if (act && grow == wrow) {
        act = false;
        pos = j;
      } else if (act) {
        const z_t l = zmul(own, ipv);
        if (h > hj) v[cj] = zfms(l, prow[cj * TPR + h], v[cj]);
        else if (h == hj) v[cj] = l;
#pragma unroll
        for (int c = cj + 1; c < 16; ++c) v[c] = zfms(l, prow[c * TPR + h], v[c]);
        if (pos == j) pos = bp;
      } else if (have && pos == j) {
        pos = bp;
      }
      if (tid < NB) blk[j * LD + tid] = prow[tid];
      if (tid == 0) {
        piv_s[j] = bp;
        pval_s[j] = prow[j];
        prow_s[j] = wrow;
      }
    }
  });
  __syncthreads();
  if (q == 0 && warp == 0) {  // ipiv, |pivot| range, singularity
    double mx = 0.0, mn = INFINITY;
    int bad = 0;
    for (int t = lane; t < w; t += 32) {
      ipiv[(long long)b * n + k0 + t] = k0 + piv_s[t];
      const double m = hypot(pval_s[t].x, pval_s[t].y);
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
      const double pmx = k0 == 0 ? 0.0 : umaxmin[2 * b], pmn = k0 == 0 ? INFINITY : umaxmin[2 * b + 1];
      umaxmin[2 * b] = fmax(pmx, mx);
      umaxmin[2 * b + 1] = fmin(pmn, mn);
      if (bad && aux.status) atomicCAS(aux.status + b, 0, aux.status_code);
    }
  }
  // row maps: rows above the panel stay, the non-pivot rows follow their final position
  if (have && pos >= w && h == 0) {
    map_src[(long long)b * n + k0 + pos - w] = k0 + grow;
  }
  for (int m = q * blockDim.x + tid; m < n - w; m += C * blockDim.x) {
    map_dst[(long long)b * n + m] = m < k0 ? m : m + w;
    if (m < k0) map_src[(long long)b * n + m] = m;
  }
  // Pinv = U^-1 L^-1 (every CTA, for its share of T)
  if (tid < w) rdiag_s[tid] = zinv(blk[tid * LD + tid]);
  __syncthreads();
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
      if (q == 0) pinv[(long long)b * w * w + lane * w + c] = y;
      pinv_s[lane * LD + c] = y;
    }
  }
  __syncthreads();
  // rows K of A_new = [T | Pinv], T = Pinv R; columns split over the cluster
  z_t* an = Anew + (long long)b * sAn;
  {
    constexpr int TB = 8;
    const int tblocks = (w + TB - 1) / TB;
    const int cols = (n + C - 1) / C, j0 = q * cols, j1 = j0 + cols < n ? j0 + cols : n;
    const int nc = j1 - j0;
    for (int e = tid; e < tblocks * nc; e += blockDim.x) {
      const int j = j0 + e % nc, t0 = (e / nc) * TB;
      const int t1 = t0 + TB < w ? t0 + TB : w;
      if (j >= k0 && j < k0 + w) {
        for (int t = t0; t < t1; ++t) an[(long long)(k0 + t) * n + j] = pinv_s[t * LD + (j - k0)];
        continue;
      }
      z_t acc[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int q0 = 0; q0 < w; q0 += 8) {
        z_t rq[8];
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          rq[qq] = q0 + qq < w ? a[(long long)(k0 + prow_s[q0 + qq]) * n + j] : make_double2(0.0, 0.0);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
#pragma unroll
          for (int u = 0; u < TB; ++u) acc[u] = zfma(pinv_s[(t0 + u) * LD + q0 + qq], rq[qq], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < TB; ++u)
        if (t0 + u < t1) an[(long long)(k0 + t0 + u) * n + j] = acc[u];
    }
  }
  // no CTA may exit while a peer can still write into its shared memory
  cluster.sync();
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
                                      long long sX, int ldx, const int* active, int R) {
  extern __shared__ __align__(16) unsigned char raw_u[];
  z_t* rows = reinterpret_cast<z_t*>(raw_u);           // R x n
  int* perm = reinterpret_cast<int*>(rows + (size_t)R * n);
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  for (int j = threadIdx.x; j < n; j += blockDim.x) perm[j] = perm_g[(long long)b * n + j];
  const z_t* a = A + (long long)b * sA;
  z_t* x = X + (long long)b * sX;
  const int r0 = blockIdx.x * R;
  for (int e = threadIdx.x; e < R * n; e += blockDim.x) {
    const int i = r0 + e / n;
    if (i < n) rows[e] = a[(long long)i * n + e % n];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * n; e += blockDim.x) {
    const int i = r0 + e / n, j = e % n;
    if (i < n) x[(long long)i * ldx + j] = rows[(e / n) * n + perm[j]];
  }
}

constexpr int kInvPanelMax = 512;   // one-CTA register panel limit
#ifndef NEGF_ZINV_FUSED_T
#define NEGF_ZINV_FUSED_T 1  // one-CTA panels leave T = Pinv R to the sweep (zinv_sweep_fused_kernel)
#endif
#ifndef NEGF_ZINV_FUSED_T_MAXB
#define NEGF_ZINV_FUSED_T_MAXB 64  // ... for batches up to this size
#endif
#ifndef NEGF_ZINV_SWEEP_MAX
// streamed sweep kernel (zgemm.cu zinv_sweep_kernel, 32-row CTAs) up to this block size, grouped
// row-mapped GEMMs above (experiments): 256 x 128 1.40 -> 1.24 ms, 512 x 8 1.83 -> 1.67 ms,
// 1024 x 8 7.70 -> 7.31 ms, 2048 x 8 38.4 -> 31.4 ms, 4096 x 1 53.3 -> 50.5 ms (profiles/zinv_sweep_r02.txt)
#define NEGF_ZINV_SWEEP_MAX 4096
#endif
#ifndef NEGF_ZINV_NT256_MAX
#define NEGF_ZINV_NT256_MAX 1024  // 256-thread cluster CTAs up to this block size (3-5% at 768-1024)
#endif
#ifndef NEGF_ZINV_NB32_MAX
#define NEGF_ZINV_NB32_MAX 4096  // cluster panels of 32 columns (256 rows per CTA, up to 16 CTAs: non-portable above 8)
#endif
constexpr int kInvClusterMax = 4096;  // cluster panel limit (16 CTAs x 256 rows)

// cudaFuncSetAttribute is per device context: remember it per device.
bool attr_once(const void* fn, int bytes, unsigned* done_mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32) return false;
  if (__atomic_load_n(done_mask, __ATOMIC_ACQUIRE) & (1u << dev)) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  __atomic_fetch_or(done_mask, 1u << dev, __ATOMIC_RELEASE);
  return true;
}

}  // namespace

size_t zinv_workspace_bytes(int n, int batch) {
  if (n <= kInvSmallMax) return 0;
  const int nb = zinv_panel_width(n, batch);
  size_t per = 4 * sizeof(int) * (size_t)n + sizeof(double) * 2 + sizeof(z_t) * (size_t)nb * nb + sizeof(int) * 32;
  return per * batch + 256 * 8;
}

// Which panel kernel a (n, batch) inverse uses. Above 512 only the cluster
// panel exists. For 256 < n <= 512 the cluster panel (32-column panels, 2 CTAs
// of 256 rows per matrix) halves the panel count and gives the sweeps K = 32,
// which wins once the batch fills the GPU (128 x 512^2: 9.4 vs 12.6 ms), while
// at 8-16 matrices its per-column cluster barrier costs more than it gains
// (2.0 vs 1.8 ms; profiles/zinv_cluster_r02.txt). NEGF_ZINV_CLUSTER_MIN=n
// forces the cluster panel for blocks >= n at any batch.
static int cluster_min() {
  static int v = [] {
    const char* e = getenv("NEGF_ZINV_CLUSTER_MIN");
    const int x = e ? atoi(e) : 0;
    return x > 256 ? x : kInvClusterMax + 1;
  }();
  return v;
}
constexpr int kClusterBatchMin = 64;
static bool use_cluster(int n, int batch) {
  return n > kInvPanelMax || (n > 256 && (batch >= kClusterBatchMin || n >= cluster_min()));
}

int zinv_panel_width(int n, int batch) {
  // one-CTA register panel: n * (nb/16) threads <= 512; cluster panel:
  // 512 * 16 / nb rows per CTA, <= kClusterMax CTAs
  if (n <= 256) return 32;
  if (!use_cluster(n, batch)) return 16;
  if (n <= NEGF_ZINV_NB32_MAX) return 32;
  return 16;
}

// Invert `batch` n x n matrices S (in place for the blocked path: S is
// overwritten) into X. Status/u_spread are reported through `aux`.
int zinv_batched(z_t* S, long long sS, int lds, z_t* X, long long sX, int ldx, int n, int batch,
                 InvAux aux, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (batch <= 0) return 0;
  if (n <= kInvSmallMax) {
    size_t smem = (size_t)n * (n + 1) * sizeof(z_t) + 2 * n * sizeof(int) + 16;
    static unsigned attr = 0;
    if (!attr_once((const void*)zinv_small_kernel, 200 * 1024, &attr)) return -6;
    ProfScope ps_(PROF_ZINV, stream);
    zinv_small_kernel<<<batch, 256, smem, stream>>>(S, sS, lds, X, sX, ldx, n, aux);
    NEGF_LAUNCHED();
    return 0;
  }
  if (lds != n || ldx != n) return -2;  // blocked path works on packed matrices
  const int nb = zinv_panel_width(n, batch);
  if (ws_bytes < zinv_workspace_bytes(n, batch)) return -4;
  if (n > kInvClusterMax) return -5;
  // carve workspace
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = w; w += (bytes + 255) & ~size_t(255); return r; };
  int* ipiv = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  double* umm = reinterpret_cast<double*>(take(sizeof(double) * 2 * (size_t)batch));
  z_t* pinv = reinterpret_cast<z_t*>(take(sizeof(z_t) * (size_t)nb * nb * batch));
  int* map_src = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  int* map_dst = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  int* perm = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  // pivot rows per panel for the fused sweep (one-CTA panels): T = Pinv R leaves the panel kernel.
  // Only while the one-CTA panels leave most SMs idle: 512 x 8 -10 %, 300 x 7 -13 %, but 256 x 128
  // (a panel CTA on most SMs already) +4 % (profiles/zinv_sweep_r02.txt)
  int* prow = (NEGF_ZINV_FUSED_T && batch <= NEGF_ZINV_FUSED_T_MAXB && !use_cluster(n, batch) &&
               n <= NEGF_ZINV_SWEEP_MAX)
                  ? reinterpret_cast<int*>(take(sizeof(int) * 32 * (size_t)batch))
                  : nullptr;
  const int panel_threads = ((n * (nb / 16) + 31) / 32) * 32;
  static unsigned attr_u = 0;
  if (!attr_once((const void*)zinv_unpermute_kernel, 160 * 1024, &attr_u)) return -6;
  // Gauss-Jordan sweeps ping-pong between S and X (X is the destination).
  z_t* cur = S;
  z_t* nxt = X;
  long long cs = sS, ns = sX;
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int wd = nb < n - k0 ? nb : n - k0;  // last panel may be narrower
    {
      ProfScope ps_(PROF_ZINV, stream);
      ProfScope psp_(5, stream);
      if (!use_cluster(n, batch)) {
        if (nb == 32)
          zinv_panel_kernel<32><<<batch, panel_threads, 0, stream>>>(cur, cs, nxt, ns, n, k0, wd, ipiv, pinv,
                                                                     umm, map_src, map_dst, aux, prow);
        else
          zinv_panel_kernel<16><<<batch, panel_threads, 0, stream>>>(cur, cs, nxt, ns, n, k0, wd, ipiv, pinv,
                                                                     umm, map_src, map_dst, aux, prow);
      } else {
        // 32-column panels: 256-thread CTAs (128 rows) while the cluster stays
        // within 16 CTAs for 512 < n <= NEGF_ZINV_NT256_MAX, else 512-thread CTAs (256 rows)
        const int nt = (nb == 32 && n > 512 && n <= NEGF_ZINV_NT256_MAX) ? 256 : 512;
        const int rpc = nt * 16 / nb;
        const int ncta = (n - k0 + rpc - 1) / rpc;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta, batch, 1);
        cfg.blockDim = dim3(nt, 1, 1);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ncta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (ncta > 8) {  // non-portable cluster size (B200: up to 16)
          static unsigned np_done = 0;
          int dv = 0;
          NEGF_CUDA_CHECK(cudaGetDevice(&dv));
          if (!(__atomic_load_n(&np_done, __ATOMIC_ACQUIRE) & (1u << dv))) {
            NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_panel_cluster_kernel<32>,
                                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_panel_cluster_kernel<32, 256>,
                                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_panel_cluster_kernel<16>,
                                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            __atomic_fetch_or(&np_done, 1u << dv, __ATOMIC_RELEASE);
          }
        }
        if (nb == 32 && nt == 256)
          NEGF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zinv_panel_cluster_kernel<32, 256>, (const z_t*)cur, cs, nxt,
                                             ns, n, k0, wd, ipiv, pinv, umm, map_src, map_dst, aux));
        else if (nb == 32)
          NEGF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zinv_panel_cluster_kernel<32>, (const z_t*)cur, cs, nxt, ns, n,
                                             k0, wd, ipiv, pinv, umm, map_src, map_dst, aux));
        else
          NEGF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zinv_panel_cluster_kernel<16>, (const z_t*)cur, cs, nxt, ns, n,
                                             k0, wd, ipiv, pinv, umm, map_src, map_dst, aux));
      }
      NEGF_LAUNCHED();
    }
    if (n - wd > 0 && n <= NEGF_ZINV_SWEEP_MAX) {
      // rows outside K (row-mapped):  A_new[:, j not in K] = A_old - C' T,  A_new[:, K] = -C' Pinv,
      // with C' = A_old[src][K] and T, Pinv = rows K of A_new (written by the panel kernel)
      SweepArgs sa;
      sa.cur = cur; sa.cs = cs; sa.nxt = nxt; sa.ns = ns;
      sa.n = n; sa.k0 = k0; sa.wd = wd;
      sa.map_src = map_src; sa.map_dst = map_dst; sa.active = aux.active; sa.ng = 1;
      sa.pinv = pinv; sa.prow = prow;
      const int rc = zinv_sweep_launch(sa, batch, stream);
      if (rc) return rc;
    } else if (n - wd > 0) {
      // the same sweep as grouped row-mapped GEMMs
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
    int R = (int)(144 * 1024 / ((size_t)n * sizeof(z_t)));
    R = R < 1 ? 1 : (R > 8 ? 8 : R);
    dim3 gu((n + R - 1) / R, batch);
    zinv_unpermute_kernel<<<gu, 256, (size_t)R * n * sizeof(z_t) + n * sizeof(int), stream>>>(
        cur, cs, n, perm, X, sX, ldx, aux.active, R);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // namespace negf
