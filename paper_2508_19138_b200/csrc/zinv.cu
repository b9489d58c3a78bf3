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
// Panel LU (rows k0..n-1, columns k0..k0+nb-1) in smem; writes pivots and Pinv.
__global__ void zinv_panel_kernel(const z_t* __restrict__ A, long long sA, int n, int k0, int nb,
                                  int* ipiv, z_t* pinv, double* umaxmin, InvAux aux) {
  extern __shared__ __align__(16) unsigned char raw[];
  const int rows = n - k0;
  const int ld = nb + 1;
  z_t* p = reinterpret_cast<z_t*>(raw);
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int sbad;
  __shared__ double smax, smin;
  const int b = blockIdx.x;
  if (aux.active && !aux.active[b]) return;
  const z_t* a = A + (long long)b * sA;
  for (int e = threadIdx.x; e < rows * nb; e += blockDim.x) {
    int i = e / nb, j = e % nb;
    p[i * ld + j] = a[(long long)(k0 + i) * n + k0 + j];
  }
  if (threadIdx.x == 0) {
    sbad = 0;
    smax = k0 == 0 ? 0.0 : umaxmin[2 * b];
    smin = k0 == 0 ? INFINITY : umaxmin[2 * b + 1];
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    double v = -1.0;
    int idx = rows;
    for (int i = j + threadIdx.x; i < rows; i += blockDim.x) {
      double c = zabs1(p[i * ld + j]);
      if (c != c) c = INFINITY;
      if (c > v) { v = c; idx = i; }
    }
    double bv; int pr;
    block_argmax(v, idx, sv, si, bv, pr);
    if (threadIdx.x == 0) ipiv[(long long)b * n + k0 + j] = k0 + pr;
    if (pr != j)
      for (int c = threadIdx.x; c < nb; c += blockDim.x) {
        z_t t = p[j * ld + c]; p[j * ld + c] = p[pr * ld + c]; p[pr * ld + c] = t;
      }
    __syncthreads();
    const z_t pv = p[j * ld + j];
    if (threadIdx.x == 0) {
      double m = hypot(pv.x, pv.y);
      if (!(m > 0.0) || !isfinite(m)) sbad = 1;
      smax = fmax(smax, m);
      smin = fmin(smin, m);
    }
    const z_t ip = zinv(pv);
    const int nr = rows - j - 1, nc = nb - j - 1;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      z_t* l = &p[(j + 1 + i) * ld + j];
      *l = zmul(*l, ip);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
      int i = j + 1 + e / nc, c = j + 1 + e % nc;
      p[i * ld + c] = zsub(p[i * ld + c], zmul(p[i * ld + j], p[j * ld + c]));
    }
    __syncthreads();
  }
  // Pinv = U^-1 L^-1 of the top nb x nb block; one thread per column of the identity.
  z_t* q = p + rows * ld;  // nb x nb scratch, ld
  for (int c = threadIdx.x; c < nb; c += blockDim.x) {
    // forward: L y = e_c (unit lower)
    for (int i = 0; i < nb; ++i) {
      z_t s = zmake(i == c ? 1.0 : 0.0, 0.0);
      for (int k = 0; k < i; ++k) s = zsub(s, zmul(p[i * ld + k], q[k * ld + c]));
      q[i * ld + c] = s;
    }
    // backward: U x = y
    for (int i = nb - 1; i >= 0; --i) {
      z_t s = q[i * ld + c];
      for (int k = i + 1; k < nb; ++k) s = zsub(s, zmul(p[i * ld + k], q[k * ld + c]));
      q[i * ld + c] = zmul(s, zinv(p[i * ld + i]));
    }
  }
  __syncthreads();
  z_t* pi = pinv + (long long)b * nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) pi[e] = q[(e / nb) * ld + e % nb];
  if (threadIdx.x == 0) {
    umaxmin[2 * b] = smax;
    umaxmin[2 * b + 1] = smin;
    if (sbad && aux.status) atomicCAS(aux.status + b, 0, aux.status_code);
  }
}

// Apply the panel's row interchanges to every column, and emit
// C' = A[:,K] with rows K zeroed   (n x nb)
// R  = A[K,:]                      (nb x n)
__global__ void zinv_swap_kernel(z_t* A, long long sA, int n, int k0, int nb, const int* ipiv,
                                 z_t* Cp, z_t* R, const int* active) {
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  z_t* a = A + (long long)b * sA;
  const int* pv = ipiv + (long long)b * n;
  if (col < n) {
    for (int j = 0; j < nb; ++j) {
      int r = pv[k0 + j];
      if (r != k0 + j) {
        z_t t = a[(long long)(k0 + j) * n + col];
        a[(long long)(k0 + j) * n + col] = a[(long long)r * n + col];
        a[(long long)r * n + col] = t;
      }
    }
    z_t* rr = R + (long long)b * nb * n;
    for (int j = 0; j < nb; ++j) rr[(long long)j * n + col] = a[(long long)(k0 + j) * n + col];
  }
  // The CTA owning columns K (k0 is a multiple of the 128-column tile when
  // nb divides 128; otherwise two CTAs share the range) copies the swapped
  // panel columns cooperatively, rows K zeroed.
  const int c0 = blockIdx.x * blockDim.x, c1 = c0 + blockDim.x;
  const int lo = k0 > c0 ? k0 : c0, hi = (k0 + nb) < c1 ? (k0 + nb) : c1;
  if (lo >= hi) return;
  __syncthreads();
  const int w = hi - lo;
  z_t* cp = Cp + (long long)b * n * nb;
  for (long long e = threadIdx.x; e < (long long)n * w; e += blockDim.x) {
    const int i = (int)(e / w), c = lo + (int)(e % w);
    cp[(long long)i * nb + (c - k0)] =
        (i >= k0 && i < k0 + nb) ? make_double2(0.0, 0.0) : a[(long long)i * n + c];
  }
}

// Rows K of the swept matrix: A[K, j] = T[:, j] (j not in K), A[K, K] = Pinv.
__global__ void zinv_rows_kernel(z_t* A, long long sA, int n, int k0, int nb, const z_t* T,
                                 long long sT, const z_t* pinv, const int* active) {
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  z_t* a = A + (long long)b * sA;
  const z_t* t = T + (long long)b * sT;
  const z_t* pi = pinv + (long long)b * nb * nb;
  const bool inK = col >= k0 && col < k0 + nb;
  for (int r = 0; r < nb; ++r)
    a[(long long)(k0 + r) * n + col] = inK ? pi[r * nb + col - k0] : t[(long long)r * n + col];
}

// X = inv(PA) P: undo the interchanges on the columns while copying out.
__global__ void zinv_unpermute_kernel(const z_t* __restrict__ A, long long sA, int n,
                                      const int* ipiv, const double* umaxmin, z_t* X,
                                      long long sX, int ldx, InvAux aux) {
  extern __shared__ int perm[];
  const int b = blockIdx.x;
  if (aux.active && !aux.active[b]) return;
  const int* pv = ipiv + (long long)b * n;
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) perm[j] = j;
    for (int k = n - 1; k >= 0; --k) {
      int r = pv[k];
      int t = perm[k]; perm[k] = perm[r]; perm[r] = t;
    }
    if (aux.u_spread) aux.u_spread[(long long)b * aux.spread_stride] = umaxmin[2 * b] / umaxmin[2 * b + 1];
  }
  __syncthreads();
  const z_t* a = A + (long long)b * sA;
  z_t* x = X + (long long)b * sX;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    int i = (int)(e / n), j = (int)(e % n);
    x[(long long)i * ldx + j] = a[(long long)i * n + perm[j]];
  }
}

}  // namespace

size_t zinv_workspace_bytes(int n, int batch) {
  if (n <= kInvSmallMax) return 0;
  const int nb = zinv_panel_width(n);
  size_t per = sizeof(int) * n + sizeof(double) * 2 + sizeof(z_t) * ((size_t)nb * nb + 2 * (size_t)n * nb);
  return (per * batch + 1024) + 256 * 4;
}

int zinv_panel_width(int n) {
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
  if (lds != n) return -2;  // blocked path works on packed scratch
  const int nb = zinv_panel_width(n);
  if (ws_bytes < zinv_workspace_bytes(n, batch)) return -4;
  // carve workspace
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = w; w += (bytes + 255) & ~size_t(255); return r; };
  int* ipiv = reinterpret_cast<int*>(take(sizeof(int) * (size_t)n * batch));
  double* umm = reinterpret_cast<double*>(take(sizeof(double) * 2 * (size_t)batch));
  z_t* pinv = reinterpret_cast<z_t*>(take(sizeof(z_t) * (size_t)nb * nb * batch));
  z_t* Cp = reinterpret_cast<z_t*>(take(sizeof(z_t) * (size_t)n * nb * batch));
  z_t* R = reinterpret_cast<z_t*>(take(sizeof(z_t) * (size_t)n * nb * batch));
  size_t panel_smem = (size_t)(n + nb) * (nb + 1) * sizeof(z_t);
  static bool attr2 = false;
  if (!attr2) {
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_panel_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr2 = true;
  }
  if (panel_smem > 220 * 1024) return -5;
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int w = nb < n - k0 ? nb : n - k0;  // last panel may be narrower
    dim3 g((n + 127) / 128, batch);
    {
    ProfScope ps_(PROF_ZINV, stream);
    zinv_panel_kernel<<<batch, 256, panel_smem, stream>>>(S, sS, n, k0, w, ipiv, pinv, umm, aux);
    NEGF_LAUNCHED();
    zinv_swap_kernel<<<g, 128, 0, stream>>>(S, sS, n, k0, w, ipiv, Cp, R, aux.active);
    NEGF_LAUNCHED();
    }
    // T = Pinv R, staged in the caller's destination X (w x n per matrix;
    // X is only written for real by the final unpermute kernel).
    ZGemmGroup grp;
    grp.n = 1;
    z_t* T = X;
    {
      ZGemmDesc& d = grp.d[0];
      d.M = w; d.N = n; d.batch = batch; d.nterms = 1;
      d.t[0] = zterm(pinv, (long long)w * w, w, OP_N, R, (long long)w * n, n, OP_N, w);
      d.t[1] = d.t[0];
      d.alpha = make_double2(1.0, 0.0); d.beta = make_double2(0.0, 0.0);
      d.C = nullptr; d.sC = 0; d.ldc = 0;
      d.D = T; d.sD = sX; d.ldd = n; d.transD = 0;
      d.active = aux.active;
    }
    int rc = zgemm_group_launch(grp, stream);
    if (rc) return rc;
    // Gauss-Jordan sweep, one grouped launch over disjoint column ranges:
    //   A[:, j] -= C' T[:, j]   (j left / right of K)      A[:, K] = -C' Pinv
    grp.n = 0;
    auto upd = [&](int c0, int nc) {
      if (nc <= 0) return;
      ZGemmDesc& d = grp.d[grp.n++];
      d.M = n; d.N = nc; d.batch = batch; d.nterms = 1;
      d.t[0] = zterm(Cp, (long long)n * w, w, OP_N, T + c0, sX, n, OP_N, w);
      d.t[1] = d.t[0];
      d.alpha = make_double2(-1.0, 0.0); d.beta = make_double2(1.0, 0.0);
      d.C = S + c0; d.sC = sS; d.ldc = n;
      d.D = S + c0; d.sD = sS; d.ldd = n; d.transD = 0;
      d.active = aux.active;
    };
    upd(0, k0);
    upd(k0 + w, n - k0 - w);
    {
      ZGemmDesc& d = grp.d[grp.n++];
      d.M = n; d.N = w; d.batch = batch; d.nterms = 1;
      d.t[0] = zterm(Cp, (long long)n * w, w, OP_N, pinv, (long long)w * w, w, OP_N, w);
      d.t[1] = d.t[0];
      d.alpha = make_double2(-1.0, 0.0); d.beta = make_double2(0.0, 0.0);
      d.C = nullptr; d.sC = 0; d.ldc = 0;
      d.D = S + k0; d.sD = sS; d.ldd = n; d.transD = 0;
      d.active = aux.active;
    }
    rc = zgemm_group_launch(grp, stream);
    if (rc) return rc;
    ProfScope ps2_(PROF_ZINV, stream);
    zinv_rows_kernel<<<g, 128, 0, stream>>>(S, sS, n, k0, w, T, sX, pinv, aux.active);
    NEGF_LAUNCHED();
  }
  ProfScope ps3_(PROF_ZINV, stream);
  zinv_unpermute_kernel<<<batch, 256, n * sizeof(int), stream>>>(S, sS, n, ipiv, umm, X, sX, ldx,
                                                                 aux);
  NEGF_LAUNCHED();
  return 0;
}

}  // namespace negf
