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
// One CTA owns one entry row: the series live in shared memory (2 x L
// complex), forward transforms are in-place radix-2 decimation-in-frequency
// (natural -> bit-reversed), pointwise products happen in bit-reversed order,
// inverse transforms are decimation-in-time (bit-reversed -> natural), so no
// permutation pass is ever needed. Polarization uses
//   P^<_hat = G^<_hat * (-conj G^>_hat)   and   P^>[k] = conj(p^<[-k]),
// i.e. one inverse transform yields both P^< and P^>.
#include "../../include/negf_b200.h"
#include "common.cuh"
#include "prof.cuh"

namespace negf {
namespace {

__device__ __forceinline__ void fft_dif(z_t* x, int L, const z_t* __restrict__ tw) {
  for (int h = L >> 1, ts = 1; h >= 1; h >>= 1, ts <<= 1) {
    for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) {
      const int pos = j & (h - 1);
      const int i0 = ((j - pos) << 1) + pos, i1 = i0 + h;
      const z_t a = x[i0], b = x[i1];
      x[i0] = zadd(a, b);
      x[i1] = zmul(zsub(a, b), __ldg(&tw[pos * ts]));
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void fft_dif2(z_t* x, z_t* y, int L, const z_t* __restrict__ tw) {
  for (int h = L >> 1, ts = 1; h >= 1; h >>= 1, ts <<= 1) {
    for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) {
      const int pos = j & (h - 1);
      const int i0 = ((j - pos) << 1) + pos, i1 = i0 + h;
      const z_t w = __ldg(&tw[pos * ts]);
      z_t a = x[i0], b = x[i1];
      x[i0] = zadd(a, b);
      x[i1] = zmul(zsub(a, b), w);
      a = y[i0]; b = y[i1];
      y[i0] = zadd(a, b);
      y[i1] = zmul(zsub(a, b), w);
    }
    __syncthreads();
  }
}

// unscaled inverse: bit-reversed -> natural
__device__ __forceinline__ void ifft_dit2(z_t* x, z_t* y, int L, const z_t* __restrict__ tw) {
  for (int h = 1, ts = L >> 1; h < L; h <<= 1, ts >>= 1) {
    for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) {
      const int pos = j & (h - 1);
      const int i0 = ((j - pos) << 1) + pos, i1 = i0 + h;
      const z_t w = zconj(__ldg(&tw[pos * ts]));
      z_t a = x[i0], t = zmul(x[i1], w);
      x[i0] = zadd(a, t);
      x[i1] = zsub(a, t);
      if (y) {
        a = y[i0]; t = zmul(y[i1], w);
        y[i0] = zadd(a, t);
        y[i1] = zsub(a, t);
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ z_t proj(z_t v, bool diag) {
  // (v - conj v)/2 on diagonal entries (scba.py:406-409)
  return diag ? make_double2(0.0, v.y) : v;
}

// d = x^> - x^< (length n, zero padded in smem B) -> r_up = K*d, r_lo = -conj(conj(K)*d)
__device__ __forceinline__ void retarded_tail(z_t* A, z_t* B, int n, int L, const z_t* tw,
                                              const z_t* kf, const z_t* kcf, z_t* r_up, z_t* r_lo) {
  fft_dif(B, L, tw);
  for (int q = threadIdx.x; q < L; q += blockDim.x) {
    const z_t d = B[q];
    A[q] = zmul(d, __ldg(&kf[q]));
    B[q] = zmul(d, __ldg(&kcf[q]));
  }
  __syncthreads();
  ifft_dit2(A, B, L, tw);
  const double inv = 1.0 / L;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    if (r_up) r_up[k] = zscale(inv, A[k]);
    if (r_lo) r_lo[k] = zscale(-inv, zconj(B[k]));
  }
}

__global__ void pol_kernel(const z_t* __restrict__ gl, const z_t* __restrict__ gg, int n, int L,
                           const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                           const z_t* __restrict__ kcf, const unsigned char* __restrict__ diag,
                           double2 scale, z_t* pl, z_t* pg, z_t* pr_up, z_t* pr_lo) {
  extern __shared__ __align__(16) z_t sm[];
  z_t* A = sm;
  z_t* B = sm + L;
  const long long row = blockIdx.x;
  const long long o = row * n;
  const bool dg = diag && diag[row];
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    A[k] = k < n ? gl[o + k] : make_double2(0.0, 0.0);
    B[k] = k < n ? gg[o + k] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_dif2(A, B, L, tw);
  for (int q = threadIdx.x; q < L; q += blockDim.x) {
    const z_t b = B[q];
    A[q] = zmul(A[q], make_double2(-b.x, b.y));  // * (-conj b)
  }
  __syncthreads();
  ifft_dit2(A, nullptr, L, tw);
  const z_t s = zscale(1.0 / L, scale);
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    z_t d = make_double2(0.0, 0.0);
    if (k < n) {
      const z_t lo = proj(zmul(s, A[k]), dg);
      const z_t gr = proj(zmul(s, zconj(A[(L - k) & (L - 1)])), dg);
      pl[o + k] = lo;
      pg[o + k] = gr;
      d = zsub(gr, lo);
    }
    B[k] = d;
  }
  __syncthreads();
  retarded_tail(A, B, n, L, tw, kf, kcf, pr_up ? pr_up + o : nullptr, pr_lo ? pr_lo + o : nullptr);
}

__global__ void sigma_kernel(const z_t* __restrict__ gl, const z_t* __restrict__ gg,
                             const z_t* __restrict__ wl, const z_t* __restrict__ wg,
                             const long long* __restrict__ w_rows, int n, int L,
                             const z_t* __restrict__ tw, const z_t* __restrict__ kf,
                             const z_t* __restrict__ kcf, const unsigned char* __restrict__ diag,
                             double2 scale, z_t* sl, z_t* sg, z_t* sr_up, z_t* sr_lo) {
  extern __shared__ __align__(16) z_t sm[];
  z_t* A = sm;
  z_t* B = sm + L;
  const long long row = blockIdx.x;
  const long long o = row * n;
  const long long ow = (w_rows ? w_rows[row] : row) * n;
  const bool dg = diag && diag[row];
  const z_t s = zscale(1.0 / L, scale);
  for (int kind = 0; kind < 2; ++kind) {
    const z_t* g = kind ? gg : gl;
    const z_t* w = kind ? wg : wl;
    z_t* out = kind ? sg : sl;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      A[k] = k < n ? g[o + k] : make_double2(0.0, 0.0);
      B[k] = k < n ? w[ow + k] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    fft_dif2(A, B, L, tw);
    for (int q = threadIdx.x; q < L; q += blockDim.x) A[q] = zmul(A[q], B[q]);
    __syncthreads();
    ifft_dit2(A, nullptr, L, tw);
    for (int k = threadIdx.x; k < n; k += blockDim.x) out[o + k] = proj(zmul(s, A[k]), dg);
    __syncthreads();
  }
  // each thread re-reads only the values it wrote itself
  for (int k = threadIdx.x; k < L; k += blockDim.x)
    B[k] = k < n ? zsub(sg[o + k], sl[o + k]) : make_double2(0.0, 0.0);
  __syncthreads();
  retarded_tail(A, B, n, L, tw, kf, kcf, sr_up ? sr_up + o : nullptr, sr_lo ? sr_lo + o : nullptr);
}

// Generic convolve_energy (convolve.py:39-71): mode 0 convolution, 1 correlation.
__global__ void conv_kernel(const z_t* __restrict__ x1, const z_t* __restrict__ x2, int n, int L,
                            int mode, const z_t* __restrict__ tw, double2 scale, z_t* out) {
  extern __shared__ __align__(16) z_t sm[];
  z_t* A = sm;
  z_t* B = sm + L;
  const long long o = (long long)blockIdx.x * n;
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    A[k] = k < n ? x1[o + k] : make_double2(0.0, 0.0);
    // correlation: y[j] = x2[-j] placed circularly
    z_t v = make_double2(0.0, 0.0);
    if (mode == 0) {
      if (k < n) v = x2[o + k];
    } else {
      const int j = (L - k) & (L - 1);
      if (j < n) v = x2[o + j];
    }
    B[k] = v;
  }
  __syncthreads();
  fft_dif2(A, B, L, tw);
  for (int q = threadIdx.x; q < L; q += blockDim.x) A[q] = zmul(A[q], B[q]);
  __syncthreads();
  ifft_dit2(A, nullptr, L, tw);
  const z_t s = zscale(1.0 / L, scale);
  for (int k = threadIdx.x; k < n; k += blockDim.x) out[o + k] = zmul(s, A[k]);
}

__global__ void ret_kernel(const z_t* __restrict__ xl, const z_t* __restrict__ xg, int n, int L,
                           const z_t* __restrict__ tw, const z_t* __restrict__ kf, z_t* out) {
  extern __shared__ __align__(16) z_t sm[];
  z_t* A = sm;
  z_t* B = sm + L;
  const long long o = (long long)blockIdx.x * n;
  for (int k = threadIdx.x; k < L; k += blockDim.x)
    B[k] = k < n ? zsub(xg[o + k], xl[o + k]) : make_double2(0.0, 0.0);
  __syncthreads();
  retarded_tail(A, B, n, L, tw, kf, kf, out + o, nullptr);
}

int threads_for(int L) { return L >= 512 ? 256 : (L / 2 >= 32 ? L / 2 : 32); }

int smem_setup(const void* fn, int L) {
  size_t need = 2 * (size_t)L * sizeof(z_t);
  if (need > 200 * 1024) return -5;
  NEGF_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  return 0;
}

bool pow2(int L) { return L >= 2 && (L & (L - 1)) == 0; }

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
  int rc = smem_setup((const void*)pol_kernel, L);
  if (rc) return rc;
  {
    ProfScope ps_pol_kernel(PROF_OTHER, (cudaStream_t)(stream));
    pol_kernel<<<(unsigned)n_rows, threads_for(L), 2 * (size_t)L * sizeof(z_t), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, n_e, L, (const z_t*)tw, (const z_t*)kf, (const z_t*)kcf, diag,
        make_double2(scale_re, scale_im), (z_t*)pl, (z_t*)pg, (z_t*)pr_up, (z_t*)pr_lo);
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
  int rc = smem_setup((const void*)sigma_kernel, L);
  if (rc) return rc;
  {
    ProfScope ps_sigma_kernel(PROF_OTHER, (cudaStream_t)(stream));
    sigma_kernel<<<(unsigned)n_rows, threads_for(L), 2 * (size_t)L * sizeof(z_t), (cudaStream_t)stream>>>(
        (const z_t*)gl, (const z_t*)gg, (const z_t*)wl, (const z_t*)wg, w_rows, n_e, L, (const z_t*)tw,
        (const z_t*)kf, (const z_t*)kcf, diag, make_double2(scale_re, scale_im), (z_t*)sl, (z_t*)sg,
        (z_t*)sr_up, (z_t*)sr_lo);
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
  int rc = smem_setup((const void*)conv_kernel, L);
  if (rc) return rc;
  {
    ProfScope ps_conv_kernel(PROF_OTHER, (cudaStream_t)(stream));
    conv_kernel<<<(unsigned)n_rows, threads_for(L), 2 * (size_t)L * sizeof(z_t), (cudaStream_t)stream>>>(
        (const z_t*)x1, (const z_t*)x2, n_e, L, mode, (const z_t*)tw, make_double2(scale_re, scale_im),
        (z_t*)out);
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
  int rc = smem_setup((const void*)ret_kernel, L);
  if (rc) return rc;
  {
    ProfScope ps_ret_kernel(PROF_OTHER, (cudaStream_t)(stream));
    ret_kernel<<<(unsigned)n_rows, threads_for(L), 2 * (size_t)L * sizeof(z_t), (cudaStream_t)stream>>>(
        (const z_t*)x_lesser, (const z_t*)x_greater, n_e, L, (const z_t*)tw, (const z_t*)kf, (z_t*)out);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // extern "C"
