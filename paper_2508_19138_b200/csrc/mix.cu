// Self-energy mixing and the SCBA residual's trace reduction (scba.py:478-481,
// 1155-1167, _diag_traces :1251-1255), on the entry-major state.
#include "../../include/negf_b200.h"
#include "common.cuh"
#include "prof.cuh"

namespace negf {
namespace {

__global__ void mix_kernel(z_t* s0, z_t* s1, z_t* s2, z_t* s3, const z_t* r0, const z_t* r1,
                           const z_t* r2, const z_t* r3, long long n, double alpha) {
  const double beta = 1.0 - alpha;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    z_t* s[4] = {s0, s1, s2, s3};
    const z_t* r[4] = {r0, r1, r2, r3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!s[k]) continue;
      const z_t a = s[k][i], b = r[k][i];
      s[k][i] = make_double2(beta * a.x + alpha * b.x, beta * a.y + alpha * b.y);
    }
  }
}

// Mixing with the new Sigma read from its entry owners (fused nnz -> E):
// element (q, e) of the local (n_entries, n_own) state mixes with
// src[k][s][(q - row_start[s]) * ld + col0 + e] on rank s owning row q.
__global__ void mix_p2p_kernel(z_t* s0, z_t* s1, z_t* s2, z_t* s3, const unsigned long long* __restrict__ src,
                               int n_ranks, const long long* __restrict__ row_start, long long n_rows,
                               int n_own, long long ld, int col0, double alpha) {
  __shared__ long long rs[17];
  __shared__ unsigned long long sp[4][16];
  if (threadIdx.x <= n_ranks) rs[threadIdx.x] = row_start[threadIdx.x];
  if (threadIdx.x < 4 * n_ranks) sp[threadIdx.x / n_ranks][threadIdx.x % n_ranks] = src[threadIdx.x];
  __syncthreads();
  const double beta = 1.0 - alpha;
  const long long n = n_rows * n_own;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long q = i / n_own;
    const int e = (int)(i - q * n_own);
    int s = 0;
    while (s + 1 < n_ranks && q >= rs[s + 1]) ++s;
    const long long off = (q - rs[s]) * ld + col0 + e;
    z_t* st[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const z_t a = st[k][i], b = reinterpret_cast<const z_t*>(sp[k][s])[off];
      st[k][i] = make_double2(beta * a.x + alpha * b.x, beta * a.y + alpha * b.y);
    }
  }
}

// tr[b][e] = sum_{r < bs} x[idx[b*bs + r]][e]
__global__ void trace_kernel(const z_t* x, long long ld, int n_e, const long long* idx, int bs,
                             z_t* tr) {
  const int b = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_e) return;
  z_t s = make_double2(0.0, 0.0);
  for (int r = 0; r < bs; ++r) s = zadd(s, x[idx[(long long)b * bs + r] * ld + e]);
  tr[(long long)b * n_e + e] = s;
}

}  // namespace
}  // namespace negf

using namespace negf;

extern "C" {

int negf_mix(long long n, double alpha, void* s_lesser, void* s_greater, void* s_ret_up,
             void* s_ret_lo, const void* r_lesser, const void* r_greater, const void* r_ret_up,
             const void* r_ret_lo, void* stream) {
  if (n < 0) return -1;
  if (n == 0) return 0;
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  {
    ProfScope ps_mix_kernel(PROF_OTHER, (cudaStream_t)(stream));
    mix_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        (z_t*)s_lesser, (z_t*)s_greater, (z_t*)s_ret_up, (z_t*)s_ret_lo, (const z_t*)r_lesser,
        (const z_t*)r_greater, (const z_t*)r_ret_up, (const z_t*)r_ret_lo, n, alpha);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_mix_p2p(long long n_rows, int n_own, double alpha, void* s_lesser, void* s_greater, void* s_ret_up,
                 void* s_ret_lo, int n_ranks, const unsigned long long* src, const long long* row_start,
                 long long ld, int col0, void* stream) {
  if (n_rows < 0 || n_own < 0 || n_ranks < 1 || n_ranks > 16 || !src || !row_start || !s_lesser ||
      !s_greater || !s_ret_up || !s_ret_lo || col0 < 0 || ld < col0 + n_own)
    return -1;
  if (n_rows == 0 || n_own == 0) return 0;
  long long grid = (n_rows * n_own + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  {
    ProfScope ps_mix(PROF_OTHER, (cudaStream_t)(stream));
    mix_p2p_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
        (z_t*)s_lesser, (z_t*)s_greater, (z_t*)s_ret_up, (z_t*)s_ret_lo, src, n_ranks, row_start, n_rows, n_own,
        ld, col0, alpha);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_diag_traces(const void* x, long long ld, int n_e, const long long* diag_rows, int n_b,
                     int bs, void* tr, void* stream) {
  if (!x || !diag_rows || !tr || n_e < 0 || n_b < 1 || bs < 1) return -1;
  if (n_e == 0) return 0;
  dim3 grid((n_e + 127) / 128, n_b);
  {
    ProfScope ps_trace_kernel(PROF_OTHER, (cudaStream_t)(stream));
    trace_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>((const z_t*)x, ld, n_e, diag_rows, bs, (z_t*)tr);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // extern "C"
