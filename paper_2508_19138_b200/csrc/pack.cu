// Energy-major blocks <-> entry-major series (the E <-> nnz layout switch).
//
// Reference: EntryPattern (convolve.py:135-187, compressed, bandwidth 3):
// for every block row bi, first the upper triangle (row-major, r <= c) of
// the diagonal block (bi, bi), then every entry of the upper block
// (bi, bi+1) row-major. _gather_entries (scba.py:252-271) packs one energy,
// _scatter_lg (scba.py:295-308) unpacks with the mirror rule
// X[c][r] = -conj X[r][c] on diagonal blocks, _scatter_retarded
// (scba.py:311-325) places the (row, col) value and the (col, row) value.
//
// Layout: entry-major arrays are row-major (n_entries, ld) with the energy
// window [e0, e0 + n_e) of the columns touched; blocks are
// [n_e][n_b][bs][bs] (diag) / [n_e][n_b-1][bs][bs] (upper, lower).
// Each CTA moves a 32-entry x 32-energy tile through shared memory so both
// the block side (entries contiguous) and the series side (energies
// contiguous) are read and written coalesced.
#include "../../include/negf_b200.h"
#include "common.cuh"
#include "prof.cuh"

namespace negf {
namespace {

constexpr int T = 32;

struct Pat {
  int n_b, bs;
  long long tri, per_row, n_entries;  // tri = bs(bs+1)/2, per_row = tri + bs^2
};

// Where entry t of the pattern lives in the block stacks: block row bi,
// kind (0 = diagonal block, 1 = upper block (bi, bi+1)) and flat offset q
// inside the block.
// LocStd: the reference's compressed bandwidth-3 EntryPattern on the stacks'
//   own blocking, computed from t (tri_q = row-major upper-triangle offsets).
// LocTab: any other pattern / blocking from per-entry tables -- a subset of
//   the band (the paper's r_cut nonzero set) or a coarser
//   target blocking (the W grid with bs_w = k bs, scba.py:893-937):
//   code[t] = 2 bi + kind, qt[t] = q.
struct LocStd {
  const int* __restrict__ tri_q;
  __device__ __forceinline__ void operator()(const struct Pat& p, long long t, int& bi, int& kind, int& q) const;
};
struct LocTab {
  const int* __restrict__ code;
  const int* __restrict__ qt;
  __device__ __forceinline__ void operator()(const struct Pat&, long long t, int& bi, int& kind, int& q) const {
    const int c = code[t];
    bi = c >> 1;
    kind = c & 1;
    q = qt[t];
  }
};
__device__ __forceinline__ void LocStd::operator()(const Pat& p, long long t, int& bi, int& kind, int& q) const {
  bi = (int)(t / p.per_row);
  const long long rem = t - (long long)bi * p.per_row;
  if (rem < p.tri) {
    kind = 0;
    q = tri_q[rem];
  } else {
    kind = 1;
    q = (int)(rem - p.tri);
  }
}

// blocks -> series
template <class Loc>
__global__ void pack_lg_kernel(Pat p, Loc locate, int n_e,
                               const z_t* __restrict__ xd, const z_t* __restrict__ xu, z_t* out,
                               long long ld, int e0) {
  __shared__ z_t tile[T][T + 1];
  const long long t0 = (long long)blockIdx.x * T;
  const int eb = blockIdx.y * T;
  const long long n2 = (long long)p.bs * p.bs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long t = t0 + tx;
  int bi = 0, kind = 0, q = 0;
  const bool ok = t < p.n_entries;
  if (ok) locate(p, t, bi, kind, q);
  for (int k = ty; k < T; k += 8) {
    const int e = eb + k;
    if (ok && e < n_e) {
      const z_t* src = kind == 0 ? xd + ((long long)e * p.n_b + bi) * n2
                                 : xu + ((long long)e * (p.n_b - 1) + bi) * n2;
      tile[k][tx] = src[q];
    }
  }
  __syncthreads();
  for (int k = ty; k < T; k += 8) {
    const long long tt = t0 + k;
    const int e = eb + tx;
    if (tt < p.n_entries && e < n_e) out[tt * ld + e0 + e] = tile[tx][k];
  }
}

// blocks -> series, fused with the E -> nnz redistribution: entry row tt
// belongs to rank s (row_start[s] <= tt < row_start[s+1]) and is written
// straight into that rank's entry-major array (peer memory over NVLink,
// ld = N_E columns, this rank's energies at column col0 + e). Each warp
// stores 32 consecutive energies of one row (512 B runs).
constexpr int kMaxRanks = 16;

__global__ void pack_lg_p2p_kernel(Pat p, const int* __restrict__ tri_q, int n_e,
                                   const z_t* __restrict__ xd, const z_t* __restrict__ xu, int n_ranks,
                                   const unsigned long long* __restrict__ dest,
                                   const long long* __restrict__ row_start, long long ld, int col0) {
  __shared__ z_t tile[T][T + 1];
  __shared__ long long rs[kMaxRanks + 1];
  __shared__ unsigned long long ds[kMaxRanks];
  const long long t0 = (long long)blockIdx.x * T;
  const int eb = blockIdx.y * T;
  const long long n2 = (long long)p.bs * p.bs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * T + tx;
  if (tid <= n_ranks) rs[tid] = row_start[tid];
  if (tid < n_ranks) ds[tid] = dest[tid];
  const long long t = t0 + tx;
  int bi = 0, kind = 0, q = 0;
  const bool ok = t < p.n_entries;
  if (ok) LocStd{tri_q}(p, t, bi, kind, q);
  for (int k = ty; k < T; k += 8) {
    const int e = eb + k;
    if (ok && e < n_e) {
      const z_t* src = kind == 0 ? xd + ((long long)e * p.n_b + bi) * n2
                                 : xu + ((long long)e * (p.n_b - 1) + bi) * n2;
      tile[k][tx] = src[q];
    }
  }
  __syncthreads();
  for (int k = ty; k < T; k += 8) {
    const long long tt = t0 + k;
    const int e = eb + tx;
    if (tt < p.n_entries && e < n_e) {
      int s = 0;
      while (s + 1 < n_ranks && tt >= rs[s + 1]) ++s;
      z_t* out = reinterpret_cast<z_t*>(ds[s]);
      out[(tt - rs[s]) * ld + col0 + e] = tile[tx][k];
    }
  }
}

// series -> blocks. mode 0: lg (mirror rule on diagonal blocks);
// mode 1: retarded (upper values at (r,c), lower values at (c,r)).
// Peer sources of the fused nnz -> E unpack: entry row tt lives on rank s
// (row_start[s] <= tt < row_start[s+1]) at row tt - row_start[s] of that
// rank's entry-major array(s).
struct PeerSrc {
  int n_ranks;
  const unsigned long long* up;  // device arrays of n_ranks pointers
  const unsigned long long* lo;
  const long long* row_start;
};

template <bool P2P, class Loc>
__global__ void unpack_kernel(Pat p, Loc locate, int n_e,
                              const z_t* __restrict__ in_up, const z_t* __restrict__ in_lo,
                              long long ld, int e0, int mode, z_t* xd, z_t* xu, z_t* xl, PeerSrc ps) {
  __shared__ z_t tu[T][T + 1];
  __shared__ z_t tl[T][T + 1];
  __shared__ long long rs[kMaxRanks + 1];
  __shared__ unsigned long long su[kMaxRanks], sl[kMaxRanks];
  const long long t0 = (long long)blockIdx.x * T;
  const int eb = blockIdx.y * T;
  const long long n2 = (long long)p.bs * p.bs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if constexpr (P2P) {
    const int tid = ty * T + tx;
    if (tid <= ps.n_ranks) rs[tid] = ps.row_start[tid];
    if (tid < ps.n_ranks) {
      su[tid] = ps.up[tid];
      sl[tid] = ps.lo ? ps.lo[tid] : 0ull;
    }
    __syncthreads();
  }
  for (int k = ty; k < T; k += 8) {
    const long long tt = t0 + k;
    const int e = eb + tx;
    if (tt < p.n_entries && e < n_e) {
      const z_t* up = in_up;
      const z_t* lo = in_lo;
      long long row = tt;
      if constexpr (P2P) {
        int s = 0;
        while (s + 1 < ps.n_ranks && tt >= rs[s + 1]) ++s;
        up = reinterpret_cast<const z_t*>(su[s]);
        lo = reinterpret_cast<const z_t*>(sl[s]);
        row = tt - rs[s];
      }
      tu[k][tx] = up[row * ld + e0 + e];
      if (mode == 1) tl[k][tx] = lo[row * ld + e0 + e];
    }
  }
  __syncthreads();
  const long long t = t0 + tx;
  if (t >= p.n_entries) return;
  int bi, kind, q;
  locate(p, t, bi, kind, q);
  const int r = q / p.bs, c = q % p.bs;
  const int qt = c * p.bs + r;
  for (int k = ty; k < T; k += 8) {
    const int e = eb + k;
    if (e >= n_e) continue;
    const z_t v = tu[tx][k];
    if (kind == 0) {
      z_t* d = xd + ((long long)e * p.n_b + bi) * n2;
      if (mode == 0) {
        d[q] = v;
        if (r != c) d[qt] = make_double2(-v.x, v.y);
      } else {
        const z_t w = tl[tx][k];
        if (r != c) d[q] = v;
        d[qt] = w;  // diagonal elements take the lower value (scba.py:319-321 write order)
      }
    } else {
      z_t* u = xu + ((long long)e * (p.n_b - 1) + bi) * n2;
      u[q] = v;
      if (mode == 1) {
        z_t* l = xl + ((long long)e * (p.n_b - 1) + bi) * n2;
        l[qt] = tl[tx][k];
      }
    }
  }
}

Pat make_pat(int n_b, int bs) {
  Pat p;
  p.n_b = n_b;
  p.bs = bs;
  p.tri = (long long)bs * (bs + 1) / 2;
  p.per_row = p.tri + (long long)bs * bs;
  p.n_entries = (long long)n_b * p.tri + (long long)(n_b - 1) * bs * bs;
  return p;
}

}  // namespace
}  // namespace negf

using namespace negf;

extern "C" {

long long negf_pattern_entries(int n_b, int bs) { return make_pat(n_b, bs).n_entries; }

int negf_pack_lg(int n_e, int n_b, int bs, const int* tri_q, const void* x_diag,
                 const void* x_upper, void* out, long long ld, int e0, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !tri_q || !x_diag || !out || e0 < 0 || ld < e0 + n_e) return -1;
  if (n_b > 1 && !x_upper) return -1;
  if (n_e == 0) return 0;
  Pat p = make_pat(n_b, bs);
  dim3 grid((unsigned)((p.n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    ProfSpan ps_pack_lg_kernel(PROF_LAYOUT, (cudaStream_t)(stream), 0.0, 32.0 * (double)p.n_entries * n_e);
    pack_lg_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(p, LocStd{tri_q}, n_e, (const z_t*)x_diag,
                                                             (const z_t*)x_upper, (z_t*)out, ld, e0);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_pack_lg_p2p(int n_e, int n_b, int bs, const int* tri_q, const void* x_diag, const void* x_upper,
                     int n_ranks, const unsigned long long* dest, const long long* row_start, long long ld,
                     int col0, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !tri_q || !x_diag || n_ranks < 1 || n_ranks > kMaxRanks || !dest ||
      !row_start || col0 < 0 || ld < col0 + n_e)
    return -1;
  if (n_b > 1 && !x_upper) return -1;
  if (n_e == 0) return 0;
  Pat p = make_pat(n_b, bs);
  dim3 grid((unsigned)((p.n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    ProfSpan ps_pack(PROF_LAYOUT, (cudaStream_t)(stream), 0.0, 32.0 * (double)p.n_entries * n_e);
    pack_lg_p2p_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(p, tri_q, n_e, (const z_t*)x_diag,
                                                                 (const z_t*)x_upper, n_ranks, dest, row_start,
                                                                 ld, col0);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_unpack_lg(int n_e, int n_b, int bs, const int* tri_q, const void* in, long long ld,
                   int e0, void* x_diag, void* x_upper, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !tri_q || !in || !x_diag || e0 < 0 || ld < e0 + n_e) return -1;
  if (n_b > 1 && !x_upper) return -1;
  if (n_e == 0) return 0;
  Pat p = make_pat(n_b, bs);
  dim3 grid((unsigned)((p.n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    const double blocks = (2.0 * n_b - 1.0) * bs * bs;  // diag + upper blocks written
    ProfSpan ps_unpack_kernel(PROF_LAYOUT, (cudaStream_t)(stream), 0.0, 16.0 * ((double)p.n_entries + blocks) * n_e);
    unpack_kernel<false><<<grid, block, 0, (cudaStream_t)stream>>>(p, LocStd{tri_q}, n_e, (const z_t*)in, nullptr, ld,
                                                                   e0, 0, (z_t*)x_diag, (z_t*)x_upper, nullptr,
                                                                   PeerSrc{});
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_unpack_retarded(int n_e, int n_b, int bs, const int* tri_q, const void* in_upper,
                         const void* in_lower, long long ld, int e0, void* x_diag, void* x_upper,
                         void* x_lower, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !tri_q || !in_upper || !in_lower || !x_diag || e0 < 0 ||
      ld < e0 + n_e)
    return -1;
  if (n_b > 1 && (!x_upper || !x_lower)) return -1;
  if (n_e == 0) return 0;
  Pat p = make_pat(n_b, bs);
  dim3 grid((unsigned)((p.n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    const double blocks = (3.0 * n_b - 2.0) * bs * bs;  // diag + upper + lower blocks written
    ProfSpan ps_unpack_kernel(PROF_LAYOUT, (cudaStream_t)(stream), 0.0,
                              16.0 * (2.0 * (double)p.n_entries + blocks) * n_e);
    unpack_kernel<false><<<grid, block, 0, (cudaStream_t)stream>>>(
        p, LocStd{tri_q}, n_e, (const z_t*)in_upper, (const z_t*)in_lower, ld, e0, 1, (z_t*)x_diag,
        (z_t*)x_upper, (z_t*)x_lower, PeerSrc{});
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_unpack_p2p(int n_e, int n_b, int bs, const int* tri_q, int retarded, int n_ranks,
                    const unsigned long long* src_upper, const unsigned long long* src_lower,
                    const long long* row_start, long long ld, int col0, void* x_diag, void* x_upper,
                    void* x_lower, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !tri_q || n_ranks < 1 || n_ranks > kMaxRanks || !src_upper ||
      !row_start || !x_diag || col0 < 0 || ld < col0 + n_e || (retarded && !src_lower))
    return -1;
  if (n_b > 1 && (!x_upper || (retarded && !x_lower))) return -1;
  if (n_e == 0) return 0;
  Pat p = make_pat(n_b, bs);
  dim3 grid((unsigned)((p.n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    const double blocks = (retarded ? 3.0 * n_b - 2.0 : 2.0 * n_b - 1.0) * bs * bs;
    ProfSpan ps_unpack(PROF_LAYOUT, (cudaStream_t)(stream), 0.0,
                       16.0 * ((retarded ? 2.0 : 1.0) * p.n_entries + blocks) * n_e);
    unpack_kernel<true><<<grid, block, 0, (cudaStream_t)stream>>>(
        p, LocStd{tri_q}, n_e, nullptr, nullptr, ld, col0, retarded ? 1 : 0, (z_t*)x_diag, (z_t*)x_upper,
        (z_t*)x_lower, PeerSrc{n_ranks, src_upper, retarded ? src_lower : nullptr, row_start});
    NEGF_LAUNCHED();
  }
  return 0;
}

/* Table-driven layout (LocTab above): n_entries pattern entries located in
 * block stacks of n_bt blocks of bs_t orbitals by code[t] = 2 bi + kind and
 * q[t]. zero_fill clears the target stacks first (patterns that do not cover
 * every stored block element). */
int negf_pack_lg_table(int n_e, long long n_entries, int n_bt, int bs_t, const int* code, const int* q,
                       const void* x_diag, const void* x_upper, void* out, long long ld, int e0, void* stream) {
  if (n_e < 0 || n_entries < 0 || n_bt < 1 || bs_t < 1 || !code || !q || !x_diag || !out || e0 < 0 ||
      ld < e0 + n_e)
    return -1;
  if (n_bt > 1 && !x_upper) return -1;
  if (n_e == 0 || n_entries == 0) return 0;
  Pat p = make_pat(n_bt, bs_t);
  p.n_entries = n_entries;
  dim3 grid((unsigned)((n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    ProfSpan ps_(PROF_LAYOUT, (cudaStream_t)(stream), 0.0, 32.0 * (double)n_entries * n_e);
    pack_lg_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(p, LocTab{code, q}, n_e, (const z_t*)x_diag,
                                                             (const z_t*)x_upper, (z_t*)out, ld, e0);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_unpack_table(int n_e, long long n_entries, int n_bt, int bs_t, const int* code, const int* q,
                      int retarded, const void* in_upper, const void* in_lower, long long ld, int e0,
                      void* x_diag, void* x_upper, void* x_lower, int zero_fill, void* stream) {
  if (n_e < 0 || n_entries < 0 || n_bt < 1 || bs_t < 1 || !code || !q || !in_upper || !x_diag || e0 < 0 ||
      ld < e0 + n_e || (retarded && !in_lower))
    return -1;
  if (n_bt > 1 && (!x_upper || (retarded && !x_lower))) return -1;
  if (n_e == 0) return 0;
  const size_t n2 = (size_t)bs_t * bs_t * sizeof(z_t);
  if (zero_fill) {
    NEGF_CUDA_CHECK(cudaMemsetAsync(x_diag, 0, n2 * n_bt * n_e, (cudaStream_t)stream));
    if (n_bt > 1) {
      NEGF_CUDA_CHECK(cudaMemsetAsync(x_upper, 0, n2 * (n_bt - 1) * n_e, (cudaStream_t)stream));
      if (retarded) NEGF_CUDA_CHECK(cudaMemsetAsync(x_lower, 0, n2 * (n_bt - 1) * n_e, (cudaStream_t)stream));
    }
  }
  if (n_entries == 0) return 0;
  Pat p = make_pat(n_bt, bs_t);
  p.n_entries = n_entries;
  dim3 grid((unsigned)((n_entries + T - 1) / T), (n_e + T - 1) / T), block(T, 8);
  {
    ProfSpan ps_(PROF_LAYOUT, (cudaStream_t)(stream), 0.0,
                 16.0 * ((retarded ? 2.0 : 1.0) * n_entries + (retarded ? 2.0 : 1.5) * n_entries) * n_e);
    unpack_kernel<false><<<grid, block, 0, (cudaStream_t)stream>>>(
        p, LocTab{code, q}, n_e, (const z_t*)in_upper, (const z_t*)in_lower, ld, e0, retarded ? 1 : 0,
        (z_t*)x_diag, (z_t*)x_upper, (z_t*)x_lower, PeerSrc{});
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // extern "C"
