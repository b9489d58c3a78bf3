// Observables reduced on the device per energy (scba.py:1313-1376):
//   dos               -Im tr G^R_bb / pi               (per energy, block)
//   electron_density  tr G^<_bb                        (summed over energies on host)
//   current_spectrum  2 Re sum_ij H_{b,b+1}[i,j] G^<_{b+1,b}[j,i]  * C_OBS
//                     with G^<_{b+1,b} = -G^<_{b,b+1}^dag (lg symmetry)
//   terminal_current  tr(S^<_c G^>_cc) - tr(S^>_c G^<_cc) at each contact corner c
// Only these O(n_e n_b) numbers leave the device: the reference instead
// replicates every G block of every energy to every rank (scba.py:1258-1308).
#include "../../include/negf_b200.h"
#include "common.cuh"
#include "prof.cuh"

namespace negf {
namespace {

__device__ z_t block_zsum(z_t v, z_t* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  z_t s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) s = zadd(s, red[i]);
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

__global__ void observables_kernel(int n_b, int bs, const z_t* gr, const z_t* gl, const z_t* gg,
                                   const z_t* gl_up, const z_t* h_up, const z_t* sl_l,
                                   const z_t* sg_l, const z_t* sl_r, const z_t* sg_r, z_t* tr_gr,
                                   z_t* tr_gl, double* cur, z_t* term) {
  __shared__ z_t red[32];
  const int b = blockIdx.x, e = blockIdx.y;
  const long long n2 = (long long)bs * bs;
  const long long od = ((long long)e * n_b + b) * n2;
  z_t a = make_double2(0.0, 0.0), c = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < bs; i += blockDim.x) {
    a = zadd(a, gr[od + (long long)i * bs + i]);
    if (gl) c = zadd(c, gl[od + (long long)i * bs + i]);
  }
  a = block_zsum(a, red);
  c = block_zsum(c, red);
  if (threadIdx.x == 0) {
    tr_gr[(long long)e * n_b + b] = a;
    if (tr_gl) tr_gl[(long long)e * n_b + b] = c;
  }
  if (cur && gl_up && b < n_b - 1) {
    const long long oo = ((long long)e * (n_b - 1) + b) * n2;
    z_t s = make_double2(0.0, 0.0);
    for (long long q = threadIdx.x; q < n2; q += blockDim.x)
      s = zsub(s, zmul(h_up[(long long)b * n2 + q], zconj(gl_up[oo + q])));
    s = block_zsum(s, red);
    if (threadIdx.x == 0) cur[(long long)e * (n_b - 1) + b] = 2.0 * s.x * 0.15915494309189535;
  }
  if (term && gl && gg && (b == 0 || b == n_b - 1)) {
    const z_t* sl = b == 0 ? sl_l : sl_r;
    const z_t* sg = b == 0 ? sg_l : sg_r;
    const long long oc = (long long)e * n2;
    z_t s = make_double2(0.0, 0.0);
    for (long long q = threadIdx.x; q < n2; q += blockDim.x) {
      const int i = (int)(q / bs), j = (int)(q % bs);
      const long long t = od + (long long)j * bs + i;
      s = zadd(s, zsub(zmul(sl[oc + q], gg[t]), zmul(sg[oc + q], gl[t])));
    }
    s = block_zsum(s, red);
    if (threadIdx.x == 0) term[(long long)e * 2 + (b == 0 ? 0 : 1)] = s;
  }
}

// max |v| over the block into out (as the bit pattern of a non-negative double)
__device__ void block_max_to(double v, unsigned long long* out, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;  // 1-D or 2-D blocks of whole warps
  const int lane = tid & 31, w = tid >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (int)(blockDim.x * blockDim.y + 31) / 32; ++i) m = fmax(m, red[i]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
  __syncthreads();
}

// G identity defect (scba.py:1223-1238): max |X^> - X^< - (X^R - X^R^dag)| over
// the diagonal blocks and |X^>_up - X^<_up - (X^R_up - X^R_lo^dag)| over the
// upper blocks, and max |X^R - X^R^dag| (resp. |X^R_up - X^R_lo^dag|) as the
// scale. grid (blocks of tiles, n_e * (2 n_b - 1)); one 32x32 tile per CTA.
__global__ void g_defect_kernel(int n_b, int bs, const z_t* rd, const z_t* ru, const z_t* rl, const z_t* ld,
                                const z_t* lu, const z_t* gd, const z_t* gu, unsigned long long* out) {
  __shared__ z_t tt[32][33];
  __shared__ double red[32];
  const int nblk = 2 * n_b - 1;
  const int e = blockIdx.y / nblk, q = blockIdx.y % nblk;
  const bool diag = q < n_b;
  const int i = diag ? q : q - n_b;
  const long long n2 = (long long)bs * bs;
  const long long od = ((long long)e * n_b + i) * n2, oo = ((long long)e * (n_b - 1) + i) * n2;
  const z_t* R = diag ? rd + od : ru + oo;
  const z_t* RH = diag ? rd + od : rl + oo;  // block whose dagger is subtracted
  const z_t* L = diag ? ld + od : lu + oo;
  const z_t* G = diag ? gd + od : gu + oo;
  const int tiles_c = (bs + 31) / 32;
  const int r0 = (blockIdx.x / tiles_c) * 32, c0 = (blockIdx.x % tiles_c) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int rr = c0 + k, cc = r0 + tx;
    if (rr < bs && cc < bs) tt[k][tx] = RH[(long long)rr * bs + cc];
  }
  __syncthreads();
  double dmax = 0.0, smax = 0.0;
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;
    if (r >= bs || c >= bs) continue;
    const long long x = (long long)r * bs + c;
    const z_t gam = zsub(R[x], zconj(tt[tx][k]));
    const z_t diff = zsub(G[x], L[x]);
    dmax = fmax(dmax, hypot(diff.x - gam.x, diff.y - gam.y));
    smax = fmax(smax, hypot(gam.x, gam.y));
  }
  block_max_to(dmax, out, red);
  block_max_to(smax, out + 1, red);
}

// entry-major defect (scba.py:1241-1248): max |(g - l) - (ru - conj rl)|, max |ru - conj rl|
__global__ void entry_defect_kernel(long long n, const z_t* l, const z_t* g, const z_t* ru, const z_t* rl,
                                    unsigned long long* out) {
  __shared__ double red[32];
  double dmax = 0.0, smax = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const z_t gam = zsub(ru[k], zconj(rl[k]));
    const z_t diff = zsub(g[k], l[k]);
    dmax = fmax(dmax, hypot(diff.x - gam.x, diff.y - gam.y));
    smax = fmax(smax, hypot(gam.x, gam.y));
  }
  block_max_to(dmax, out, red);
  block_max_to(smax, out + 1, red);
}

}  // namespace
}  // namespace negf

using namespace negf;

extern "C" int negf_observables(int n_e, int n_b, int bs, const void* gr_diag,
                                const void* gl_diag, const void* gg_diag, const void* gl_upper,
                                const void* h_upper, const void* sl_left, const void* sg_left,
                                const void* sl_right, const void* sg_right, void* tr_gr,
                                void* tr_gl, double* current_spectrum, void* terminal,
                                void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !gr_diag || !tr_gr) return -1;
  if (terminal && (!sl_left || !sg_left || !sl_right || !sg_right || !gl_diag || !gg_diag))
    return -1;
  if (current_spectrum && (!gl_upper || !h_upper)) return -1;
  if (n_e == 0) return 0;
  dim3 grid(n_b, n_e);
  {
    ProfScope ps_observables_kernel(PROF_OTHER, (cudaStream_t)(stream));
    observables_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        n_b, bs, (const z_t*)gr_diag, (const z_t*)gl_diag, (const z_t*)gg_diag, (const z_t*)gl_upper,
        (const z_t*)h_upper, (const z_t*)sl_left, (const z_t*)sg_left, (const z_t*)sl_right,
        (const z_t*)sg_right, (z_t*)tr_gr, (z_t*)tr_gl, current_spectrum, (z_t*)terminal);
    NEGF_LAUNCHED();
  }
  return 0;
}

extern "C" {

int negf_g_identity_defect(int n_e, int n_b, int bs, const void* xr_diag, const void* xr_upper,
                           const void* xr_lower, const void* xl_diag, const void* xl_upper, const void* xg_diag,
                           const void* xg_upper, double* out, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !xr_diag || !xl_diag || !xg_diag || !out) return -1;
  if (n_b > 1 && (!xr_upper || !xr_lower || !xl_upper || !xg_upper)) return -1;
  if (n_e == 0) return 0;
  const int tiles = ((bs + 31) / 32) * ((bs + 31) / 32);
  dim3 grid(tiles, n_e * (2 * n_b - 1)), block(32, 8);
  {
    negf::ProfScope ps(negf::PROF_OTHER, (cudaStream_t)stream);
    negf::g_defect_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(
        n_b, bs, (const negf::z_t*)xr_diag, (const negf::z_t*)xr_upper, (const negf::z_t*)xr_lower,
        (const negf::z_t*)xl_diag, (const negf::z_t*)xl_upper, (const negf::z_t*)xg_diag, (const negf::z_t*)xg_upper,
        (unsigned long long*)out);
    NEGF_LAUNCHED();
  }
  return 0;
}

int negf_entry_identity_defect(long long n, const void* lesser, const void* greater, const void* ret_upper,
                               const void* ret_lower, double* out, void* stream) {
  if (n < 0 || !lesser || !greater || !ret_upper || !ret_lower || !out) return -1;
  if (n == 0) return 0;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  {
    negf::ProfScope ps(negf::PROF_OTHER, (cudaStream_t)stream);
    negf::entry_defect_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        n, (const negf::z_t*)lesser, (const negf::z_t*)greater, (const negf::z_t*)ret_upper,
        (const negf::z_t*)ret_lower, (unsigned long long*)out);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // extern "C"
