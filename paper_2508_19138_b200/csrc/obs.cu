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
