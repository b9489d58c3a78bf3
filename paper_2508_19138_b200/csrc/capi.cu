// extern "C" entry points declared in include/negf_b200.h.
#include "../../include/negf_b200.h"
#include "rgf.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

using namespace negf;

extern "C" {

int negf_abi_version(void) { return 100; }

size_t negf_rgf_workspace_bytes(int n_e, int n_b, int bs) {
  return rgf_workspace_bytes(n_e, n_b, bs);
}

int negf_rgf_selected_solve_batched(int n_e, int n_b, int bs, const void* m_diag,
                                    const void* m_upper, const void* m_lower, const void* bl_diag,
                                    const void* bl_upper, const void* bg_diag,
                                    const void* bg_upper, void* xr_diag, void* xr_upper,
                                    void* xr_lower, void* xl_diag, void* xl_upper, void* xg_diag,
                                    void* xg_upper, int symmetrize, int* status, double* u_spread,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !m_diag || !xr_diag) return -1;
  if (n_b > 1 && (!m_upper || !m_lower || !xr_upper || !xr_lower)) return -1;
  if ((bl_diag && !xl_diag) || (bg_diag && !xg_diag)) return -1;
  if (n_b > 1 && ((bl_diag && (!bl_upper || !xl_upper)) || (bg_diag && (!bg_upper || !xg_upper))))
    return -1;
  RgfArgs a;
  a.n_e = n_e; a.n_b = n_b; a.bs = bs;
  a.m_diag = (const z_t*)m_diag; a.m_upper = (const z_t*)m_upper; a.m_lower = (const z_t*)m_lower;
  a.b_diag[0] = (const z_t*)bl_diag; a.b_upper[0] = (const z_t*)bl_upper;
  a.b_diag[1] = (const z_t*)bg_diag; a.b_upper[1] = (const z_t*)bg_upper;
  a.xr_diag = (z_t*)xr_diag; a.xr_upper = (z_t*)xr_upper; a.xr_lower = (z_t*)xr_lower;
  a.xl_diag[0] = (z_t*)xl_diag; a.xl_upper[0] = (z_t*)xl_upper;
  a.xl_diag[1] = (z_t*)xg_diag; a.xl_upper[1] = (z_t*)xg_upper;
  a.symmetrize = symmetrize;
  a.status = status;
  a.u_spread = u_spread;
  return rgf_selected_solve(a, workspace, workspace_bytes, (cudaStream_t)stream);
}

int negf_zgemm_batched(int m, int n, int k, int batch, double alpha_re, double alpha_im,
                       const void* a, long long stride_a, int lda, int op_a, const void* b,
                       long long stride_b, int ldb, int op_b, double beta_re, double beta_im,
                       const void* c, long long stride_c, int ldc, void* d, long long stride_d,
                       int ldd, void* stream) {
  if (m < 0 || n < 0 || k < 0 || batch < 0 || !d) return -1;
  if (op_a < 0 || op_a > 3 || op_b < 0 || op_b > 3) return -1;
  ZGemmDesc g;
  g.M = m; g.N = n; g.batch = batch; g.nterms = 1;
  g.t[0] = zterm((const z_t*)a, stride_a, lda, op_a, (const z_t*)b, stride_b, ldb, op_b, k);
  g.t[1] = g.t[0];
  g.alpha = make_double2(alpha_re, alpha_im);
  g.beta = make_double2(beta_re, beta_im);
  g.C = (const z_t*)c; g.sC = stride_c; g.ldc = ldc;
  g.D = (z_t*)d; g.sD = stride_d; g.ldd = ldd; g.transD = 0;
  return zgemm_launch(g, (cudaStream_t)stream);
}

size_t negf_zinv_workspace_bytes(int n, int batch) { return zinv_workspace_bytes(n, batch); }

int negf_zinv_batched(int n, int batch, void* s, void* x, int* status, double* u_spread,
                      void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || batch < 0 || !s || !x) return -1;
  InvAux aux;
  aux.status = status; aux.status_code = 1; aux.u_spread = u_spread; aux.spread_stride = 1;
  long long s2 = (long long)n * n;
  return zinv_batched((z_t*)s, s2, n, (z_t*)x, s2, n, n, batch, aux, workspace, workspace_bytes,
                      (cudaStream_t)stream);
}

}  // extern "C"
